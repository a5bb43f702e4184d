"""Launch timeline of one untimed build + solve (gaps = host work / syncs)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2404_11894_b200 import _native as N
from paper_2404_11894_b200.harness.config import RenderConfig
from paper_2404_11894_b200.pathgraph import build_graph, solve
from paper_2404_11894_b200.scenes import WORKLOADS
from paper_2404_11894_b200.transport import render_pt

wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
cfg = RenderConfig(spp=wl.spp, max_depth=wl.max_depth, seed=0)
out = render_pt(wl.scene(), cfg, with_records=True)
for _ in range(2):
    g = build_graph(out, 32, seed=0); solve(g, wl.iterations, 0.0); del g
torch.cuda.synchronize()
N.profile_reset(); N.profile(True)
g = build_graph(out, 32, seed=0); solve(g, wl.iterations, 0.0)
torch.cuda.synchronize()
tl = N.profile_timeline(); N.profile(False)
prev_end = 0.0
for name, st, du in tl:
    gap = st - prev_end
    print(f"{st:8.3f} {du:7.3f} gap {gap:6.3f}  {name}")
    prev_end = max(prev_end, st + du)
print("end", round(prev_end, 3), "ms")
