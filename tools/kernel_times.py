"""Per-kernel device times (CUDA events around each launch) of build+solve."""
import sys, json
sys.path.insert(0, ".")
import torch
from paper_2404_11894_b200 import _native as N
from paper_2404_11894_b200.scenes import WORKLOADS
from paper_2404_11894_b200.harness.config import RenderConfig
from paper_2404_11894_b200.transport import render_pt
from paper_2404_11894_b200.pathgraph import build_graph, solve
wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
cfg = RenderConfig(spp=wl.spp, max_depth=wl.max_depth, seed=0)
out = render_pt(wl.scene(), cfg, with_records=True)
for rep in range(2):
    g = build_graph(out, 32, seed=0); solve(g, wl.iterations, 0.0); del g
torch.cuda.synchronize()
N.profile_reset(); N.profile(True)
g = build_graph(out, 32, seed=0); solve(g, wl.iterations, 0.0)
torch.cuda.synchronize()
prof = N.profile_read(); N.profile(False)
tot = sum(ms for _, ms in prof.values())
for k, (c, ms) in sorted(prof.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:40s} {c:4d} {ms:8.3f} ms {100*ms/tot:5.1f}%")
print("kernel total", round(tot, 3), "ms")
