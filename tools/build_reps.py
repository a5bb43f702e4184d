"""Wall time of repeated build+solve calls on one traced C2 frame (diagnostic)."""
import sys, time, json
sys.path.insert(0, sys.argv[2] if len(sys.argv) > 2 else ".")
import torch
from paper_2404_11894_b200.scenes import WORKLOADS
from paper_2404_11894_b200.harness.config import RenderConfig
from paper_2404_11894_b200.transport import render_pt
from paper_2404_11894_b200.pathgraph import build_graph, solve
wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
cfg = RenderConfig(spp=wl.spp, max_depth=wl.max_depth, seed=0)
out = render_pt(wl.scene(), cfg, with_records=True)
bt, st = [], []
g = None
import os
for rep in range(int(os.environ.get("REPS", "25"))):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    g = build_graph(out, 32, seed=0)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    r = solve(g, 10, 0.0); torch.cuda.synchronize(); t2 = time.perf_counter()
    bt.append(round((t1 - t0) * 1e3, 2)); st.append(round((t2 - t1) * 1e3, 2))
print(json.dumps({"build_ms": bt, "solve_ms": st}))
