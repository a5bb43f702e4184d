"""Per-stage wall times of build_graph on a workload (diagnostic)."""
import sys, time, json
sys.path.insert(0, ".")
import torch
from paper_2404_11894_b200.scenes import WORKLOADS
from paper_2404_11894_b200.harness.config import RenderConfig
from paper_2404_11894_b200.transport import render_pt
from paper_2404_11894_b200.pathgraph import build_graph, solve
wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
cfg = RenderConfig(spp=wl.spp, max_depth=wl.max_depth, seed=0)
out = render_pt(wl.scene(), cfg, with_records=True)
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    g = build_graph(out, 32, seed=0, timings=True)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    r = solve(g, 10, 0.0); torch.cuda.synchronize(); t2 = time.perf_counter()
    info = g.info()
    print(json.dumps({"n": out.records.n, "build_total_ms": (t1-t0)*1e3, "solve_ms": (t2-t1)*1e3,
                      "stages_ms": [round(x, 3) for x in info["build_ms"]], "splits": info["n_splits"], "fallback": info["n_fallback"], "staged": info["n_staged"], "visits": info["split_visits"]}))
# wall time without stage synchronisation (the overlap is only real then)
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    g = build_graph(out, 32, seed=0, timings=False)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    r = solve(g, 10, 0.0); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(json.dumps({"untimed_build_ms": (t1 - t0) * 1e3, "solve_ms": (t2 - t1) * 1e3}))
