"""The kernel bench.py's roofline names, launched under ncu by bench.py for
its in-run DRAM traffic: trace the workload, build, run 3 iterations (bench.py
profiles the third k_solve_iter launch, a steady-state one)."""
import sys

sys.path.insert(0, ".")
from paper_2404_11894_b200.harness.config import RenderConfig  # noqa: E402
from paper_2404_11894_b200.pathgraph import build_graph, solve  # noqa: E402
from paper_2404_11894_b200.scenes import WORKLOADS  # noqa: E402
from paper_2404_11894_b200.transport import render_pt  # noqa: E402

wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
out = render_pt(wl.scene(), RenderConfig(spp=wl.spp, max_depth=wl.max_depth, seed=0),
                with_records=True)
g = build_graph(out, 32, seed=0)
solve(g, iterations=3, tol=0.0)
