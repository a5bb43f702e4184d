"""A small end-to-end pass for compute-sanitizer (memcheck / racecheck):
golden C1 records (46 k, one class: speculative center draw, deferred
splits, part B on its own stream) and the two-class floor set, build +
solve + splat, plus the VPGR device codec."""
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from conftest import GOLDEN, golden  # noqa: E402
from test_gpu_graph import _trace_from_golden  # noqa: E402
from paper_2404_11894_b200.pathgraph import build_graph, solve, splat_output  # noqa: E402
from paper_2404_11894_b200.transport import load_records, save_records  # noqa: E402

for name, K in (("c1_16", 32), ("c1floor_16", 8)):
    z = golden(name)
    t = _trace_from_golden(z)
    g = build_graph(t, K, seed=int(z["seed"]))
    r = solve(g, iterations=5, tol=0.0)
    img = splat_output(g, r)
    print(name, K, g.info()["n_clusters"], float(np.abs(img).sum()))
dev = load_records(os.path.join(GOLDEN, "c1_8.vpgr"), device=True)
with tempfile.TemporaryDirectory() as d:
    save_records(os.path.join(d, "x.vpgr"), dev)
torch.cuda.synchronize()
print("sanitize run ok")
