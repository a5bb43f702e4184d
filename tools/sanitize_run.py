"""A small end-to-end pass for compute-sanitizer (memcheck / racecheck /
synccheck): the reference's C1 record set at full size (46 k records, one
class: speculative center draw, deferred splits, part B on its own stream;
conftest.scale_case), the two-class floor set at K = 8 (many splits), the
mixed scene (stored W blocks for the Lambertian classes beside recomputed
ones), the device tracer, reconstruct_path_estimate and the VPGR codec."""
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from conftest import GOLDEN, golden, scale_case  # noqa: E402
from test_gpu_graph import _trace_from_golden  # noqa: E402
from paper_2404_11894_b200 import scenes as S  # noqa: E402
from paper_2404_11894_b200.harness.config import RenderConfig  # noqa: E402
from paper_2404_11894_b200.pathgraph import build_graph, render_pg, solve, splat_output  # noqa: E402
from paper_2404_11894_b200.transport import (load_records, reconstruct_path_estimates,  # noqa: E402
                                             save_records)
from paper_2404_11894_b200.transport.records import PathSoA, RecordSoA, TraceOutput  # noqa: E402

z, rec, paths = scale_case("c1_s0")
t = TraceOutput(None, RecordSoA(**rec), PathSoA(**paths), 64, 64, 4)
g = build_graph(t, 32, seed=0)
r = solve(g, iterations=5, tol=0.0)
print("c1 full", t.records.n, g.info()["n_clusters"], float(np.abs(splat_output(g, r)).sum()))
for name, K in (("c1floor_16", 8), ("mixed_12", 16)):
    zz = golden(name)
    tt = _trace_from_golden(zz)
    gg = build_graph(tt, K, seed=int(zz["seed"]))
    rr = solve(gg, iterations=5, tol=0.0)
    print(name, K, gg.info()["n_clusters"], float(np.abs(splat_output(gg, rr)).sum()))
    _ = gg.w_indirect  # the CSR export, recomputed and stored blocks
pg = render_pg(S.scene_mixed((16, 16)), RenderConfig(mode="pg", spp=2, max_depth=16, seed=2,
                                                     iterations=4, tol=0.0))
est, diff = reconstruct_path_estimates(pg.trace.records, pg.trace.paths)
print("render_pg mixed", pg.trace.records.n, float(np.abs(est).sum()))
dev = load_records(os.path.join(GOLDEN, "c1_8.vpgr"), device=True)
with tempfile.TemporaryDirectory() as d:
    save_records(os.path.join(d, "x.vpgr"), dev)
torch.cuda.synchronize()
print("sanitize run ok")
