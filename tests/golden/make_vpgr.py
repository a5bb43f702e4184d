"""VPGR fixture from the reference itself (records.py:191-256 format).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_vpgr.py

Writes tests/golden/c1_8.vpgr (a record dump written by the reference's
save_records) and c1_8_vpgr.npz (the reference's solve_from_records image
and SolveResult on that dump).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

from make_golden import to_ref  # noqa: E402
from volpg.harness.config import RenderConfig as RefConfig  # noqa: E402
from volpg.pathgraph.pipeline import solve_from_records  # noqa: E402
from volpg.transport import load_records, render_pt, save_records  # noqa: E402

from paper_2404_11894_b200 import scenes as S  # noqa: E402

K, ITERS, SEED = 8, 6, 3


def main():
    scene = to_ref(S.scene_c1((8, 8), floor=True))
    cfg = RefConfig(mode="pg", spp=2, max_depth=16, seed=SEED)
    out = render_pt(scene, cfg, with_records=True)
    path = os.path.join(HERE, "c1_8.vpgr")
    save_records(path, out)
    trace = load_records(path)
    image, graph, result = solve_from_records(trace, K, iterations=ITERS, tol=0.0, seed=SEED)
    np.savez_compressed(os.path.join(HERE, "c1_8_vpgr.npz"), image=image,
                        incoming=result.incoming, i_bar=result.i_bar,
                        residuals=np.array(result.residuals), K=K, iterations=ITERS, seed=SEED,
                        cluster_id=trace.records.cluster_id)
    print(path, out.records.n, "records")


if __name__ == "__main__":
    main()
