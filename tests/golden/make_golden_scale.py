"""Golden vectors at the benchmarked scenes' scale, by running the reference
in this container (C1 at full size for seeds 0/1/2, and the
C2/C3/C4 slices 96²x8, 64²x16, 96²x16 — 0.3-0.7 M vertices each).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden_scale.py [case ...]

Compact fixtures (tests/golden/scale_<case>.npz), because the record sets are
tens of MB:

- the records themselves are NOT stored.  The test regenerates them with the
  oracle's C tracer restatement (oracle/tracer_oracle.c) and applies a stored
  bitwise XOR patch per field, which this script computes against the
  reference's own records (all zero where the restatement is already
  bit-identical, so it compresses to almost nothing).  After the patch the
  test holds exactly the reference's record set (checked by sha256);
- cluster_id / centers / member lists / CSR indptr+indices: sha256 of their
  int64 bytes (bit-exact parity), plus counts;
- p-hat, D-bar, W rows, incoming, i_bar on 4096 sampled rows (fp64);
  residuals and the full pg and PT images (fp64);
- C1 seeds 0/1/2 also keep the reference's end-to-end `render_pg` image
  (pipeline.py:25-42) for the image-band parity test.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from volpg.harness.config import RenderConfig as RefConfig  # noqa: E402
from volpg.pathgraph import build_graph, render_pg, solve, splat_output  # noqa: E402
from volpg.transport import render_pt  # noqa: E402

from make_golden import PATH_FIELDS, REC_FIELDS, to_ref  # noqa: E402
from oracle import tracer_oracle as T  # noqa: E402
from paper_2404_11894_b200 import scenes as S  # noqa: E402
from paper_2404_11894_b200.harness.config import RenderConfig  # noqa: E402

# name: (scene factory, spp, max_depth, seed, iterations, render_pg too)
CASES = {
    "c1_s0": (lambda: S.scene_c1((64, 64)), 4, 16, 0, 10, True),
    "c1_s1": (lambda: S.scene_c1((64, 64)), 4, 16, 1, 10, True),
    "c1_s2": (lambda: S.scene_c1((64, 64)), 4, 16, 2, 10, True),
    "c2_slice": (lambda: S.scene_c2((96, 96)), 8, 64, 0, 10, False),
    "c3_slice": (lambda: S.scene_c3((64, 64)), 16, 64, 0, 10, False),
    "c4_slice": (lambda: S.scene_c4((96, 96)), 16, 64, 0, 16, False),
}
K = 32
N_SAMPLE = 4096
PATCHED_PATH_FIELDS = ["cam_weight", "d_cam", "direct0", "direct0_nee", "direct0_phase",
                       "pt_estimate"]


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


def sha_raw(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def xor_patch(ref: np.ndarray, mine: np.ndarray) -> np.ndarray:
    ref = np.ascontiguousarray(ref)
    mine = np.ascontiguousarray(mine, dtype=ref.dtype)
    u = {1: np.uint8, 4: np.uint32, 8: np.uint64}[ref.dtype.itemsize]
    return ref.view(u) ^ mine.view(u)


def dump(name, factory, spp, max_depth, seed, iters, with_pg):
    t0 = time.time()
    scene = factory()
    ref_scene = to_ref(scene)
    cfg = RefConfig(spp=spp, max_depth=max_depth, seed=seed)
    trace = render_pt(ref_scene, cfg, with_records=True)
    rec_o, path_o = T.trace_records(scene, RenderConfig(spp=spp, max_depth=max_depth, seed=seed))
    r, p = trace.records, trace.paths
    if not np.array_equal(p.rec_count, path_o["rec_count"]):
        bad = np.flatnonzero(p.rec_count != path_o["rec_count"])
        raise SystemExit(f"{name}: {bad.size} paths differ in length between the reference and "
                         "the C tracer restatement; a patch cannot bridge that")
    out = {"width": trace.width, "height": trace.height, "spp": spp, "seed": seed,
           "max_depth": max_depth, "iterations": iters, "cluster_size": K, "n": r.n}
    n_patched = 0
    for f in REC_FIELDS:
        x = xor_patch(getattr(r, f), rec_o[f])
        n_patched += int(np.count_nonzero(x))
        out["xrec_" + f] = x
        out["sha_rec_" + f] = sha_raw(getattr(r, f))
    for f in PATCHED_PATH_FIELDS:
        x = xor_patch(getattr(p, f), path_o[f])
        n_patched += int(np.count_nonzero(x))
        out["xpath_" + f] = x
    out["n_patched_words"] = n_patched
    out["pt_image"] = trace.image
    t1 = time.time()
    graph = build_graph(trace, K, seed=seed)
    t2 = time.time()
    res = solve(graph, iterations=iters, tol=0.0)
    t3 = time.time()
    cl = graph.clusters
    sizes = np.array([len(c.members) for c in cl], dtype=np.int64)
    out["n_clusters"] = len(cl)
    out["sha_cluster_id"] = sha(graph.records.cluster_id)
    out["sha_centers"] = sha([c.center for c in cl])
    out["sha_cl_off"] = sha(np.concatenate([[0], np.cumsum(sizes)]))
    out["sha_members"] = sha(np.concatenate([c.members for c in cl]))
    out["sha_next_idx"] = sha(graph.next_idx)
    W = graph.w_indirect
    out["sha_w_indptr"] = sha(W.indptr)
    out["sha_w_indices"] = sha(W.indices)
    out["nnz"] = W.nnz
    rows = np.sort(np.random.default_rng(12345).choice(r.n, min(N_SAMPLE, r.n), replace=False))
    out["sample_rows"] = rows
    for a in ("phat_ind", "phat_dir_phase", "phat_dir_emit", "d_bar"):
        out["s_" + a] = getattr(graph, a)[rows]
    for a in ("included_phase", "included_emit"):
        out["sha_" + a] = sha(getattr(graph, a))
    out["s_w_data"] = np.concatenate([W.data[W.indptr[q]:W.indptr[q + 1]] for q in rows])
    out["s_incoming"], out["s_i_bar"] = res.incoming[rows], res.i_bar[rows]
    out["residuals"] = np.array(res.residuals)
    out["image"] = splat_output(graph, res)
    out["ref_seconds"] = np.array([t1 - t0, t2 - t1, t3 - t2])
    if with_pg:
        pg = render_pg(ref_scene, RefConfig(mode="pg", spp=spp, max_depth=max_depth, seed=seed,
                                            iterations=iters))
        out["render_pg_image"] = pg.image
        out["render_pg_iterations"] = pg.result.iterations
    np.savez_compressed(os.path.join(HERE, f"scale_{name}.npz"), **out)
    print(f"{name}: {r.n} records, {len(cl)} clusters, {n_patched} patched words, "
          f"trace {t1 - t0:.1f} s, build {t2 - t1:.1f} s, solve {t3 - t2:.1f} s", flush=True)


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for nm in names:
        dump(nm, *CASES[nm])
