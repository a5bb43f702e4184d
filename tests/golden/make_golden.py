"""Generate golden vectors by running the reference package in this container.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

The reference (/root/reference, `volpg` 0.1.0) is imported read-only; it does
not exist on the GPU box, so its outputs are committed here as small .npz
fixtures.  Scenes come from paper_2404_11894_b200.scenes (my scene vocabulary
mirrors the reference's field names, so they convert 1:1).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import volpg  # noqa: E402  (the reference)
from volpg.harness.config import RenderConfig as RefConfig  # noqa: E402
from volpg.pathgraph import build_graph, solve, splat_output  # noqa: E402
from volpg.pathgraph.clustering import cluster_points  # noqa: E402
from volpg.pathgraph.dense import dense_solve  # noqa: E402
from volpg.transport import record_extra_direct, render_pt  # noqa: E402

from paper_2404_11894_b200 import scenes as S  # noqa: E402

REC_FIELDS = ["pos", "omega_out", "normal", "coeff", "g", "phase_dir", "pdf_phase",
              "pdf_emit_at_phase", "emit_dir", "pdf_emit", "d_emit", "d_phase", "i_pt", "w_cont",
              "kind", "emit_delta", "class_id", "path_idx", "depth"]
PATH_FIELDS = ["pixel_idx", "rec_start", "rec_count", "cam_weight", "d_cam", "direct0",
               "direct0_nee", "direct0_phase", "extra_direct", "pt_estimate"]


def to_ref(scene):
    """My Scene -> the reference's Scene (identical field names)."""
    from dataclasses import asdict, fields

    def conv(obj, cls):
        kw = {f.name: getattr(obj, f.name) for f in fields(obj)}
        return cls(**kw)

    return volpg.Scene(
        camera=conv(scene.camera, volpg.Camera),
        media=[conv(m, volpg.Medium) for m in scene.media],
        surfaces=[conv(s, volpg.Surface) for s in scene.surfaces],
        emitters=[conv(e, volpg.Emitter) for e in scene.emitters],
    )


CASES = {
    # name: (scene factory, spp, max_depth, seed, K list, n_extra)
    "c1_16": (lambda: S.scene_c1((16, 16)), 4, 16, 0, [32, 8, 1], 0),
    "c1floor_16": (lambda: S.scene_c1((16, 16), floor=True), 4, 16, 1, [32], 3),
    "cloud_16": (lambda: S.scene_c2((16, 16), grid_n=16), 4, 64, 2, [32], 0),
    "dense_12": (lambda: S.scene_c3((12, 12)), 2, 64, 0, [32], 0),
    "mixed_12": (lambda: S.scene_mixed((12, 12)), 4, 32, 4, [16], 2),
}


def dump_case(name, factory, spp, max_depth, seed, ks, n_extra):
    scene = to_ref(factory())
    cfg = RefConfig(spp=spp, max_depth=max_depth, seed=seed)
    img_free = render_pt(scene, cfg, with_records=False).image
    trace = render_pt(scene, cfg, with_records=True)
    out = {"width": trace.width, "height": trace.height, "spp": trace.spp, "seed": seed,
           "max_depth": max_depth, "pt_image": trace.image, "pt_image_free": img_free}
    if n_extra:
        out["extra_direct"] = record_extra_direct(scene, trace, n_extra, seed=seed).copy()
        out["n_extra"] = n_extra
    for f in REC_FIELDS:
        out["rec_" + f] = getattr(trace.records, f)
    for f in PATH_FIELDS:
        out["path_" + f] = getattr(trace.paths, f)
    for K in ks:
        graph = build_graph(trace, K, seed=seed)
        p = f"K{K}_"
        out[p + "cluster_id"] = graph.records.cluster_id.copy()
        out[p + "centers"] = np.array([c.center for c in graph.clusters], dtype=np.int64)
        sizes = np.array([len(c.members) for c in graph.clusters], dtype=np.int64)
        out[p + "cl_off"] = np.concatenate([[0], np.cumsum(sizes)])
        out[p + "members"] = (np.concatenate([c.members for c in graph.clusters])
                              if graph.clusters else np.zeros(0, dtype=np.int64))
        out[p + "next_idx"] = graph.next_idx
        for a in ("phat_ind", "phat_dir_phase", "phat_dir_emit", "included_phase",
                  "included_emit", "d_bar"):
            out[p + a] = getattr(graph, a)
        W = graph.w_indirect
        out[p + "w_indptr"], out[p + "w_indices"], out[p + "w_data"] = W.indptr, W.indices, W.data
        for iters in (0, 1, 10):
            res = solve(graph, iterations=iters, tol=0.0)
            q = f"{p}it{iters}_"
            out[q + "incoming"], out[q + "i_bar"] = res.incoming, res.i_bar
            out[q + "residuals"] = np.array(res.residuals)
            out[q + "image"] = splat_output(graph, res)
            out[q + "image_aggdirect"] = splat_output(graph, res, aggregate_direct_term=True)
            if n_extra:
                out[q + "image_extra"] = splat_output(graph, res, extra_direct=True)
        res = solve(graph, iterations=10, tol=1e-3)  # default tol: early stop path
        out[p + "tol_residuals"] = np.array(res.residuals)
        out[p + "tol_iterations"] = res.iterations
        out[p + "tol_incoming"] = res.incoming
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, "records", trace.records.n, "paths", trace.paths.n)


def dump_clustering():
    """Clustering-only goldens at sizes that take numpy's tail-shuffle branch."""
    out = {}
    for tag, factory, spp, seed in (("c1_48", lambda: S.scene_c1((48, 48)), 4, 0),
                                    ("c1floor_40", lambda: S.scene_c1((40, 40), floor=True), 4, 5)):
        scene = to_ref(factory())
        trace = render_pt(scene, RefConfig(spp=spp, max_depth=16, seed=seed), with_records=True)
        r = trace.records
        keys = r.kind.astype(np.int64) * (1 << 32) + r.class_id.astype(np.int64)
        rng = np.random.default_rng(np.random.SeedSequence([seed & 0xFFFFFFFF, 0xC1A5]))
        cid, clusters = cluster_points(r.pos, keys, 32, rng)
        out[tag + "_pos"] = r.pos
        out[tag + "_keys"] = keys
        out[tag + "_seed"] = seed
        out[tag + "_cluster_id"] = cid
        out[tag + "_centers"] = np.array([c.center for c in clusters], dtype=np.int64)
        out[tag + "_rng_after"] = np.array([int(x) for x in rng.integers(0, 2**62, size=4)])
        print(tag, "points", r.n, "clusters", len(clusters))
    np.savez_compressed(os.path.join(HERE, "clustering.npz"), **out)


def dump_dense():
    """Dense-operator oracle (dense.py) on micro graphs (SPEC acceptance 2)."""
    out = {}
    scene = to_ref(S.scene_c1((6, 6), floor=True))
    trace = render_pt(scene, RefConfig(spp=2, max_depth=16, seed=3), with_records=True)
    for f in REC_FIELDS:
        out["rec_" + f] = getattr(trace.records, f)
    for f in PATH_FIELDS:
        out["path_" + f] = getattr(trace.paths, f)
    out["width"], out["height"], out["spp"] = trace.width, trace.height, trace.spp
    for K in (1, 2, 4, 8):
        graph = build_graph(trace, K, seed=3)
        inc, ib = dense_solve(graph, 6)
        out[f"K{K}_incoming"], out[f"K{K}_i_bar"] = inc, ib
        out[f"K{K}_cluster_id"] = graph.records.cluster_id.copy()
    np.savez_compressed(os.path.join(HERE, "dense_micro.npz"), **out)
    print("dense micro records", trace.records.n)


if __name__ == "__main__":
    for name, spec in CASES.items():
        dump_case(name, *spec)
    dump_clustering()
    dump_dense()
