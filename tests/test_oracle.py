"""The CPU oracle is pinned against the reference's own outputs (goldens made
by tests/golden/make_golden.py running /root/reference in this container)."""

import numpy as np
import pytest

from conftest import golden
from oracle import pathgraph_oracle as O

CASES = [("c1_16", 32), ("c1_16", 8), ("c1_16", 1), ("c1floor_16", 32), ("cloud_16", 32),
         ("mixed_12", 16),
         ("dense_12", 32)]


def _graph(name, K):
    z = golden(name)
    rec, paths = O.load_golden_records(z)
    g = O.build_graph(rec, paths, int(z["width"]), int(z["height"]), int(z["spp"]), K,
                      int(z["seed"]))
    return z, g


@pytest.mark.parametrize("name,K", CASES)
def test_oracle_graph_matches_reference(name, K):
    z, g = _graph(name, K)
    p = f"K{K}_"
    assert np.array_equal(g.cluster_id, z[p + "cluster_id"])
    assert np.array_equal([c.center for c in g.clusters], z[p + "centers"])
    assert np.array_equal(np.concatenate([c.members for c in g.clusters]), z[p + "members"])
    assert np.array_equal(g.next_idx, z[p + "next_idx"])
    assert np.array_equal(g.w.indptr, z[p + "w_indptr"])
    assert np.array_equal(g.w.indices, z[p + "w_indices"])
    np.testing.assert_allclose(g.w.data, z[p + "w_data"], rtol=1e-12, atol=0)
    for a in ("phat_ind", "phat_dir_phase", "phat_dir_emit", "d_bar"):
        np.testing.assert_allclose(getattr(g, a), z[p + a], rtol=1e-12, atol=1e-300)
    for a in ("included_phase", "included_emit"):
        assert np.array_equal(getattr(g, a), z[p + a])


@pytest.mark.parametrize("name,K", CASES)
def test_oracle_solve_and_splat_match_reference(name, K):
    z, g = _graph(name, K)
    p = f"K{K}_"
    for iters in (0, 1, 10):
        inc, ib, res, perf = O.solve(g, iters, 0.0)
        q = f"{p}it{iters}_"
        np.testing.assert_allclose(inc, z[q + "incoming"], rtol=1e-11, atol=1e-300)
        np.testing.assert_allclose(ib, z[q + "i_bar"], rtol=1e-11, atol=1e-300)
        np.testing.assert_allclose(res, z[q + "residuals"], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(O.splat(g, ib), z[q + "image"], rtol=1e-11, atol=1e-300)
        np.testing.assert_allclose(O.splat(g, ib, "aggregated"), z[q + "image_aggdirect"],
                                   rtol=1e-11, atol=1e-300)
    inc, ib, res, perf = O.solve(g, 10, 1e-3)
    assert perf == int(z[p + "tol_iterations"])
    np.testing.assert_allclose(res, z[p + "tol_residuals"], rtol=1e-9, atol=1e-12)


def test_oracle_clustering_tail_shuffle_sizes():
    z = golden("clustering")
    for tag in ("c1_48", "c1floor_40"):
        rng = np.random.default_rng(np.random.SeedSequence([int(z[tag + "_seed"]) & 0xFFFFFFFF,
                                                            0xC1A5]))
        cid, cl = O.cluster_points(z[tag + "_pos"], z[tag + "_keys"], 32, rng)
        assert np.array_equal(cid, z[tag + "_cluster_id"])
        assert np.array_equal([c.center for c in cl], z[tag + "_centers"])
        after = np.array([int(x) for x in rng.integers(0, 2**62, size=4)])
        assert np.array_equal(after, z[tag + "_rng_after"])  # same RNG consumption


def test_oracle_dense_matches_reference_dense():
    z = golden("dense_micro")
    rec, paths = O.load_golden_records(z)
    for K in (1, 2, 4, 8):
        g = O.build_graph(rec, paths, int(z["width"]), int(z["height"]), int(z["spp"]), K, 3)
        assert np.array_equal(g.cluster_id, z[f"K{K}_cluster_id"])
        inc, ib = O.dense_solve(g, 6)
        np.testing.assert_allclose(inc, z[f"K{K}_incoming"], rtol=1e-10, atol=1e-300)
        np.testing.assert_allclose(ib, z[f"K{K}_i_bar"], rtol=1e-10, atol=1e-300)
        # matrix-free equals dense (SPEC.md acceptance 2)
        inc2, ib2, _, _ = O.solve(g, 6, 0.0)
        np.testing.assert_allclose(inc2, inc, rtol=1e-9, atol=1e-14)


def test_oracle_pt_image_and_k1_identity():
    z = golden("c1_16")
    rec, paths = O.load_golden_records(z)
    w, h, spp = int(z["width"]), int(z["height"]), int(z["spp"])
    np.testing.assert_array_equal(O.splat_pt(paths, w, h, spp), z["pt_image"])
    np.testing.assert_array_equal(z["pt_image"], z["pt_image_free"])
    g = O.build_graph(rec, paths, w, h, spp, 1, int(z["seed"]))
    inc, ib, _, _ = O.solve(g, 10, 0.0)
    np.testing.assert_allclose(O.splat(g, ib), z["pt_image"], rtol=1e-5, atol=1e-12)


# the C tracer restatement vs the reference's own records (same scenes and
# settings as tests/golden/make_golden.py)
TRACE_GOLDENS = {
    "c1_16": ("scene_c1", dict(res=(16, 16)), 4, 16, 0),
    "c1floor_16": ("scene_c1", dict(res=(16, 16), floor=True), 4, 16, 1),
    "cloud_16": ("scene_c2", dict(res=(16, 16), grid_n=16), 4, 64, 2),
    "dense_12": ("scene_c3", dict(res=(12, 12)), 2, 64, 0),
    "mixed_12": ("scene_mixed", dict(res=(12, 12)), 4, 32, 4),
}


@pytest.mark.parametrize("name", list(TRACE_GOLDENS))
def test_tracer_oracle_matches_reference_records(name):
    from oracle import tracer_oracle as T
    from paper_2404_11894_b200 import scenes as S
    from paper_2404_11894_b200.harness.config import RenderConfig

    fac, kw, spp, md, seed = TRACE_GOLDENS[name]
    z = golden(name)
    rec, paths = T.trace_records(getattr(S, fac)(**kw), RenderConfig(spp=spp, max_depth=md,
                                                                       seed=seed))
    ref_rec, ref_paths = O.load_golden_records(z)
    assert np.array_equal(paths["rec_count"], ref_paths["rec_count"])
    for f, v in rec.items():
        np.testing.assert_allclose(v, ref_rec[f], rtol=1e-12, atol=0, err_msg=f)
    for f in ("cam_weight", "d_cam", "direct0", "pt_estimate"):
        np.testing.assert_allclose(paths[f], ref_paths[f], rtol=1e-12, atol=0, err_msg=f)


def test_faithful_clustering_equals_fast_clustering():
    """The cost-faithful variant (the reference's per-cell loop and per-center
    groups, used by bench.py's reference arm) gives the reference's clusters."""
    z = golden("c1_16")
    rec, paths = O.load_golden_records(z)
    for K in (32, 8):
        g = O.build_graph(rec, paths, int(z["width"]), int(z["height"]), int(z["spp"]), K,
                          int(z["seed"]), faithful=True)
        assert np.array_equal(g.cluster_id, z[f"K{K}_cluster_id"])
