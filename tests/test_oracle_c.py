"""The C restatement of the path-graph build (oracle/graph_oracle.c) is
pinned against the reference's own outputs (goldens made by
tests/golden/make_golden.py running /root/reference in this container) and
against numpy's Generator draws, so it can stand in for the reference at the
benchmarked sizes where neither the reference nor the numpy oracle finish in
seconds."""

import numpy as np
import pytest

from conftest import golden
from oracle import graph_oracle as G
from oracle import pathgraph_oracle as O

CASES = [("c1_16", 32), ("c1_16", 8), ("c1_16", 1), ("c1floor_16", 32), ("cloud_16", 32),
         ("mixed_12", 16), ("dense_12", 32)]


@pytest.mark.parametrize("n,m", [(10, 10), (10, 3), (5000, 200), (10001, 250), (10001, 201),
                                 (20000, 400), (20000, 401), (100000, 3125), (50, 0), (1, 1),
                                 (70000, 70000)])
def test_choice_matches_numpy(n, m):
    """Generator.choice(n, m, replace=False): both branches (tail shuffle for
    n > 10000 and m > n // 50, Floyd otherwise) and the state after."""
    a = np.random.default_rng(np.random.SeedSequence([n * 7 + m, 0xC1A5]))
    b = np.random.default_rng(np.random.SeedSequence([n * 7 + m, 0xC1A5]))
    a.integers(5)  # leave a buffered 32-bit half behind
    b.integers(5)
    assert np.array_equal(G.rng_choice(a, n, m), b.choice(n, size=m, replace=False))
    assert a.bit_generator.state == b.bit_generator.state


def test_integers_matches_numpy():
    a = np.random.default_rng(3)
    b = np.random.default_rng(3)
    for k in [1, 2, 3, 7, 64, 65, 100, 1000, 2**31 - 1, 2**32 - 1, 2**32, 2**33 + 5, 2**62]:
        for _ in range(5):
            assert G.rng_integers(a, k) == int(b.integers(k))
    assert a.bit_generator.state == b.bit_generator.state


@pytest.mark.parametrize("name,K", CASES)
def test_c_oracle_graph_matches_reference(name, K):
    z = golden(name)
    rec, paths = O.load_golden_records(z)
    g = G.build_graph(rec, paths, int(z["width"]), int(z["height"]), int(z["spp"]), K,
                      int(z["seed"]))
    p = f"K{K}_"
    assert np.array_equal(g.cluster_id, z[p + "cluster_id"])
    assert np.array_equal(g.centers, z[p + "centers"])
    assert np.array_equal(g.members, z[p + "members"])
    assert np.array_equal(g.member_off, z[p + "cl_off"])
    for a in ("phat_ind", "phat_dir_phase", "phat_dir_emit", "d_bar"):
        np.testing.assert_allclose(getattr(g, a), z[p + a], rtol=1e-12, atol=1e-300)
    for a in ("included_phase", "included_emit"):
        assert np.array_equal(getattr(g, a), z[p + a])
    # W: the reference's CSR rows are the cluster blocks' rows (graph.py:167)
    indptr, indices, data = z[p + "w_indptr"], z[p + "w_indices"], z[p + "w_data"]
    for c in range(g.centers.shape[0]):
        mem = g.members[g.member_off[c]:g.member_off[c + 1]]
        blk = g.w.row_block(c)
        for rr, r in enumerate(mem):
            assert np.array_equal(indices[indptr[r]:indptr[r + 1]], mem)
            np.testing.assert_allclose(blk[rr], data[indptr[r]:indptr[r + 1]], rtol=1e-12, atol=0)
    for iters in (0, 1, 10):
        inc, ib, res, perf = O.solve(g, iters, 0.0)
        q = f"{p}it{iters}_"
        np.testing.assert_allclose(inc, z[q + "incoming"], rtol=1e-11, atol=1e-300)
        np.testing.assert_allclose(ib, z[q + "i_bar"], rtol=1e-11, atol=1e-300)
        np.testing.assert_allclose(O.splat(g, ib), z[q + "image"], rtol=1e-11, atol=1e-300)


def test_c_oracle_clustering_tail_shuffle_sizes():
    z = golden("clustering")
    for tag in ("c1_48", "c1floor_40"):
        rng = np.random.default_rng(np.random.SeedSequence([int(z[tag + "_seed"]) & 0xFFFFFFFF,
                                                            0xC1A5]))
        cid, off, mem, cen, _ = G.cluster_points(z[tag + "_pos"], z[tag + "_keys"], 32, rng)
        assert np.array_equal(cid, z[tag + "_cluster_id"])
        assert np.array_equal(cen, z[tag + "_centers"])
        after = np.array([int(x) for x in rng.integers(0, 2**62, size=4)])
        assert np.array_equal(after, z[tag + "_rng_after"])  # same RNG consumption


@pytest.mark.parametrize("seed", [0, 1])
def test_c_oracle_equals_numpy_oracle_on_hard_sets(seed):
    """Clumps, coincident points, far outliers (the brute-force fallback) and
    several classes: the C clustering equals the numpy restatement."""
    r = np.random.default_rng(seed)
    clumps = r.normal(size=(40, 3)) * 3
    pts = np.concatenate([clumps[r.integers(0, 40, 30000)] + r.normal(size=(30000, 3)) * 0.05,
                          np.repeat(r.normal(size=(3, 3)), 700, axis=0),  # coincident
                          r.normal(size=(300, 3)) * 200.0,                 # far outliers
                          r.random((5000, 3)) * [4, 0, 4]])                # flat class
    keys = np.concatenate([np.zeros(32400, np.int64), np.full(5000, (1 << 32) + 2)])
    perm = r.permutation(pts.shape[0])
    pts, keys = pts[perm], keys[perm]
    for K in (32, 7):
        ra = np.random.default_rng(seed)
        rb = np.random.default_rng(seed)
        cid, off, mem, cen, stats = G.cluster_points(pts, keys, K, ra)
        cid2, cl = O.cluster_points(pts, keys, K, rb)
        assert np.array_equal(cid, cid2)
        assert np.array_equal(cen, [c.center for c in cl])
        assert np.array_equal(mem, np.concatenate([c.members for c in cl]))
        assert ra.bit_generator.state == rb.bit_generator.state
        assert stats["fallback"] > 0 and stats["splits"] > 0
