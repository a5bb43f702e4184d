"""GPU parity at the benchmarked scale.

1. On the reference's own record sets at scale (C1 full for seeds 0/1/2 and
   the C2/C3/C4 slices, 0.05-0.7 M vertices; conftest.scale_case): cluster
   ids, centers, member lists, next_idx, inclusion masks and CSR topology
   bit-exact against the reference's sha256; sampled p-hat / D-bar / W rows
   within 1e-5; incoming / i_bar after K iterations and the image within the
   north-star 1e-4 relative (zeros exact); residuals within 1e-4.
2. End to end: device `render_pg` (pipeline.py:25-42) against the
   reference's own `render_pg` image over seeds 0/1/2 at C1 full size.
3. On the FULL benchmark record sets traced on the device (C2 8.3 M, C3 37 M,
   C4 75 M vertices) against the C restatement of the reference's build
   (oracle/graph_oracle.c, pinned to the reference by tests/test_oracle_c.py
   and tests/test_oracle_scale.py): cluster ids, centers and member lists
   bit-exact; at C2 also the CSR topology and the 10-iteration solve within
   1e-4; at C3/C4 the operators of 2048 sampled clusters (A+ v and D-bar
   within 1e-5).
"""

import numpy as np
import pytest

from conftest import SCALE_CASES, assert_rel, scale_case, sha64
from oracle import graph_oracle as G
from oracle import pathgraph_oracle as O

pytestmark = pytest.mark.gpu


def _trace(z, rec, paths):
    from paper_2404_11894_b200.transport.records import PathSoA, RecordSoA, TraceOutput

    return TraceOutput(None, RecordSoA(**rec), PathSoA(**paths), int(z["width"]),
                       int(z["height"]), int(z["spp"]))


@pytest.mark.parametrize("name", SCALE_CASES)
def test_device_graph_matches_reference_at_scale(cuda, name):
    from paper_2404_11894_b200.pathgraph import build_graph, solve, splat_output

    z, rec, paths = scale_case(name)
    K, seed, iters = int(z["cluster_size"]), int(z["seed"]), int(z["iterations"])
    trace = _trace(z, rec, paths)
    g = build_graph(trace, K, seed=seed)
    cid, off, mem, cen = g.native.export_clusters()
    assert cen.shape[0] == int(z["n_clusters"])
    assert sha64(cid) == str(z["sha_cluster_id"])
    assert sha64(cen) == str(z["sha_centers"])
    assert sha64(off) == str(z["sha_cl_off"])
    assert sha64(mem) == str(z["sha_members"])
    assert sha64(g.next_idx) == str(z["sha_next_idx"])
    W = g.w_indirect
    assert sha64(W.indptr) == str(z["sha_w_indptr"])
    assert sha64(W.indices) == str(z["sha_w_indices"])
    for a in ("included_phase", "included_emit"):
        assert sha64(getattr(g, a)) == str(z["sha_" + a]), a
    rows = z["sample_rows"]
    for a in ("phat_ind", "phat_dir_phase", "phat_dir_emit"):
        assert_rel(getattr(g, a)[rows], z["s_" + a], 1e-5, floor=1e-300, what=a)
    assert_rel(g.d_bar[rows], z["s_d_bar"], 1e-5, what="d_bar")
    wd = np.concatenate([W.data[W.indptr[q]:W.indptr[q + 1]] for q in rows])
    assert_rel(wd, z["s_w_data"], 1e-5, what="W rows")
    del W
    res = solve(g, iterations=iters, tol=0.0)
    assert res.iterations == iters
    assert_rel(np.asarray(res.incoming)[rows], z["s_incoming"], 1e-4, what="incoming")
    assert_rel(np.asarray(res.i_bar)[rows], z["s_i_bar"], 1e-4, what="i_bar")
    np.testing.assert_allclose(res.residuals, z["residuals"], rtol=1e-4, atol=1e-6)
    assert_rel(splat_output(g, res), z["image"], 1e-4, what="image")


def test_render_pg_matches_reference_render_pg(cuda):
    """pipeline.py:25-42 end to end at C1 full size (64x64, 4 spp), seeds
    0/1/2, the reference's default solve settings (10 iterations, tol 1e-3).

    Band: when the device tracer's record set equals the reference's in
    structure (every path the same length), the clusters are the same, so the
    image must match within the 1e-4 relative bar of the propagated radiance
    (relative to the image maximum, since pixels are means of many paths).
    Paths whose length differs (device libm ulps flipping a Russian-roulette
    or tracking decision, <= 0.5% of paths) shift later record indices and
    so the clustering: then the image may differ at the noise level, and the
    relative RMS difference must stay below a quarter of the seed-to-seed
    difference of the reference's own renders."""
    from paper_2404_11894_b200 import scenes as S
    from paper_2404_11894_b200.harness.config import RenderConfig
    from paper_2404_11894_b200.pathgraph import render_pg

    ref = {}
    for name in ("c1_s0", "c1_s1", "c1_s2"):
        z = np.load(f"tests/golden/scale_{name}.npz")
        ref[int(z["seed"])] = z
    seeds = sorted(ref)

    def rel_rms(a, b):
        return float(np.sqrt(np.mean((a - b) ** 2)) / np.sqrt(np.mean(b ** 2)))

    seed_spread = min(rel_rms(ref[a]["render_pg_image"], ref[b]["render_pg_image"])
                      for a in seeds for b in seeds if a < b)
    report = []
    for s in seeds:
        z = ref[s]
        cfg = RenderConfig(mode="pg", spp=int(z["spp"]), max_depth=int(z["max_depth"]), seed=s,
                           iterations=int(z["iterations"]))
        pg = render_pg(S.scene_c1((64, 64)), cfg)
        img, want = pg.image, z["render_pg_image"]
        n_ref = int(z["n"])
        counts_equal = pg.trace.records.n == n_ref and np.array_equal(
            np.asarray(pg.trace.paths.rec_count), scale_case(f"c1_s{s}")[2]["rec_count"])
        err = float(np.abs(img - want).max() / np.abs(want).max())
        rr = rel_rms(img, want)
        report.append((s, counts_equal, err, rr))
        if counts_equal:
            assert err <= 1e-4, (s, err)
            assert pg.result.iterations == int(z["render_pg_iterations"])
        else:
            assert rr <= 0.25 * seed_spread, (s, rr, seed_spread)
    print("render_pg vs reference (seed, same record structure, max rel, rel rms):", report,
          "seed spread", seed_spread)


# ------------------------------------------------------------ full size
K = 32
FIELDS = ("pos", "omega_out", "normal", "g", "phase_dir", "emit_dir", "pdf_emit_at_phase",
          "pdf_emit", "emit_delta", "kind", "coeff", "d_emit", "d_phase", "class_id",
          "path_idx", "w_cont", "i_pt")


@pytest.fixture(scope="module", params=["C2", "C3", "C4"])
def full(request, cuda):
    import torch

    from paper_2404_11894_b200.harness.config import RenderConfig
    from paper_2404_11894_b200.pathgraph import build_graph
    from paper_2404_11894_b200.scenes import WORKLOADS
    from paper_2404_11894_b200.transport import render_pt

    wl = WORKLOADS[request.param]
    out = render_pt(wl.scene(), RenderConfig(spp=wl.spp, max_depth=wl.max_depth, seed=0),
                    with_records=True)
    g = build_graph(out, K, seed=0)
    dev = out.records.device_tensors()
    pos = dev["pos"].cpu().numpy()
    keys = O.class_keys(dev["kind"].cpu().numpy(), dev["class_id"].cpu().numpy())
    rng = np.random.default_rng(np.random.SeedSequence([0, 0xC1A5]))
    ocid, ooff, omem, ocen, stats = G.cluster_points(pos, keys, K, rng)
    del pos, keys
    yield request.param, wl, out, g, (ocid, ooff, omem, ocen, stats)
    del g, out
    torch.cuda.empty_cache()


def test_full_size_clusters_equal_oracle(full):
    name, wl, out, g, (ocid, ooff, omem, ocen, stats) = full
    cid, off, mem, cen = g.native.export_clusters()
    n = out.records.n
    assert n > {"C2": 8_000_000, "C3": 30_000_000, "C4": 70_000_000}[name]
    assert cen.shape[0] == ocen.shape[0]
    assert np.array_equal(cid, ocid)
    assert np.array_equal(cen, ocen)
    assert np.array_equal(off, ooff)
    assert np.array_equal(mem, omem)
    gi = g.info()
    assert gi["n_splits"] == stats["splits"] and gi["n_clusters"] == stats["clusters"]


def _sampled_subgraph(out, off, mem, cen, pick):
    import torch

    sizes = np.diff(off)
    rows = np.concatenate([mem[off[c]:off[c + 1]] for c in pick])
    dev = out.records.device_tensors()
    idx = torch.as_tensor(rows, device=dev["pos"].device)
    sub = {f: dev[f][idx].cpu().numpy() for f in FIELDS}
    soff = np.zeros(len(pick) + 1, np.int64)
    np.cumsum(sizes[pick], out=soff[1:])
    return rows, sub, soff


def test_full_size_sampled_operators_match_oracle(full):
    """graph.py:94-168 restated (C) on 2048 sampled clusters (plus the 8
    largest) of the device's own clustering (equal to the oracle's, above):
    A+ v (operators.py:17-19) and D-bar within 1e-5 relative."""
    from paper_2404_11894_b200.pathgraph import aggregate_direct, aggregate_indirect

    name, wl, out, g, _ = full
    _, off, mem, cen = g.native.export_clusters()
    m = cen.shape[0]
    sizes = np.diff(off)
    rng = np.random.default_rng(11)
    pick = np.unique(np.concatenate([rng.choice(m, 2048, replace=False), np.argsort(sizes)[-8:]]))
    rows, sub, soff = _sampled_subgraph(out, off, mem, cen, pick)
    phat, inc_p, inc_e, w, d_bar = G.operators(sub, soff, np.arange(rows.shape[0]))
    n = out.records.n
    v = rng.random((n, 3))
    want = sub["coeff"] * (w @ v[rows])
    assert_rel(aggregate_indirect(g, v)[rows], want, 1e-5, what=f"{name} A+ v")
    assert_rel(aggregate_direct(g)[rows], d_bar, 1e-5, what=f"{name} d_bar")
    assert np.array_equal(g.included_phase[rows], inc_p)
    assert np.array_equal(g.included_emit[rows], inc_e)


def test_full_size_c2_topology_and_solve_match_oracle(full):
    """C2 in full: CSR topology (graph.py:167) bit-exact and the 10-iteration
    solve (solve.py:64-98) + splat within 1e-4 of the oracle's fp64 run over
    the whole 8.3 M-vertex graph."""
    from conftest import csr_topology_hashes

    from paper_2404_11894_b200.pathgraph import solve, splat_output

    name, wl, out, g, (ocid, ooff, omem, ocen, _) = full
    if name != "C2":
        pytest.skip("full solve parity at C2 (the C3/C4 graphs are checked by sampled clusters)")
    W = g.w_indirect
    ip, ix = csr_topology_hashes(ocid, ooff, omem)
    assert sha64(W.indptr) == ip and sha64(W.indices) == ix
    del W
    rec = {f: v for f, v in out.records.host_arrays().items()}
    paths = out.paths.host_arrays()
    og = O.Graph(rec, paths, out.width, out.height, out.spp, ocid, None,
                 O.next_index(rec["path_idx"]))
    phat, og.included_phase, og.included_emit, og.w, og.d_bar = G.operators(rec, ooff, omem)
    og.phat_ind, og.phat_dir_phase, og.phat_dir_emit = phat
    assert np.array_equal(g.included_phase, og.included_phase)
    assert_rel(g.phat_ind, og.phat_ind, 1e-5, floor=1e-300, what="phat_ind")
    assert_rel(g.d_bar, og.d_bar, 1e-5, what="d_bar")
    inc, ib, res_ref, _ = O.solve(og, wl.iterations, 0.0)
    res = solve(g, iterations=wl.iterations, tol=0.0)
    assert_rel(res.incoming, inc, 1e-4, what="incoming")
    assert_rel(res.i_bar, ib, 1e-4, what="i_bar")
    np.testing.assert_allclose(res.residuals, res_ref, rtol=1e-4, atol=1e-6)
    assert_rel(splat_output(g, res), O.splat(og, ib), 1e-4, what="image")
