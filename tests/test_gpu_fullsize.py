"""Full-size (BASELINE C2: 512x512, 8 spp, 8.3 M vertices) properties of the
device build and operators, where the oracle cannot cluster the whole set in
seconds:

- the clusters partition the records (graph.py:56-69, clustering.py:87-93):
  every record in exactly one cluster, sizes 1..2K, members ascending, one
  class key per cluster, the center among its members;
- the build and the solve are deterministic (same seed -> same clusters,
  bit-identical images);
- the operators of a sample of the device's own clusters match the oracle's
  graph.py:94-168 restated on just those clusters' records: A+ v
  (operators.py:17-19) and D-bar (operators.py:22-24) within the 1e-5
  relative bar of the golden tests.
"""

import numpy as np
import pytest

from conftest import assert_rel
from oracle import pathgraph_oracle as O

pytestmark = pytest.mark.gpu

K = 32
FIELDS = ("pos", "omega_out", "normal", "g", "phase_dir", "emit_dir", "pdf_emit_at_phase",
          "pdf_emit", "emit_delta", "kind", "coeff", "d_emit", "d_phase", "class_id",
          "path_idx")


@pytest.fixture(scope="module")
def c2(cuda):
    from paper_2404_11894_b200.harness.config import RenderConfig
    from paper_2404_11894_b200.pathgraph import build_graph
    from paper_2404_11894_b200.scenes import WORKLOADS
    from paper_2404_11894_b200.transport import render_pt

    wl = WORKLOADS["C2"]
    out = render_pt(wl.scene(), RenderConfig(spp=wl.spp, max_depth=wl.max_depth, seed=0),
                    with_records=True)
    g = build_graph(out, K, seed=0)
    return out, g


def test_c2_clusters_partition_the_records(c2):
    out, g = c2
    cid, off, mem, cen = g.native.export_clusters()
    n, m = out.records.n, cen.shape[0]
    assert n > 8_000_000
    sizes = np.diff(off)
    assert sizes.min() >= 1 and sizes.max() <= 2 * K
    assert np.array_equal(np.sort(mem), np.arange(n))
    assert np.array_equal(cid[mem], np.repeat(np.arange(m), sizes))
    inner = np.ones(n - 1, dtype=bool)
    inner[off[1:-1] - 1] = False  # pairs that straddle two clusters
    assert np.all(mem[1:][inner] > mem[:-1][inner])
    key = O.class_keys(out.records.kind, out.records.class_id)
    assert np.array_equal(key[mem], np.repeat(key[mem[off[:-1]]], sizes))
    assert np.array_equal(cid[cen], np.arange(m))
    assert 0.8 * n / 31.0 < m < 1.2 * n / 31.0  # mean size 31.0-31.1
    assert np.array_equal(g.next_idx, O.next_index(out.records.path_idx))


def test_c2_build_and_solve_are_deterministic(c2):
    from paper_2404_11894_b200.pathgraph import build_graph, solve, splat_output

    out, g = c2
    cid = g.native.export_clusters()[0]
    img = splat_output(g, solve(g, iterations=3, tol=0.0))
    g2 = build_graph(out, K, seed=0)
    assert np.array_equal(g2.native.export_clusters()[0], cid)
    img2 = splat_output(g2, solve(g2, iterations=3, tol=0.0))
    assert np.array_equal(img, img2)
    del g2
    g3 = build_graph(out, K, seed=1)
    assert not np.array_equal(g3.native.export_clusters()[0], cid)


def test_c2_sampled_cluster_operators_match_oracle(c2):
    from paper_2404_11894_b200.pathgraph import aggregate_direct, aggregate_indirect

    out, g = c2
    _, off, mem, cen = g.native.export_clusters()
    n, m = out.records.n, cen.shape[0]
    rng = np.random.default_rng(7)
    sizes = np.diff(off)
    pick = np.unique(np.concatenate([rng.choice(m, 400, replace=False),
                                     np.argsort(sizes)[-8:]]))
    rows = np.concatenate([mem[off[c]:off[c + 1]] for c in pick])
    sub = {f: getattr(out.records, f)[rows] for f in FIELDS}
    at = 0
    clusters = []
    for c in pick:
        s = int(sizes[c])
        members = np.arange(at, at + s)
        clusters.append(O.Cluster(int(at + np.searchsorted(mem[off[c]:off[c + 1]], cen[c])),
                                  members))
        at += s
    og = O.Graph(sub, None, 0, 0, 0, None, clusters, None)
    O.build_operators(og)

    v = rng.random((n, 3))
    assert_rel(aggregate_indirect(g, v)[rows], O.aggregate_indirect(og, v[rows]), 1e-5,
               what="A+ v")
    assert_rel(aggregate_direct(g)[rows], og.d_bar, 1e-5, what="d_bar")


def test_c2_one_more_iteration_is_one_operator_application(c2):
    """solve.py:64-98 at full size: incoming after k+1 iterations equals
    P (A+ I_k + D-bar) with terminal rows keeping i_pt (operators.py:27-38),
    evaluated through the operator API on the solve's own I_k; the last
    iteration's i_bar is A+ I_k (solve.py:78)."""
    from paper_2404_11894_b200.pathgraph import (aggregate_direct, aggregate_indirect, propagate,
                                                 solve)

    _, g = c2
    inc_k = np.array(solve(g, iterations=4, tol=0.0).incoming)
    r = solve(g, iterations=5, tol=0.0)
    inc, ibar = np.array(r.incoming), np.array(r.i_bar)
    a = aggregate_indirect(g, inc_k)
    floor = 1e-7 * float(np.abs(inc).max())
    assert_rel(ibar, a, 1e-4, floor=floor, what="i_bar")
    assert_rel(inc, propagate(g, a + aggregate_direct(g)), 1e-4, floor=floor, what="incoming")
