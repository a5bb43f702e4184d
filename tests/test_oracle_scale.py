"""The oracle pinned at the benchmarked scenes' scale: C1 at
full size (seeds 0/1/2) and the C2/C3/C4 slices (0.3-0.7 M vertices), against
the reference's own outputs (tests/golden/make_golden_scale.py).

The record sets are the reference's exactly (C tracer restatement + the
committed XOR patch, sha256-checked in conftest.scale_case).  On them the C
clustering + operators restatement (oracle/graph_oracle.c) and the numpy
solve / splat must reproduce the reference: cluster ids, centers, member
lists, next_idx, inclusion masks and CSR topology bit-exact (sha256), sampled
p-hat / D-bar / W rows, incoming and i_bar to 1e-11 relative, residuals and
the image."""

import numpy as np
import pytest

from conftest import SCALE_CASES, csr_topology_hashes, scale_case, sha64
from oracle import graph_oracle as G
from oracle import pathgraph_oracle as O


@pytest.mark.parametrize("name", SCALE_CASES)
def test_oracle_matches_reference_at_scale(name):
    z, rec, paths = scale_case(name)
    K, seed, iters = int(z["cluster_size"]), int(z["seed"]), int(z["iterations"])
    g = G.build_graph(rec, paths, int(z["width"]), int(z["height"]), int(z["spp"]), K, seed)
    assert g.centers.shape[0] == int(z["n_clusters"])
    assert sha64(g.cluster_id) == str(z["sha_cluster_id"])
    assert sha64(g.centers) == str(z["sha_centers"])
    assert sha64(g.member_off) == str(z["sha_cl_off"])
    assert sha64(g.members) == str(z["sha_members"])
    assert sha64(g.next_idx) == str(z["sha_next_idx"])
    ip, ix = csr_topology_hashes(g.cluster_id, g.member_off, g.members)
    assert ip == str(z["sha_w_indptr"]) and ix == str(z["sha_w_indices"])
    for a in ("included_phase", "included_emit"):
        assert sha64(getattr(g, a)) == str(z["sha_" + a]), a
    rows = z["sample_rows"]
    for a in ("phat_ind", "phat_dir_phase", "phat_dir_emit", "d_bar"):
        np.testing.assert_allclose(getattr(g, a)[rows], z["s_" + a], rtol=1e-12, atol=1e-300)
    # W rows of the sampled records: the row of the record's cluster block
    pos_in = np.empty_like(g.members)
    pos_in[g.members] = np.arange(g.members.shape[0]) - np.repeat(g.member_off[:-1],
                                                                  np.diff(g.member_off))
    wrows = [g.w.row_block(g.cluster_id[r])[pos_in[r]] for r in rows]
    np.testing.assert_allclose(np.concatenate(wrows), z["s_w_data"], rtol=1e-12, atol=0)
    inc, ib, res, _ = O.solve(g, iters, 0.0)
    np.testing.assert_allclose(inc[rows], z["s_incoming"], rtol=1e-11, atol=1e-300)
    np.testing.assert_allclose(ib[rows], z["s_i_bar"], rtol=1e-11, atol=1e-300)
    np.testing.assert_allclose(res, z["residuals"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(O.splat(g, ib), z["image"], rtol=1e-11, atol=1e-300)
    np.testing.assert_array_equal(O.splat_pt(paths, int(z["width"]), int(z["height"]),
                                             int(z["spp"])), z["pt_image"])
