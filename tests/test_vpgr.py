"""VPGR record dumps (reference: transport/records.py:191-256) against a dump
written by the reference itself (tests/golden/make_vpgr.py): byte-exact
round trip, the error cases, and the graph solve on the loaded dump."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, assert_rel
from oracle import pathgraph_oracle as O
from paper_2404_11894_b200.transport import load_records, save_records

DUMP = os.path.join(GOLDEN, "c1_8.vpgr")


def _ref():
    return np.load(os.path.join(GOLDEN, "c1_8_vpgr.npz"))


def test_load_then_save_is_byte_identical(tmp_path):
    t = load_records(DUMP)
    assert t.records.n == 491 and t.paths.n == 8 * 8 * 2
    assert (t.width, t.height, t.spp) == (8, 8, 2)
    out = tmp_path / "again.vpgr"
    save_records(str(out), t)
    assert out.read_bytes() == open(DUMP, "rb").read()


def test_bad_dumps_raise_ioerror(tmp_path):
    raw = open(DUMP, "rb").read()
    cases = {"magic": b"XXXX" + raw[4:], "version": raw[:4] + b"\x63\x00\x00\x00" + raw[8:],
             "truncated": raw[:-100]}
    for name, data in cases.items():
        p = tmp_path / f"{name}.vpgr"
        p.write_bytes(data)
        with pytest.raises(IOError):
            load_records(str(p))


def test_oracle_solve_on_loaded_dump_matches_reference():
    z = _ref()
    t = load_records(DUMP)
    rec, paths = t.records.host_arrays(), t.paths.host_arrays()
    g = O.build_graph(rec, paths, t.width, t.height, t.spp, int(z["K"]), int(z["seed"]))
    assert np.array_equal(g.cluster_id, z["cluster_id"])
    inc, ib, res, _ = O.solve(g, int(z["iterations"]), 0.0)
    np.testing.assert_allclose(O.splat(g, ib), z["image"], rtol=1e-12, atol=1e-300)
    np.testing.assert_allclose(inc, z["incoming"], rtol=1e-12, atol=1e-300)


@pytest.mark.gpu
def test_solve_from_records_on_reference_dump(cuda):
    from paper_2404_11894_b200.pathgraph import solve_from_records

    z = _ref()
    t = load_records(DUMP, pin=True)
    image, graph, result = solve_from_records(t, int(z["K"]), iterations=int(z["iterations"]),
                                              tol=0.0, seed=int(z["seed"]))
    assert np.array_equal(t.records.cluster_id, z["cluster_id"])
    assert_rel(image, z["image"], 1e-4, what="image")
    assert_rel(result.incoming, z["incoming"], 1e-4, what="incoming")
    assert_rel(result.i_bar, z["i_bar"], 1e-4, what="i_bar")
