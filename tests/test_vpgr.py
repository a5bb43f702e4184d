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


@pytest.mark.gpu
def test_device_load_matches_host_load(cuda, monkeypatch):
    import paper_2404_11894_b200.transport.records as R

    host = load_records(DUMP)
    # small staging chunks so the double-buffered path runs several chunks
    monkeypatch.setattr(R, "_CODEC_CHUNK", 290 * 37)
    monkeypatch.setattr(R, "_STAGING", {})
    dev = load_records(DUMP, device=True)
    assert dev.records.on_device() and dev.paths.on_device()
    assert (dev.width, dev.height, dev.spp) == (host.width, host.height, host.spp)
    for soa_h, soa_d in ((host.records, dev.records), (host.paths, dev.paths)):
        th = soa_h.host_arrays()
        td = {k: v.cpu().numpy() for k, v in soa_d.device_tensors().items()}
        for name in th:
            assert td[name].dtype == th[name].dtype, name
            np.testing.assert_array_equal(td[name], th[name], err_msg=name)


@pytest.mark.gpu
@pytest.mark.parametrize("chunk", [290 * 5, 32 << 20])
def test_device_save_is_byte_identical(cuda, monkeypatch, tmp_path, chunk):
    import paper_2404_11894_b200.transport.records as R

    monkeypatch.setattr(R, "_CODEC_CHUNK", chunk)
    monkeypatch.setattr(R, "_STAGING", {})
    dev = load_records(DUMP, device=True)
    dev.records.drop_host()
    out = tmp_path / "dev.vpgr"
    save_records(str(out), dev)
    assert out.read_bytes() == open(DUMP, "rb").read()


@pytest.mark.gpu
def test_device_trace_dump_round_trip(cuda, tmp_path):
    """A device trace saved from HBM and loaded back into HBM is bit-identical
    field by field, and the host save of the same trace is the same file."""
    from paper_2404_11894_b200 import scenes as S
    from paper_2404_11894_b200.harness.config import RenderConfig
    from paper_2404_11894_b200.transport import render_pt

    t = render_pt(S.scene_mixed((12, 12)), RenderConfig(spp=2, max_depth=24, seed=3),
                  with_records=True)
    assert t.records.on_device()
    a, b = tmp_path / "dev.vpgr", tmp_path / "host.vpgr"
    save_records(str(a), t)
    back = load_records(str(a), device=True)
    for soa, soa2 in ((t.records, back.records), (t.paths, back.paths)):
        d1, d2 = soa.device_tensors(), soa2.device_tensors()
        for name in d1:
            assert cuda.equal(d1[name], d2[name]), name
    host = load_records(str(a))
    save_records(str(b), host)
    assert a.read_bytes() == b.read_bytes()


@pytest.mark.gpu
def test_device_load_truncated_raises(cuda, tmp_path):
    raw = open(DUMP, "rb").read()
    for cut in (100, 290 * 491 // 2):
        p = tmp_path / f"cut{cut}.vpgr"
        p.write_bytes(raw[:-cut])
        with pytest.raises(IOError):
            load_records(str(p), device=True)


@pytest.mark.gpu
def test_pinned_solve_uploads_only_what_it_reads(cuda):
    """solve_from_records on pinned records copies only the fields the build,
    solve and splat read; the others stay readable on the host and reach the
    device on first device use (PT image, device save)."""
    from paper_2404_11894_b200.pathgraph import solve_from_records
    from paper_2404_11894_b200.transport import records as R

    z = _ref()
    host = load_records(DUMP)
    t = load_records(DUMP, pin=True)
    before = R.h2d_bytes()
    image, graph, result = solve_from_records(t, int(z["K"]), iterations=int(z["iterations"]),
                                              tol=0.0, seed=int(z["seed"]))
    moved = R.h2d_bytes() - before
    full = sum(a.nbytes for a in host.records.host_arrays().values()) + \
        sum(a.nbytes for a in host.paths.host_arrays().values())
    skipped = host.records.depth.nbytes + host.records.pdf_phase.nbytes + sum(
        getattr(host.paths, f).nbytes for f in ("pixel_idx", "direct0_nee", "direct0_phase",
                                                "pt_estimate", "extra_direct"))
    if not np.any(host.records.kind):  # no surface records: normals stay on the host
        skipped += host.records.normal.nbytes
    assert moved == full - skipped
    assert_rel(image, z["image"], 1e-4, what="image")
    np.testing.assert_array_equal(t.records.depth, host.records.depth)
    # first device use of a skipped field uploads it
    np.testing.assert_array_equal(t.image, host.image)
    assert not (t.paths.__dict__.get("_missing") or set()) & {"pt_estimate"}
    # a 0-iteration solve on the same graph brings pdf_phase over and agrees
    # with a graph built from fully uploaded records
    from paper_2404_11894_b200.pathgraph import build_graph, solve

    r0 = solve(graph, iterations=0)
    full = load_records(DUMP)
    g2 = build_graph(full, int(z["K"]), seed=int(z["seed"]))
    np.testing.assert_array_equal(r0.i_bar, solve(g2, iterations=0).i_bar)
