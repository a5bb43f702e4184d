"""Host-side checks of libvolpg_b200.so that need no GPU: it loads, exports
every symbol include/volpg_b200.h declares, its ABI structs match the ctypes
mirrors, and its host logic (numpy RNG replica, split loop) is exact."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from oracle import pathgraph_oracle as O
from paper_2404_11894_b200 import _native as N


def _declared_symbols():
    text = open(os.path.join(ROOT, "include", "volpg_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*|uint64_t|size_t)\s+(vpg_\w+)\(",
                                 text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    syms = _declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert lib.vpg_abi_version() == 1


def test_struct_sizes_match_bindings():
    lib = N.lib()
    for which, st in enumerate((N.Pcg64State, N.Records, N.Paths, N.GraphInfo, N.SceneStruct,
                                N.TraceCfg)):
        assert lib.vpg_struct_size(which) == ctypes.sizeof(st), st.__name__


@pytest.mark.parametrize("n,m,seed", [(20000, 625, 0), (45718, 1429, 4), (500, 16, 1),
                                      (10001, 300, 2), (10001, 200, 2), (100, 100, 7), (1, 1, 3),
                                      (7, 0, 1), (3_000_000, 93_750, 9)])
def test_rng_choice_matches_numpy(n, m, seed):
    g = np.random.default_rng(np.random.SeedSequence([seed, 0xC1A5]))
    g.integers(5)  # leave a buffered 32-bit half behind
    st = N.Pcg64State.from_generator(g)
    out = np.empty(max(m, 1), dtype=np.int64)
    N.check(N.lib().vpg_rng_choice(ctypes.byref(st), n, m, out.ctypes.data))
    assert np.array_equal(out[:m], g.choice(n, m, replace=False))
    # the states continue identically
    probe = np.empty(8, dtype=np.int64)
    N.check(N.lib().vpg_rng_integers(ctypes.byref(st), 1000003, 8, probe.ctypes.data))
    assert np.array_equal(probe, g.integers(1000003, size=8))


def test_rng_integers_and_state_roundtrip():
    g = np.random.default_rng(12345)
    st = N.Pcg64State.from_generator(g)
    ks = [1, 2, 3, 64, 65, 1 << 31, (1 << 32) - 1, 1 << 32, (1 << 32) + 1, 1 << 40]
    for k in ks:
        o = np.empty(3, dtype=np.int64)
        N.check(N.lib().vpg_rng_integers(ctypes.byref(st), k, 3, o.ctypes.data))
        assert [int(g.integers(k)) for _ in range(3)] == list(o)
    h = np.random.default_rng(0)
    st.store_into(h)
    assert h.bit_generator.state == g.bit_generator.state


def test_rng_errors_map_to_valueerror():
    st = N.Pcg64State.from_generator(np.random.default_rng(0))
    out = np.empty(4, dtype=np.int64)
    with pytest.raises(ValueError):
        N.check(N.lib().vpg_rng_choice(ctypes.byref(st), 3, 4, out.ctypes.data))


def _groups_from_assign(assign, m):
    order = np.argsort(assign, kind="stable")
    bounds = np.searchsorted(assign[order], np.arange(m + 1))
    return [order[bounds[c]:bounds[c + 1]] for c in range(m)]


@pytest.mark.parametrize("seed,K", [(0, 4), (1, 8), (2, 2)])
def test_split_loop_matches_oracle(seed, K):
    rs = np.random.default_rng(seed)
    pts = np.concatenate([rs.normal(size=(600, 3)), rs.normal(size=(300, 3)) * 0.05 + 2,
                          np.repeat(rs.normal(size=(1, 3)), 40, axis=0)])  # coincident block
    m = 9  # few centers -> many oversize groups and deep splits
    centers = list(range(0, 9 * 97, 97))[:m]
    assign = O.nearest_center(pts, pts[centers])
    groups = _groups_from_assign(assign, m)
    g_ref = np.random.default_rng(100 + seed)
    g_nat = np.random.default_rng(100 + seed)
    ref_groups = [x.copy() for x in groups]
    ref_centers = list(centers)
    O._split_loop(pts, ref_groups, ref_centers, K, g_ref)

    off = np.concatenate([[0], np.cumsum([len(x) for x in groups])]).astype(np.int64)
    mem = np.concatenate(groups).astype(np.int64)
    cap = 4 * len(pts)
    st = N.Pcg64State.from_generator(g_nat)
    n_out = ctypes.c_int64()
    o_off = np.zeros(cap + 1, np.int64)
    o_mem = np.zeros(len(pts), np.int64)
    o_cen = np.zeros(cap, np.int64)
    N.check(N.lib().vpg_split_groups(ctypes.byref(st), np.ascontiguousarray(pts).ctypes.data,
                                     m, off.ctypes.data, mem.ctypes.data,
                                     np.array(centers, np.int64).ctypes.data, 2 * K, cap,
                                     ctypes.byref(n_out), o_off.ctypes.data, o_mem.ctypes.data,
                                     o_cen.ctypes.data))
    st.store_into(g_nat)
    got = [o_mem[o_off[k]:o_off[k + 1]] for k in range(n_out.value)]
    assert len(got) == len(ref_groups)
    for a, b in zip(got, ref_groups):
        assert np.array_equal(a, b)
    assert list(o_cen[:n_out.value]) == ref_centers
    assert g_nat.bit_generator.state == g_ref.bit_generator.state
    assert max(len(x) for x in got) <= 2 * K


@pytest.mark.gpu
@pytest.mark.parametrize("n,m,seed", [(20000, 625, 0), (500, 16, 1), (3_000_000, 93_750, 9)])
def test_rng_choice_device_matches_numpy(cuda, n, m, seed):
    g = np.random.default_rng(np.random.SeedSequence([seed, 0xC1A5]))
    g.integers(5)
    st = N.Pcg64State.from_generator(g)
    out = cuda.empty(m, dtype=cuda.int32, device="cuda")
    N.check(N.lib().vpg_rng_choice_device(ctypes.byref(st), n, m, out.data_ptr(),
                                          N.stream_handle()))
    assert np.array_equal(out.cpu().numpy(), g.choice(n, m, replace=False))
    h = np.random.default_rng(0)
    st.store_into(h)
    assert h.bit_generator.state == g.bit_generator.state
