"""TEST INFRASTRUCTURE ONLY — ctypes driver of oracle/graph_oracle.c, the C
restatement of the reference's path-graph build (clustering.py:28-148,
graph.py:56-168, operators.py:17-19) for record sets of millions of vertices.

`build_graph` returns an `oracle.pathgraph_oracle.Graph` whose `w` is a
block operator (`w @ v` = W v over the clusters' dense blocks), so the numpy
oracle's `solve` / `splat` (solve.py:41-132) run on it unchanged.  The RNG
is numpy's own Generator (graph.py:60): its PCG64 state goes in, the state
after the build comes back into the Generator.  Pinned by
tests/test_oracle_c.py against the numpy oracle and the reference goldens.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from oracle import pathgraph_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "build", "libgraph_oracle.so")
_lib = None


class Pcg(C.Structure):
    _fields_ = [("s_hi", C.c_uint64), ("s_lo", C.c_uint64), ("i_hi", C.c_uint64),
                ("i_lo", C.c_uint64), ("has_u32", C.c_int32), ("u32", C.c_uint32)]

    @classmethod
    def of(cls, rng: np.random.Generator) -> "Pcg":
        st = rng.bit_generator.state
        s, i = st["state"]["state"], st["state"]["inc"]
        m = (1 << 64) - 1
        return cls(s >> 64, s & m, i >> 64, i & m, st["has_uint32"], st["uinteger"])

    def store(self, rng: np.random.Generator) -> None:
        st = rng.bit_generator.state
        st["state"]["state"] = (self.s_hi << 64) | self.s_lo
        st["has_uint32"] = int(self.has_u32)
        st["uinteger"] = int(self.u32)
        rng.bit_generator.state = st


class Records(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in (
        "omega_out", "normal", "g", "phase_dir", "emit_dir", "pdf_emit_at_phase", "pdf_emit",
        "coeff", "d_emit", "d_phase", "emit_delta", "kind")]


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            import subprocess

            subprocess.run(["make", "-s", "-C", HERE], check=True)
        L = C.CDLL(LIB)
        p = C.c_void_p
        L.og_rng_choice.argtypes = [C.POINTER(Pcg), C.c_int64, C.c_int64, p]
        L.og_rng_integers.argtypes = [C.POINTER(Pcg), C.c_int64]
        L.og_rng_integers.restype = C.c_int64
        L.og_cluster.argtypes = [p, p, C.c_int64, C.c_int32, C.POINTER(Pcg), p, p, p, p, p]
        L.og_operators.argtypes = [C.POINTER(Records), C.c_int64, p, p, p, p, p, p, p, p, p, p]
        L.og_apply_w.argtypes = [p, C.c_int64, p, p, p, p, p, p]
        L.og_set_threads.argtypes = [C.c_int]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def set_threads(n: int) -> None:
    lib().og_set_threads(int(n))


def rng_choice(rng: np.random.Generator, n: int, m: int) -> np.ndarray:
    st = Pcg.of(rng)
    out = np.empty(m, np.int64)
    if lib().og_rng_choice(C.byref(st), n, m, _ptr(out)):
        raise ValueError("bad choice arguments")
    st.store(rng)
    return out


def rng_integers(rng: np.random.Generator, k: int) -> int:
    st = Pcg.of(rng)
    v = lib().og_rng_integers(C.byref(st), k)
    st.store(rng)
    return int(v)


def cluster_points(positions, keys, K: int, rng: np.random.Generator):
    """clustering.py:28-93 -> (cluster_id, member_off, members, centers, stats)."""
    if K < 1:
        raise ValueError("cluster size K must be >= 1")
    pos = np.ascontiguousarray(positions, dtype=np.float64)
    keys = np.ascontiguousarray(keys, dtype=np.int64)
    n = pos.shape[0]
    cid = np.full(n, -1, np.int64)
    center = np.empty(n + 1, np.int64)
    off = np.empty(n + 2, np.int64)
    members = np.empty(max(n, 1), np.int64)
    counts = np.zeros(3, np.int64)
    st = Pcg.of(rng)
    rc = lib().og_cluster(_ptr(pos), _ptr(keys), n, int(K), C.byref(st), _ptr(cid), _ptr(center),
                          _ptr(off), _ptr(members), _ptr(counts))
    if rc:
        raise RuntimeError(f"og_cluster failed ({rc})")
    st.store(rng)
    m = int(counts[0])
    return cid, off[:m + 1].copy(), members[:n].copy(), center[:m].copy(), \
        {"clusters": m, "splits": int(counts[1]), "fallback": int(counts[2])}


class BlockW:
    """W as dense per-cluster blocks; `w @ v` = W v (graph.py:167's CSR product)."""

    def __init__(self, off, members, w_off, blocks, n):
        self.off, self.members, self.w_off, self.blocks, self.n = off, members, w_off, blocks, n
        self.shape = (n, n)

    def __matmul__(self, v):
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.zeros((self.n, 3))
        ones = np.ones((self.n, 3))
        lib().og_apply_w(_ptr(ones), self.off.shape[0] - 1, _ptr(self.off), _ptr(self.members),
                         _ptr(self.w_off), _ptr(self.blocks), _ptr(v), _ptr(out))
        return out

    def row_block(self, c):
        s = int(self.off[c + 1] - self.off[c])
        return self.blocks[self.w_off[c]:self.w_off[c] + s * s].reshape(s, s)


def operators(rec: dict, off: np.ndarray, members: np.ndarray, with_w: bool = True):
    """graph.py:94-168 over the given clusters -> (phat (3,n), inc_phase, inc_emit,
    BlockW or None, d_bar)."""
    n = rec["pos"].shape[0]
    keep = {}

    def f(name, dt=np.float64):
        a = np.ascontiguousarray(rec[name], dtype=dt)
        keep[name] = a
        return _ptr(a)

    R = Records(f("omega_out"), f("normal"), f("g"), f("phase_dir"), f("emit_dir"),
                f("pdf_emit_at_phase"), f("pdf_emit"), f("coeff"), f("d_emit"), f("d_phase"),
                f("emit_delta", np.uint8), f("kind", np.uint8))
    off = np.ascontiguousarray(off, np.int64)
    members = np.ascontiguousarray(members, np.int64)
    m = off.shape[0] - 1
    sizes = np.diff(off)
    w_off = np.zeros(m + 1, np.int64)
    np.cumsum(sizes * sizes, out=w_off[1:])
    blocks = np.empty(int(w_off[-1]) if with_w else 0)
    phat = np.zeros((3, n))
    inc_p = np.zeros(n, np.uint8)
    inc_e = np.zeros(n, np.uint8)
    d_bar = np.zeros((n, 3))
    lib().og_operators(C.byref(R), m, _ptr(off), _ptr(members), _ptr(phat[0]), _ptr(phat[1]),
                       _ptr(phat[2]), _ptr(inc_p), _ptr(inc_e), _ptr(w_off),
                       _ptr(blocks) if with_w else None, _ptr(d_bar))
    w = BlockW(off, members, w_off, blocks, n) if with_w else None
    return phat, inc_p.astype(bool), inc_e.astype(bool), w, d_bar


def build_graph(rec: dict, paths: dict, width, height, spp, K: int, seed: int = 0,
                with_w: bool = True) -> O.Graph:
    """graph.py:56-69: clusters + marginals + operators, as an oracle Graph."""
    rng = np.random.default_rng(np.random.SeedSequence([seed & 0xFFFFFFFF, 0xC1A5]))
    cid, off, members, centers, stats = cluster_points(
        rec["pos"], O.class_keys(rec["kind"], rec["class_id"]), K, rng)
    g = O.Graph(rec, paths, width, height, spp, cid, None, O.next_index(rec["path_idx"]))
    g.member_off, g.members, g.centers, g.stats = off, members, centers, stats
    phat, g.included_phase, g.included_emit, g.w, g.d_bar = operators(rec, off, members, with_w)
    g.phat_ind, g.phat_dir_phase, g.phat_dir_emit = phat
    return g


def clusters_as_list(off, members, centers):
    """[Cluster(center, members)] like clustering.py:93."""
    return [O.Cluster(int(centers[c]), members[off[c]:off[c + 1]]) for c in range(centers.shape[0])]
