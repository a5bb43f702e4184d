"""Path graph built on the device (reference: pathgraph/graph.py:29-168).

`build_graph` clusters the records and builds the aggregation operators in
one native call (vpg_graph_build): exact-RNG center draw, hash-grid nearest
center, split loop, marginals, the dense per-cluster kernel blocks of A+ and
D-bar.  The resulting `PathGraph` keeps everything in HBM; the attributes the
reference exposes as numpy/scipy objects (`clusters`, `phat_*`,
`included_*`, `w_indirect`, `d_bar`, `next_idx`, `records.cluster_id`) are
copied to the host on first access.
"""

from __future__ import annotations

import ctypes

import numpy as np

from paper_2404_11894_b200 import _native as N
from paper_2404_11894_b200.pathgraph.clustering import Cluster
from paper_2404_11894_b200.transport.records import PathSoA, RecordSoA, TraceOutput, as_trace


# the record fields the build and the solve read on the device: never depth;
# pdf_phase only in a 0-iteration solve (uploaded then, see solve()); normal
# only for surface records (solve_from_records keeps it on the host when
# there are none)
BUILD_FIELDS = tuple(f[0] for f in N.RECORD_FIELDS
                     if f[0] not in ("depth", "pdf_phase", "normal"))


class NativeGraph:
    """Owns a vpg_graph handle and keeps the device records it borrows alive."""

    def __init__(self, handle: int, rec_tensors: dict, rec_struct, n: int):
        self.handle = handle
        self.rec_tensors = rec_tensors
        self.rec_struct = rec_struct
        self.n = n
        self.solve_generation = 0
        self.performed = -1

    @classmethod
    def build(cls, records: RecordSoA, cluster_size: int, rng: np.random.Generator,
              flags: int = 0) -> "NativeGraph":
        # the clustering needs only pos/kind/class_id: with an upload in flight
        # the native build waits for the other fields itself, just before it
        # first reads them
        need = BUILD_FIELDS if "normal" in (records.__dict__.get("_missing") or ()) \
            else BUILD_FIELDS + ("normal",)
        st = records.device(wait="early", need=need)
        fields = records.ready_event("all")
        if flags & N.VPG_BUILD_CLUSTERS_ONLY:
            fields = None  # never read; later device() calls wait for them
        state = N.Pcg64State.from_generator(rng)
        out = ctypes.c_void_p()
        N.check(N.lib().vpg_graph_build_wait(
            ctypes.byref(st), int(cluster_size), ctypes.byref(state), int(flags), N.stream_handle(),
            fields.cuda_event if fields is not None else None, ctypes.byref(out)))
        state.store_into(rng)
        return cls(out.value, dict(records._dev), st, records.n)

    def info(self) -> N.GraphInfo:
        gi = N.GraphInfo()
        N.check(N.lib().vpg_graph_info_get(self.handle, ctypes.byref(gi)))
        return gi

    def export_clusters(self):
        info = self.info()
        n, m = self.n, int(info.n_clusters)
        cid = np.empty(n, dtype=np.int64)
        off = np.empty(m + 1, dtype=np.int64)
        mem = np.empty(n, dtype=np.int64)
        cen = np.empty(m, dtype=np.int64)
        N.check(N.lib().vpg_graph_export_clusters(self.handle, cid.ctypes.data, off.ctypes.data,
                                                  mem.ctypes.data, cen.ctypes.data,
                                                  N.stream_handle()))
        return cid, off, mem, cen

    def __del__(self):
        if getattr(self, "handle", None):
            try:
                N.lib().vpg_graph_free(self.handle)
            except Exception:
                pass
            self.handle = None


def clusters_from_csr(off: np.ndarray, members: np.ndarray, centers: np.ndarray) -> list:
    return [Cluster(center=int(centers[k]), members=members[off[k]:off[k + 1]])
            for k in range(len(centers))]


_LAZY = ("clusters", "phat_ind", "phat_dir_phase", "phat_dir_emit", "included_phase",
         "included_emit", "w_indirect", "d_bar", "next_idx")


class PathGraph:
    """Records, paths, clusters, cached marginals and operators (graph.py:29-53)."""

    def __init__(self, records: RecordSoA, paths: PathSoA, width: int, height: int, spp: int,
                 next_idx=None, clusters=None, native: NativeGraph | None = None):
        self.records = records
        self.paths = paths
        self.width = int(width)
        self.height = int(height)
        self.spp = int(spp)
        self._native = native
        self._cache = {}
        if next_idx is not None:
            self._cache["next_idx"] = np.asarray(next_idx, dtype=np.int64)
        if clusters is not None:
            self._cache["clusters"] = list(clusters)

    # -- lazily materialised reference attributes ---------------------------
    def __getattr__(self, name):
        if name in _LAZY:
            cache = self.__dict__["_cache"]
            if name not in cache:
                self._materialise(name)
            return cache[name]
        raise AttributeError(name)

    def __setattr__(self, name, value):
        if name in _LAZY:
            self._cache[name] = value
        else:
            object.__setattr__(self, name, value)

    def _materialise(self, name):
        cache = self._cache
        g = self._native
        if name == "next_idx":
            cache[name] = self.records.next_index()
            return
        if g is None:
            raise AttributeError(f"{name} is not available on this graph")
        stream = N.stream_handle()
        n = self.records.n
        if name == "clusters":
            _, off, mem, cen = g.export_clusters()
            cache[name] = clusters_from_csr(off, mem, cen)
        elif name in ("phat_ind", "phat_dir_phase", "phat_dir_emit", "included_phase",
                      "included_emit"):
            p = [np.empty(n) for _ in range(3)]
            N.check(N.lib().vpg_graph_export_marginals(g.handle, p[0].ctypes.data,
                                                       p[1].ctypes.data, p[2].ctypes.data, stream))
            cache["phat_ind"], cache["phat_dir_phase"], cache["phat_dir_emit"] = p
            cache["included_phase"] = np.isfinite(p[0]) & (p[0] > 0.0)
            cache["included_emit"] = np.isfinite(p[2]) & (p[2] > 0.0)
        elif name == "w_indirect":
            import scipy.sparse as sp

            nnz = int(g.info().nnz)
            indptr = np.empty(n + 1, dtype=np.int64)
            indices = np.empty(nnz, dtype=np.int64)
            data = np.empty(nnz)
            N.check(N.lib().vpg_graph_export_operators(g.handle, indptr.ctypes.data,
                                                       indices.ctypes.data, data.ctypes.data,
                                                       None, stream))
            cache[name] = sp.csr_matrix((data, indices, indptr), shape=(n, n))
        elif name == "d_bar":
            d = np.empty((n, 3))
            N.check(N.lib().vpg_graph_export_operators(g.handle, None, None, None, d.ctypes.data,
                                                       stream))
            cache[name] = d

    # -------------------------------------------------------------------------
    @property
    def n_records(self) -> int:
        return self.records.n

    @property
    def native(self) -> NativeGraph:
        if self._native is None:
            raise RuntimeError("graph has no device representation")
        return self._native

    def cluster_of(self, record_index: int) -> Cluster:
        return self.clusters[int(self.records.cluster_id[record_index])]

    def info(self) -> dict:
        gi = self.native.info()
        return {"n_records": gi.n_records, "n_clusters": gi.n_clusters, "nnz": gi.nnz,
                "n_classes": gi.n_classes, "n_splits": gi.n_splits,
                "n_fallback": gi.n_fallback, "build_ms": list(gi.build_ms),
                "n_staged": gi.n_staged, "split_visits": gi.split_visits}


def build_graph(out: TraceOutput, cluster_size: int, seed: int = 0, timings: bool = False) -> PathGraph:
    """Cluster the records and cache marginals and aggregation operators.

    Same RNG as the reference (graph.py:59-60); sets out.records.cluster_id
    (materialised on first access).
    """
    if cluster_size < 1:
        raise ValueError("cluster size K must be >= 1")
    foreign = not isinstance(out, TraceOutput)  # e.g. the reference's own TraceOutput
    trace = as_trace(out)
    rng = np.random.default_rng(np.random.SeedSequence([seed & 0xFFFFFFFF, 0xC1A5]))
    flags = N.VPG_BUILD_TIMINGS if timings else 0
    native = NativeGraph.build(trace.records, cluster_size, rng, flags)
    graph = PathGraph(trace.records, trace.paths, trace.width, trace.height, trace.spp,
                      native=native)
    trace.records._set_cluster_provider(lambda: native.export_clusters()[0])
    if foreign:
        out.records.cluster_id = trace.records.cluster_id  # graph.py:62 mutates the input
    return graph


def compute_marginals(graph: PathGraph) -> None:
    """Fill graph.phat_* / included_* (graph.py:94-120); the device computed
    them during build_graph, this copies them to the host."""
    graph._materialise("phat_ind")
