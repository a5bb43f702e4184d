"""Spatial clustering of shading points (reference: pathgraph/clustering.py).

Per compatibility class, ceil(n/K) centers are drawn with the caller's numpy
Generator, every point joins its exact nearest center (hash grid + exact
fallback), and clusters above 2K members are split with the same RNG, in the
reference's order, so the clusters are identical to the reference's.  The
work runs in libvolpg_b200 (cluster.cu); only the RNG draws and the split
loop's bookkeeping are host code (C++).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from paper_2404_11894_b200 import _native as N


@dataclass
class Cluster:
    center: int           # record index of the cluster center
    members: np.ndarray   # record indices, ascending


def cluster_points(positions, class_keys, K: int, rng: np.random.Generator):
    """Cluster points within compatibility classes (clustering.py:28-44).

    Returns (cluster_id per point, list of Cluster); advances `rng` exactly as
    the reference does.
    """
    if K < 1:
        raise ValueError("cluster size K must be >= 1")
    torch = N.require_cuda()
    pos = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 3)
    keys = np.asarray(class_keys)
    n = pos.shape[0]
    _, cls = np.unique(keys, return_inverse=True)  # ascending key order
    if n and cls.max() >= 65536:
        raise ValueError("more than 65536 compatibility classes")
    dev = {
        "pos": torch.from_numpy(pos).to("cuda"),
        "kind": torch.zeros(n, dtype=torch.uint8, device="cuda"),
        "class_id": torch.from_numpy(cls.astype(np.int32).reshape(-1)).to("cuda"),
    }
    st = N.Records()
    st.n = n
    for name, t in dev.items():
        setattr(st, name, t.data_ptr() if n else None)
    state = N.Pcg64State.from_generator(rng)
    handle = ctypes.c_void_p()
    N.check(N.lib().vpg_graph_build(ctypes.byref(st), int(K), ctypes.byref(state),
                                    N.VPG_BUILD_CLUSTERS_ONLY, N.stream_handle(),
                                    ctypes.byref(handle)))
    state.store_into(rng)
    from paper_2404_11894_b200.pathgraph.graph import NativeGraph, clusters_from_csr

    g = NativeGraph(handle.value, dev, st, n)
    cid, off, mem, cen = g.export_clusters()
    return cid, clusters_from_csr(off, mem, cen)
