"""Aggregation and propagation operators on arbitrary vectors
(reference: pathgraph/operators.py:17-47), evaluated on the device."""

from __future__ import annotations

import ctypes

import numpy as np

from paper_2404_11894_b200 import _native as N


def _to_device(a):
    torch = N.require_cuda()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64).reshape(-1, 3)).to("cuda")


def aggregate_indirect(graph, incoming: np.ndarray) -> np.ndarray:
    """I-bar = coeff * (W @ incoming) (operators.py:17-19)."""
    torch = N.require_cuda()
    src = _to_device(incoming)
    out = torch.empty_like(src)
    N.check(N.lib().vpg_aggregate_indirect(graph.native.handle, src.data_ptr(), out.data_ptr(),
                                           N.stream_handle()))
    return out.cpu().numpy()


def aggregate_direct(graph) -> np.ndarray:
    """D-bar per record, computed once at build (operators.py:22-24)."""
    return graph.d_bar


def _propagate(graph, l_bar, linear: int) -> np.ndarray:
    torch = N.require_cuda()
    src = _to_device(l_bar)
    out = torch.empty_like(src)
    st = graph.records.device()
    N.check(N.lib().vpg_propagate(ctypes.byref(st), src.data_ptr(), out.data_ptr(), linear,
                                  N.stream_handle()))
    return out.cpu().numpy()


def propagate(graph, l_bar: np.ndarray) -> np.ndarray:
    """I(x_{i-1}) = w_cont(x_i) * L-bar(x_i); terminal records keep i_pt (operators.py:27-38)."""
    return _propagate(graph, l_bar, 0)


def propagate_linear(graph, l_bar: np.ndarray) -> np.ndarray:
    """The linear part of propagate: zero at terminal records (operators.py:41-47)."""
    return _propagate(graph, l_bar, 1)
