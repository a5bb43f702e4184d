"""Fixed-point solve and splat on the device (reference: pathgraph/solve.py).

`solve` runs I <- P A+ I + P Ao D entirely in HBM (vpg_solve): one kernel
per iteration (block-dense W*I per cluster, fused propagation into the parent
row and residual maxima) plus a one-thread control kernel that applies the
reference's residual, tol-break and divergence rules, so the loop never
waits on the host.  `SolveResult.incoming` / `.i_bar` / `.d_bar` are copied
to the host on first access.
"""

from __future__ import annotations

import csv
import ctypes

import numpy as np

from paper_2404_11894_b200 import _native as N


class SolveDivergence(RuntimeError):
    pass


class SolveResult:
    """incoming, i_bar, d_bar (N,3), residuals, iterations (solve.py:32-38)."""

    def __init__(self, graph, residuals, iterations, incoming=None, i_bar=None, d_bar=None):
        self._graph = graph
        self._generation = graph.native.solve_generation if graph._native is not None else 0
        self.residuals = list(residuals)
        self.iterations = int(iterations)
        self._arrays = {"incoming": incoming, "i_bar": i_bar, "d_bar": d_bar}

    def _fetch(self, name):
        if self._arrays[name] is None:
            g = self._graph.native
            if g.solve_generation != self._generation:
                raise RuntimeError("the graph was solved again; this SolveResult is stale")
            n = self._graph.records.n
            if name == "d_bar":
                self._arrays[name] = self._graph.d_bar
            else:
                inc, ib = np.empty((n, 3)), np.empty((n, 3))
                N.check(N.lib().vpg_solve_export(g.handle, inc.ctypes.data, ib.ctypes.data,
                                                  N.stream_handle()))
                self._arrays["incoming"], self._arrays["i_bar"] = inc, ib
        return self._arrays[name]

    incoming = property(lambda self: self._fetch("incoming"))
    i_bar = property(lambda self: self._fetch("i_bar"))
    d_bar = property(lambda self: self._fetch("d_bar"))


def residual_norm(new: np.ndarray, old: np.ndarray) -> float:
    """max over channels of max|new-old| / max(max|new|, 1e-12) (solve.py:54-61)."""
    new = np.asarray(new)
    old = np.asarray(old)
    worst = 0.0
    for c in range(3):
        scale = max(float(np.abs(new[:, c]).max(initial=0.0)), 1e-12)
        worst = max(worst, float(np.abs(new[:, c] - old[:, c]).max(initial=0.0)) / scale)
    return worst


def solve(graph, iterations: int = 10, tol: float = 1e-3) -> SolveResult:
    """Iterate to the fixed point on the device; raises SolveDivergence when the
    residual grows over 3 consecutive iterations."""
    if iterations < 0:
        raise ValueError("iterations must be >= 0")
    g = graph.native
    if iterations == 0 and graph.records.__dict__.get("_missing"):
        # the single-strategy I-bar reads pdf_phase (and normals): bring the
        # fields the build left on the host and re-point the graph at them
        st = graph.records.device()
        g.rec_tensors = dict(graph.records._dev)
        g.rec_struct = st
        N.check(N.lib().vpg_graph_set_records(g.handle, ctypes.byref(st)))
    res = np.zeros(max(iterations, 1))
    performed = ctypes.c_int32(0)
    rc = N.lib().vpg_solve(g.handle, int(iterations), float(tol), res.ctypes.data,
                           ctypes.byref(performed), N.stream_handle())
    g.solve_generation += 1
    g.performed = performed.value
    residuals = [float(r) for r in res[:performed.value]]
    if rc == N.VPG_EDIVERGED:
        raise SolveDivergence(
            "fixed-point residuals grew over 3 consecutive iterations "
            f"({residuals[-4:]}); recorded pdfs/weights are inconsistent")
    N.check(rc)
    return SolveResult(graph, residuals, performed.value)


def splat_output_device(graph, result: SolveResult, aggregate_direct_term: bool = False,
                        extra_direct: bool = False):
    """splat_output leaving the (H, W, 3) float64 image on the device."""
    torch = N.require_cuda()
    g = graph.native
    if result._generation != g.solve_generation:
        raise RuntimeError("the graph was solved again; this SolveResult is stale")
    mode = N.DIRECT_AGGREGATED if aggregate_direct_term else (
        N.DIRECT_EXTRA if extra_direct else N.DIRECT_PT)
    pst = graph.paths.device(need=("rec_start", "rec_count", "cam_weight", "d_cam",
                                   "extra_direct" if mode == N.DIRECT_EXTRA else "direct0"))
    img = torch.empty((graph.height, graph.width, 3), dtype=torch.float64, device="cuda")
    N.check(N.lib().vpg_splat(g.handle, ctypes.byref(pst), graph.width, graph.height, graph.spp,
                              mode, img.data_ptr(), N.stream_handle()))
    return img


def splat_output(graph, result: SolveResult, aggregate_direct_term: bool = False,
                 extra_direct: bool = False) -> np.ndarray:
    """Per path: d_cam + cam_weight * (direct + i_bar[first record]), averaged
    over spp in sample order (solve.py:101-132)."""
    return splat_output_device(graph, result, aggregate_direct_term, extra_direct).cpu().numpy()


def write_residual_csv(path, residuals) -> None:
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["iteration", "residual"])
        for i, r in enumerate(residuals, start=1):
            w.writerow([i, repr(float(r))])
