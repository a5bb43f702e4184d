"""Pixel estimates recomputed from the records alone (reference:
transport/reconstruct.py:52-72), on the device.

Walking a path's records backward with the recorded pdfs, weights and raw
radiances reproduces the PT estimate the tracer accumulated forward; the
stored i_pt is cross-checked, not consumed.  `reconstruct_path_estimate` is
the reference's one-path call; `reconstruct_path_estimates` runs every path
(or a list) in one launch (vpg_reconstruct_paths).
"""

from __future__ import annotations

import ctypes

import numpy as np

from paper_2404_11894_b200 import _native as N
from paper_2404_11894_b200.transport.records import as_paths, as_records


def reconstruct_path_estimates(records, paths, path_indices=None):
    """(estimate (k,3) float64, max |stored i_pt - recomputed| (k,)) for the
    given paths (all of them by default)."""
    torch = N.require_cuda()
    records, paths = as_records(records), as_paths(paths)
    if path_indices is None:
        count, ids = paths.n, None
    else:
        idx = np.asarray(path_indices, dtype=np.int64).reshape(-1)
        if idx.size and (idx.min() < 0 or idx.max() >= paths.n):
            raise IndexError(f"path index out of range [0, {paths.n})")
        count, ids = int(idx.size), torch.as_tensor(idx, device="cuda")
    need_r = ("omega_out", "normal", "g", "coeff", "phase_dir", "pdf_phase", "pdf_emit_at_phase",
              "emit_dir", "pdf_emit", "d_emit", "d_phase", "i_pt", "w_cont", "kind", "emit_delta")
    rst = records.device(need=need_r)
    pst = paths.device(need=("rec_start", "rec_count", "d_cam"))
    est = torch.empty((count, 3), dtype=torch.float64, device="cuda")
    diff = torch.empty((count,), dtype=torch.float64, device="cuda")
    N.check(N.lib().vpg_reconstruct_paths(ctypes.byref(rst), ctypes.byref(pst),
                                          ids.data_ptr() if ids is not None else None, count,
                                          est.data_ptr(), diff.data_ptr(), N.stream_handle()))
    return est.cpu().numpy(), diff.cpu().numpy()


def reconstruct_path_estimate(records, paths, path_index: int):
    """Rebuild one path's pixel estimate from its records (reconstruct.py:52-72).

    Returns (estimate (3,), max |stored i_pt - recomputed|)."""
    est, diff = reconstruct_path_estimates(records, paths, [int(path_index)])
    return est[0], float(diff[0])
