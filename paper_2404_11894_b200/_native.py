"""ctypes binding of libvolpg_b200.so (include/volpg_b200.h).

The library is the only compute path: if it is missing or CUDA is absent the
calls raise instead of falling back to a CPU implementation.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# VPG_LIB_VARIANT=name loads _lib/variants/libvolpg_b200_<name>.so (build
# experiments: tools/build_variant.py); the default is the in-tree build
_VARIANT = os.environ.get("VPG_LIB_VARIANT")
LIB_PATH = os.path.join(_HERE, "_lib", "libvolpg_b200.so") if not _VARIANT else \
    os.path.join(_HERE, "_lib", "variants", f"libvolpg_b200_{_VARIANT}.so")

VPG_OK, VPG_EINVAL, VPG_ECUDA, VPG_EDIVERGED, VPG_ENOMEM, VPG_ELIMIT = 0, -1, -2, -3, -4, -5
VPG_BUILD_TIMINGS = 1
VPG_BUILD_CLUSTERS_ONLY = 2
SCRATCH_DOUBLES = 40  # VPG_SCRATCH_DOUBLES: one capture-scratch record
DIRECT_PT, DIRECT_EXTRA, DIRECT_AGGREGATED = 0, 1, 2
MAX_SURF, MAX_EMIT, MAX_MED = 32, 16, 8

c_i32, c_i64, c_u32, c_u64, c_f64, c_p = C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_double, C.c_void_p


class Pcg64State(C.Structure):
    _fields_ = [("state_hi", c_u64), ("state_lo", c_u64), ("inc_hi", c_u64), ("inc_lo", c_u64),
                ("has_uint32", c_i32), ("uinteger", c_u32)]

    @classmethod
    def from_generator(cls, gen: np.random.Generator) -> "Pcg64State":
        st = gen.bit_generator.state
        if st["bit_generator"] != "PCG64":
            raise ValueError("cluster_points needs a PCG64-backed numpy Generator")
        s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
        m = (1 << 64) - 1
        return cls(s >> 64, s & m, inc >> 64, inc & m, int(st["has_uint32"]), int(st["uinteger"]))

    def store_into(self, gen: np.random.Generator) -> None:
        st = gen.bit_generator.state
        st["state"]["state"] = (int(self.state_hi) << 64) | int(self.state_lo)
        st["state"]["inc"] = (int(self.inc_hi) << 64) | int(self.inc_lo)
        st["has_uint32"] = int(self.has_uint32)
        st["uinteger"] = int(self.uinteger)
        gen.bit_generator.state = st


RECORD_FIELDS = [  # (name, width, ctype pointer) in vpg_records order
    ("pos", 3, "f8"), ("omega_out", 3, "f8"), ("normal", 3, "f8"), ("coeff", 3, "f8"),
    ("g", 1, "f8"), ("phase_dir", 3, "f8"), ("pdf_phase", 1, "f8"),
    ("pdf_emit_at_phase", 1, "f8"), ("emit_dir", 3, "f8"), ("pdf_emit", 1, "f8"),
    ("d_emit", 3, "f8"), ("d_phase", 3, "f8"), ("i_pt", 3, "f8"), ("w_cont", 3, "f8"),
    ("kind", 1, "u1"), ("emit_delta", 1, "u1"), ("class_id", 1, "i4"), ("path_idx", 1, "i8"),
    ("depth", 1, "i4"),
]
PATH_FIELDS = [
    ("pixel_idx", 1, "i8"), ("rec_start", 1, "i8"), ("rec_count", 1, "i4"),
    ("cam_weight", 3, "f8"), ("d_cam", 3, "f8"), ("direct0", 3, "f8"),
    ("direct0_nee", 3, "f8"), ("direct0_phase", 3, "f8"), ("extra_direct", 3, "f8"),
    ("pt_estimate", 3, "f8"),
]


class Records(C.Structure):
    _fields_ = [("n", c_i64)] + [(name, c_p) for name, _, _ in RECORD_FIELDS]


class Paths(C.Structure):
    _fields_ = [("n", c_i64)] + [(name, c_p) for name, _, _ in PATH_FIELDS]


class GraphInfo(C.Structure):
    _fields_ = [("n_records", c_i64), ("n_clusters", c_i64), ("nnz", c_i64), ("n_classes", c_i64),
                ("n_splits", c_i64), ("n_fallback", c_i64), ("build_ms", c_f64 * 8),
                ("n_staged", c_i64), ("split_visits", c_i64)]


class GraphViews(C.Structure):
    _fields_ = ([("n", c_i64), ("m", c_i64), ("n_halo", c_i64)] +
                [(f, c_p) for f in ("perm", "clpos", "cluster_id", "cl_off", "cl_size",
                                    "cl_center", "ref_of", "internal_of", "i0")] +
                [("ibuf", c_p * 2), ("acc", c_p * 2), ("dbar", c_p), ("term_max", c_p),
                 ("red", c_p), ("ctl", c_p), ("performed", c_i32), ("_pad", c_i32)])


class CodecField(C.Structure):
    _fields_ = [("offset", c_i32), ("bytes", c_i32), ("ptr", c_p)]


def _arr(t, *dims):
    for d in reversed(dims):
        t = t * d
    return t


class SceneStruct(C.Structure):
    _fields_ = [
        ("n_surf", c_i32), ("n_emit", c_i32), ("n_med", c_i32), ("width", c_i32),
        ("height", c_i32), ("_pad0", c_i32),
        ("surf_type", _arr(c_i32, MAX_SURF)), ("mat_type", _arr(c_i32, MAX_SURF)),
        ("emitter_id", _arr(c_i32, MAX_SURF)), ("surf_params", _arr(c_f64, MAX_SURF, 9)),
        ("albedo", _arr(c_f64, MAX_SURF, 3)),
        ("em_type", _arr(c_i32, MAX_EMIT)), ("em_value", _arr(c_f64, MAX_EMIT, 3)),
        ("em_pos", _arr(c_f64, MAX_EMIT, 3)), ("em_quad", _arr(c_f64, MAX_EMIT, 9)),
        ("em_normal", _arr(c_f64, MAX_EMIT, 3)), ("em_area", _arr(c_f64, MAX_EMIT)),
        ("med_kind", _arr(c_i32, MAX_MED)), ("grid_dims", _arr(c_i32, MAX_MED, 3)),
        ("med_sigma_t", _arr(c_f64, MAX_MED, 3)), ("med_sigma_s", _arr(c_f64, MAX_MED, 3)),
        ("med_g", _arr(c_f64, MAX_MED)), ("med_bounds", _arr(c_f64, MAX_MED, 6)),
        ("med_majorant", _arr(c_f64, MAX_MED)), ("med_scale", _arr(c_f64, MAX_MED)),
        ("grid_offset", _arr(c_i64, MAX_MED)), ("grid_data", c_p), ("cam", _arr(c_f64, 15)),
    ]


class TraceCfg(C.Structure):
    _fields_ = [("spp", c_i32), ("max_depth", c_i32), ("rr_start", c_i32), ("_pad", c_i32),
                ("rr_floor", c_f64), ("seed", c_i64), ("path_begin", c_i64), ("path_count", c_i64)]


_SIGNATURES = {
    "vpg_abi_version": (C.c_int, []),
    "vpg_last_error": (C.c_char_p, []),
    "vpg_launch_count": (c_u64, []),
    "vpg_transfer_bytes": (None, [C.POINTER(c_u64), C.POINTER(c_u64)]),
    "vpg_struct_size": (C.c_size_t, [c_i32]),
    "vpg_profile_enable": (None, [c_i32]),
    "vpg_profile_reset": (C.c_int, []),
    "vpg_profile_read": (C.c_int, [C.c_char_p, c_i64, c_p, c_p, c_i64, C.POINTER(c_i64)]),
    "vpg_profile_timeline": (C.c_int, [C.c_char_p, c_i64, c_p, c_p, c_i64, C.POINTER(c_i64)]),
    "vpg_rng_choice_device": (C.c_int, [C.POINTER(Pcg64State), c_i64, c_i64, c_p, c_p]),
    "vpg_split_groups_device": (C.c_int, [C.POINTER(Pcg64State), c_p, c_p, c_p, c_p, c_p, c_i64,
                                          c_p, c_p, c_p, c_i64, c_i64, C.POINTER(c_i64), c_p, c_p,
                                          c_p, C.POINTER(c_i64), c_p]),
    "vpg_graph_set_records": (C.c_int, [c_p, C.POINTER(Records)]),
    "vpg_rng_choice": (C.c_int, [C.POINTER(Pcg64State), c_i64, c_i64, c_p]),
    "vpg_rng_integers": (C.c_int, [C.POINTER(Pcg64State), c_i64, c_i64, c_p]),
    "vpg_split_groups": (C.c_int, [C.POINTER(Pcg64State), c_p, c_i64, c_p, c_p, c_p, c_i64, c_i64,
                                   c_p, c_p, c_p, c_p]),
    "vpg_unpack_rows": (C.c_int, [c_p, c_i64, c_i32, C.POINTER(CodecField), c_i32, c_p]),
    "vpg_pack_rows": (C.c_int, [c_p, c_i64, c_i32, C.POINTER(CodecField), c_i32, c_p]),
    "vpg_split_groups_soa": (C.c_int, [C.POINTER(Pcg64State), c_p, c_p, c_p, c_p, c_p, c_i64, c_p,
                                       c_p, c_p, c_i64, c_i64, C.POINTER(c_i64), c_p, c_p, c_p,
                                       C.POINTER(c_i64)]),
    "vpg_assign_nearest": (C.c_int, [c_p, c_i64, c_p, c_i64, c_p, c_p, C.POINTER(c_i64), c_p]),
    "vpg_graph_build": (C.c_int, [C.POINTER(Records), c_i32, C.POINTER(Pcg64State), c_i32, c_p,
                                  C.POINTER(c_p)]),
    "vpg_graph_build_wait": (C.c_int, [C.POINTER(Records), c_i32, C.POINTER(Pcg64State), c_i32, c_p,
                                       c_p, C.POINTER(c_p)]),
    "vpg_graph_info_get": (C.c_int, [c_p, C.POINTER(GraphInfo)]),
    "vpg_graph_free": (C.c_int, [c_p]),
    "vpg_graph_export_clusters": (C.c_int, [c_p, c_p, c_p, c_p, c_p, c_p]),
    "vpg_graph_export_marginals": (C.c_int, [c_p, c_p, c_p, c_p, c_p]),
    "vpg_graph_export_operators": (C.c_int, [c_p, c_p, c_p, c_p, c_p, c_p]),
    "vpg_solve": (C.c_int, [c_p, c_i32, c_f64, c_p, C.POINTER(c_i32), c_p]),
    "vpg_solve_export": (C.c_int, [c_p, c_p, c_p, c_p]),
    "vpg_aggregate_indirect": (C.c_int, [c_p, c_p, c_p, c_p]),
    "vpg_propagate": (C.c_int, [C.POINTER(Records), c_p, c_p, c_i32, c_p]),
    "vpg_splat": (C.c_int, [c_p, C.POINTER(Paths), c_i32, c_i32, c_i32, c_i32, c_p, c_p]),
    "vpg_splat_pt": (C.c_int, [C.POINTER(Paths), c_i32, c_i32, c_i32, c_p, c_p]),
    "vpg_trace_image": (C.c_int, [C.POINTER(SceneStruct), C.POINTER(TraceCfg), c_p, c_p]),
    "vpg_trace_count": (C.c_int, [C.POINTER(SceneStruct), C.POINTER(TraceCfg), c_p,
                                  C.POINTER(Paths), c_p]),
    "vpg_trace_fill": (C.c_int, [C.POINTER(SceneStruct), C.POINTER(TraceCfg), C.POINTER(Records),
                                 C.POINTER(Paths), c_p]),
    "vpg_extra_direct": (C.c_int, [C.POINTER(SceneStruct), C.POINTER(Records), C.POINTER(Paths),
                                   c_i64, c_i32, c_p]),
    "vpg_trace_capture": (C.c_int, [C.POINTER(SceneStruct), C.POINTER(TraceCfg), c_p,
                                    c_i64, c_p, c_p, C.POINTER(Paths), c_p]),
    "vpg_scatter_records": (C.c_int, [c_p, c_i64, c_p, c_i64, C.POINTER(Records),
                                      c_p]),
    "vpg_graph_build_local": (C.c_int, [C.POINTER(Records), c_i64, c_p, c_p, c_p, c_i64, c_p, c_p,
                                        C.POINTER(c_p)]),
    "vpg_graph_views_get": (C.c_int, [c_p, C.POINTER(GraphViews)]),
    "vpg_solve_begin": (C.c_int, [c_p, c_i32, c_f64, c_p]),
    "vpg_solve_step": (C.c_int, [c_p, c_i32, c_p]),
    "vpg_solve_control": (C.c_int, [c_p, c_i32, c_p]),
    "vpg_solve_end": (C.c_int, [c_p, c_p, C.POINTER(c_i32), c_p]),
    "vpg_splat_arrays": (C.c_int, [C.POINTER(Paths), c_p, c_p, c_p, c_p, c_i64, c_i32, c_i32, c_p,
                                   c_p]),
    "vpg_release_cached": (C.c_int, []),
    "vpg_extra_direct_range": (C.c_int, [C.POINTER(SceneStruct), C.POINTER(Records),
                                         C.POINTER(Paths), c_i64, c_i64, c_i32, c_p]),
    "vpg_reconstruct_paths": (C.c_int, [C.POINTER(Records), C.POINTER(Paths), c_p, c_i64, c_p, c_p,
                                        c_p]),
}

_lock = threading.Lock()
_lib = None


class NativeError(RuntimeError):
    pass


def lib():
    """Load (building first if needed) libvolpg_b200.so; raise if impossible."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            from paper_2404_11894_b200 import build as _build

            _build.build()
        handle = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        for which, st in enumerate((Pcg64State, Records, Paths, GraphInfo, SceneStruct, TraceCfg,
                                    GraphViews)):
            if handle.vpg_struct_size(which) != C.sizeof(st):
                raise NativeError(f"ABI mismatch for {st.__name__}: "
                                  f"{handle.vpg_struct_size(which)} != {C.sizeof(st)}")
        _lib = handle
        return _lib


def check(rc: int) -> None:
    """Map a VPG_E* code to the reference's exception types."""
    if rc == VPG_OK:
        return
    msg = lib().vpg_last_error().decode(errors="replace")
    if rc in (VPG_EINVAL, VPG_ELIMIT):
        raise ValueError(msg)
    if rc == VPG_ENOMEM:
        raise MemoryError(msg)
    if rc == VPG_EDIVERGED:
        from paper_2404_11894_b200.pathgraph.solve import SolveDivergence

        raise SolveDivergence(msg)
    raise NativeError(msg)


def profile_timeline():
    """[(name, start_ms, dur_ms)] of every profiled launch, in launch order."""
    cap = 1 << 16
    names = C.create_string_buffer(cap * 48)
    st = np.zeros(cap)
    du = np.zeros(cap)
    n = c_i64()
    check(lib().vpg_profile_timeline(names, len(names), st.ctypes.data, du.ctypes.data, cap,
                                     C.byref(n)))
    keys = names.value.decode().split("\n")
    return [(keys[i], float(st[i]), float(du[i])) for i in range(min(n.value, cap))]


def release_cached() -> None:
    """Free the library's scratch buffers and trimmed pool memory (and torch's
    cache) so the HBM is available to other allocators."""
    import torch

    check(lib().vpg_release_cached())
    torch.cuda.empty_cache()


def launch_count() -> int:
    return int(lib().vpg_launch_count())


def transfer_bytes() -> tuple[int, int]:
    h, d = c_u64(), c_u64()
    lib().vpg_transfer_bytes(C.byref(h), C.byref(d))
    return int(h.value), int(d.value)


def profile(enable: bool) -> None:
    lib().vpg_profile_enable(1 if enable else 0)


def profile_reset() -> None:
    check(lib().vpg_profile_reset())


def profile_read() -> dict:
    """{kernel name: (launches, total device ms)} since the last reset."""
    cap = 256
    names = C.create_string_buffer(1 << 16)
    counts = np.zeros(cap, dtype=np.int64)
    ms = np.zeros(cap)
    nk = c_i64()
    check(lib().vpg_profile_read(names, len(names), counts.ctypes.data, ms.ctypes.data, cap,
                                 C.byref(nk)))
    keys = names.value.decode().split("\n")[: nk.value]
    return {k: (int(counts[i]), float(ms[i])) for i, k in enumerate(keys)}


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise NativeError("libvolpg_b200 needs a CUDA device (no CPU fallback)")
    return torch


def stream_handle() -> int:
    torch = require_cuda()
    return int(torch.cuda.current_stream().cuda_stream)
