"""Tracing API over the CUDA tracer (reference: transport/tracer.py:37-127).

render_pt captures records in one device pass (the reference traces twice:
count, exclusive scan of the counts into rec_start, fill); the record set
stays in HBM and host copies are made only for fields a caller reads.  Path ids are
(y*W + x)*spp + s and every path owns its splitmix64 stream, so a record set
is identical however the paths are partitioned (multi-GPU row partition:
`path_range`).
"""

from __future__ import annotations

import ctypes

import numpy as np

from paper_2404_11894_b200 import _native as N
from paper_2404_11894_b200.harness.config import RenderConfig
from paper_2404_11894_b200.scenecore.flatten import pack_scene
from paper_2404_11894_b200.transport.records import PathSoA, RecordSoA, TraceOutput


def _cfg(config: RenderConfig, begin: int, count: int) -> N.TraceCfg:
    c = N.TraceCfg()
    c.spp, c.max_depth, c.rr_start = int(config.spp), int(config.max_depth), int(config.rr_start)
    c.rr_floor = float(config.rr_floor)
    c.seed = int(np.int64(config.seed))
    c.path_begin, c.path_count = int(begin), int(count)
    return c


def _alloc(fields, n, torch, zero=True):
    out = {}
    dt = {"f8": torch.float64, "i8": torch.int64, "i4": torch.int32, "u1": torch.uint8}
    make = torch.zeros if zero else torch.empty
    for name, width, code in fields:
        shape = (n, width) if width > 1 else (n,)
        out[name] = make(shape, dtype=dt[code], device="cuda")
    return out


def _struct(cls, tensors, n):
    st = cls()
    st.n = n
    for name, t in tensors.items():
        setattr(st, name, t.data_ptr() if t.numel() else None)
    return st


_CAPACITY_HINT: dict = {}  # (scene id, spp, depth, seed, range) -> record count of the last trace
# Capture scratch, kept across calls (grow-only): re-allocating ~290 B x
# capacity every frame costs more than the scatter itself.
_SCRATCH: dict = {"capacity": 0, "tensors": None}


def _scratch(capacity, torch):
    """Slot-major capture scratch: capacity x SCRATCH_DOUBLES float64."""
    if _SCRATCH["capacity"] < capacity or _SCRATCH["tensors"] is None:
        _SCRATCH["tensors"] = None
        _SCRATCH["tensors"] = torch.empty((max(capacity, 1), N.SCRATCH_DOUBLES),
                                          dtype=torch.float64, device="cuda")
        _SCRATCH["capacity"] = capacity
    return _SCRATCH["tensors"], _SCRATCH["capacity"]


def release_scratch():
    """Free the capture scratch (it is otherwise kept for the next trace)."""
    _SCRATCH["tensors"], _SCRATCH["capacity"] = None, 0


def trace_records_device(scene, config: RenderConfig, path_range=None, capture: bool = True):
    """Record-capturing trace; returns (records dict, paths dict, n_records) on the device.

    Single pass (default): records land in scratch slots, then are gathered
    into path order (rec_start = exclusive scan of the per-path counts).
    capture=False runs the reference's two passes instead (count, then
    re-trace and fill at the prefix-sum offsets; tracer.py:58-70).
    """
    torch = N.require_cuda()
    packed = pack_scene(scene)
    sc = packed.device()
    n_all = packed.width * packed.height * int(config.spp)
    begin, count = (0, n_all) if path_range is None else path_range
    cfg = _cfg(config, begin, count)
    paths = _alloc(N.PATH_FIELDS, count, torch)
    pst = _struct(N.Paths, paths, count)
    stream = N.stream_handle()
    lib = N.lib()
    counts = torch.empty(count, dtype=torch.int64, device="cuda")
    if capture:
        key = (id(scene), int(config.spp), int(config.max_depth), int(config.seed), begin, count)
        capacity = _CAPACITY_HINT.get(key, max(64, 6 * count))
        counter = torch.zeros(1, dtype=torch.int64, device="cuda")
        while True:
            scratch, capacity = _scratch(capacity, torch)
            N.check(lib.vpg_trace_capture(ctypes.byref(sc), ctypes.byref(cfg), scratch.data_ptr(),
                                          capacity, counter.data_ptr(), counts.data_ptr(),
                                          ctypes.byref(pst), stream))
            n_rec = int(counter.item())
            if n_rec <= capacity:
                break
            capacity = n_rec  # dropped records: retrace with exactly enough room
        _CAPACITY_HINT[key] = n_rec
    else:
        N.check(lib.vpg_trace_count(ctypes.byref(sc), ctypes.byref(cfg), counts.data_ptr(),
                                    ctypes.byref(pst), stream))
        n_rec = int(counts.sum().item()) if count else 0
    if count:
        torch.cumsum(counts, 0, out=paths["rec_start"])
        paths["rec_start"] -= counts
    paths["rec_count"].copy_(counts)
    paths["pixel_idx"].copy_(torch.arange(begin, begin + count, device="cuda") // int(config.spp))
    recs = _alloc(N.RECORD_FIELDS, n_rec, torch, zero=False)
    rst = _struct(N.Records, recs, n_rec)
    if capture:
        if n_rec:
            N.check(lib.vpg_scatter_records(scratch.data_ptr(), n_rec, paths["rec_start"].data_ptr(),
                                            begin, ctypes.byref(rst), stream))
    else:
        N.check(lib.vpg_trace_fill(ctypes.byref(sc), ctypes.byref(cfg), ctypes.byref(rst),
                                   ctypes.byref(pst), stream))
    return recs, paths, n_rec


def render_pt(scene, config: RenderConfig, with_records: bool = False) -> TraceOutput:
    """Path-trace the scene; optionally keep the record set (on the device)."""
    torch = N.require_cuda()
    packed = pack_scene(scene)
    w, h, spp = packed.width, packed.height, int(config.spp)
    if not with_records:
        sc = packed.device()
        cfg = _cfg(config, 0, w * h * spp)
        img = torch.empty((h, w, 3), dtype=torch.float64, device="cuda")
        N.check(N.lib().vpg_trace_image(ctypes.byref(sc), ctypes.byref(cfg), img.data_ptr(),
                                        N.stream_handle()))
        return TraceOutput(img.cpu().numpy(), RecordSoA.empty(0), PathSoA.empty(0), w, h, spp)
    recs, paths, n_rec = trace_records_device(scene, config)
    out = TraceOutput(None, RecordSoA.from_device(recs, n_rec),
                      PathSoA.from_device(paths, w * h * spp), w, h, spp)
    return out


def trace_path(scene, pixel, config: RenderConfig, sample: int = 0):
    """Trace one camera path with the stream the full render uses for it."""
    packed = pack_scene(scene)
    px, py = int(pixel[0]), int(pixel[1])
    if not (0 <= px < packed.width and 0 <= py < packed.height):
        raise ValueError(f"pixel {pixel} outside resolution {(packed.width, packed.height)}")
    path_id = (py * packed.width + px) * int(config.spp) + int(sample)
    recs, paths, n_rec = trace_records_device(scene, config, (path_id, 1))
    records = RecordSoA(**{k: v.cpu().numpy() for k, v in recs.items()})
    host = {k: v.cpu().numpy() for k, v in paths.items()}
    host["pixel_idx"][0] = py * packed.width + px
    return records, PathSoA(**host)


def record_extra_direct(scene, out: TraceOutput, n_extra: int, seed=None) -> np.ndarray:
    """n_extra additional first-bounce NEE samples averaged into extra_direct."""
    if n_extra < 0:
        raise ValueError("n_extra must be >= 0")
    if n_extra == 0:
        if out.paths.on_device():
            dev = out.paths.device_tensors()
            dev["extra_direct"].copy_(dev["direct0"])
            out.paths._host.pop("extra_direct", None)
        else:
            out.paths.extra_direct = out.paths.direct0.copy()
        return out.paths.extra_direct
    packed = pack_scene(scene)
    sc = packed.device()
    rst = out.records.device()
    pst = out.paths.device()
    N.check(N.lib().vpg_extra_direct(ctypes.byref(sc), ctypes.byref(rst), ctypes.byref(pst),
                                     int(np.int64(0 if seed is None else seed)), int(n_extra),
                                     N.stream_handle()))
    out.paths._host.pop("extra_direct", None)
    return out.paths.extra_direct
