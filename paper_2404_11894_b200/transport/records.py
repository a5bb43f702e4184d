"""Vertex records and the per-path table, structure-of-arrays, host or HBM.

Same fields, dtypes and semantics as the reference (transport/records.py:27-
188): one record per scatter/surface event, contiguous per path in depth
order, paths in (pixel, sample) order.  A `RecordSoA` / `PathSoA` here can be
backed by host numpy arrays (built by a caller or loaded from a VPGR dump) or
by device tensors written by the CUDA tracer; each side is materialised on
first use and cached, so a device-traced record set never visits the host
unless a caller reads a field.

The VPGR dump format (records.py:191-256) is byte-compatible with the
reference: magic, "<IQQIII" header, packed 290-byte records, 188-byte paths.
"""

from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from paper_2404_11894_b200 import _native as N

VPGR_MAGIC = b"VPGR"
VPGR_VERSION = 1
KIND_VOLUME = 0
KIND_SURFACE = 1


def _packed_dtype(fields):
    parts = []
    for name, width, code in fields:
        base = "<" + code
        parts.append((name, base, (width,)) if width > 1 else (name, base))
    return np.dtype(parts)


RECORD_DTYPE = _packed_dtype(N.RECORD_FIELDS)
PATH_DTYPE = _packed_dtype(N.PATH_FIELDS)
assert RECORD_DTYPE.itemsize == 290 and PATH_DTYPE.itemsize == 188


def _torch():
    import torch

    return torch


class _DualSoA:
    """Fields live on the host (numpy), on the device (torch), or both."""

    _FIELDS: list = []
    _STRUCT = None

    def __init__(self, host: dict, dev: Optional[dict] = None, n: Optional[int] = None):
        object.__setattr__(self, "_host", host)
        object.__setattr__(self, "_dev", dev)
        if n is None:
            first = self._FIELDS[0][0]
            n = host[first].shape[0] if first in host else dev[first].shape[0]
        object.__setattr__(self, "_n", int(n))
        object.__setattr__(self, "_struct", None)
        object.__setattr__(self, "_pinned", None)

    @property
    def n(self) -> int:
        return self._n

    def _get(self, name):
        arr = self._host.get(name)
        if arr is None:
            if self._dev is None:
                raise AttributeError(name)
            arr = self._dev[name].cpu().numpy()
            self._host[name] = arr
        return arr

    def _set(self, name, value, width, code):
        arr = np.ascontiguousarray(value, dtype=np.dtype("<" + code))
        if self._dev is not None and name in self._dev:
            dev = self._dev[name]
            if tuple(dev.shape) == arr.shape:
                dev.copy_(_torch().from_numpy(arr))  # keep both sides in step
            else:
                # new length: the device copy is dropped (graphs keep their own reference)
                for other, _, _ in self._FIELDS:
                    self._get(other)
                object.__setattr__(self, "_dev", None)
                object.__setattr__(self, "_missing", set())
                object.__setattr__(self, "_struct", None)
                object.__setattr__(self, "_n", int(arr.shape[0]))
        self._host[name] = arr

    def on_device(self) -> bool:
        return self._dev is not None

    def pin_memory(self):
        """Re-home the host arrays in page-locked memory (fast, async H2D)."""
        torch = _torch()
        pinned = {}
        for name, _, _ in self._FIELDS:
            src = self._get(name)
            t = torch.from_numpy(np.ascontiguousarray(src)).pin_memory()
            pinned[name] = t
            self._host[name] = t.numpy()
        object.__setattr__(self, "_pinned", pinned)
        return self

    # fields a consumer may need before the rest (RecordSoA: the clustering's)
    _EARLY: tuple = ()

    def upload_async(self, skip=()):
        """Start the host->device copies of a pinned SoA on the copy stream:
        the _EARLY fields first, then the rest, each group closed by an event
        ("early", "all").  Consumers wait on the group they need (device()
        waits on "all"), so compute that needs only the early fields overlaps
        the rest of the transfer.  Fields in `skip` stay on the host until a
        device() call asks for them (the graph solve never reads them)."""
        if self._dev is not None:
            return
        torch = N.require_cuda()
        if self._pinned is None:
            self.device()
            return
        main = torch.cuda.current_stream()
        copy = _copy_stream(torch)
        copy.wait_stream(main)
        dev, events = {}, {}
        order = [f for f in self._FIELDS if f[0] in self._EARLY] + \
                [f for f in self._FIELDS if f[0] not in self._EARLY and f[0] not in skip]
        with torch.cuda.stream(copy):
            for k, (name, width, code) in enumerate(order):
                t = self._pinned[name].to("cuda", non_blocking=True)
                _count_h2d(t)
                t.record_stream(main)  # used on the main stream: no early reuse
                dev[name] = t
                if k + 1 == len(self._EARLY):
                    events["early"] = torch.cuda.Event()
                    events["early"].record(copy)
            events["all"] = torch.cuda.Event()
            events["all"].record(copy)
        object.__setattr__(self, "_dev", dev)
        object.__setattr__(self, "_events", events)
        object.__setattr__(self, "_missing", {f[0] for f in self._FIELDS} - set(dev))
        object.__setattr__(self, "_struct", None)

    def ready_event(self, group: str = "all"):
        """The upload event of a field group, None when nothing is in flight."""
        ev = self.__dict__.get("_events")
        return ev.get(group, ev.get("all")) if ev else None

    def device(self, stream=None, wait: str = "all", need=None):
        """Device tensors of the fields in `need` (all by default; uploaded on
        first use) and the ABI struct (null pointers for fields still on the
        host).  The current stream waits for the field group `wait` of an
        async upload."""
        if self._dev is None:
            torch = N.require_cuda()
            if self._pinned is not None:
                self.upload_async()
            else:
                dev = {}
                for name, width, code in self._FIELDS:
                    src = torch.from_numpy(np.ascontiguousarray(self._get(name)))
                    dev[name] = src.to("cuda")
                    _count_h2d(dev[name])
                object.__setattr__(self, "_dev", dev)
                object.__setattr__(self, "_struct", None)
        missing = self.__dict__.get("_missing") or set()
        lack = missing if need is None else missing & set(need)
        if lack:
            torch = N.require_cuda()
            for name in sorted(lack):
                src = self._pinned[name] if self._pinned is not None else \
                    torch.from_numpy(np.ascontiguousarray(self._get(name)))
                self._dev[name] = src.to("cuda", non_blocking=self._pinned is not None)
                _count_h2d(self._dev[name])
            object.__setattr__(self, "_missing", missing - lack)
            object.__setattr__(self, "_struct", None)
        ev = self.ready_event(wait)
        if ev is not None:
            _torch().cuda.current_stream().wait_event(ev)
        if self._struct is None:
            st = self._STRUCT()
            st.n = self._n
            for name, _, _ in self._FIELDS:
                t = self._dev.get(name)
                setattr(st, name, t.data_ptr() if t is not None and t.numel() else None)
            object.__setattr__(self, "_struct", st)
        return self._struct

    def device_tensors(self) -> dict:
        self.device()
        return self._dev

    def drop_host(self):
        """Forget cached host copies of device-resident fields."""
        if self._dev is not None:
            for name in list(self._host):
                if name in self._dev:
                    del self._host[name]

    def host_arrays(self) -> dict:
        return {name: self._get(name) for name, _, _ in self._FIELDS}


_COPY = {}
_H2D = [0]  # bytes this module has copied host -> device (upload accounting)


def _count_h2d(t):
    _H2D[0] += t.numel() * t.element_size()


def h2d_bytes() -> int:
    """Bytes of record / path fields copied to the device so far."""
    return _H2D[0]


def _copy_stream(torch):
    dev = torch.cuda.current_device()
    if dev not in _COPY:
        _COPY[dev] = torch.cuda.Stream()
    return _COPY[dev]


def _install_fields(cls):
    for name, width, code in cls._FIELDS:
        def getter(self, _n=name):
            return self._get(_n)

        def setter(self, value, _n=name, _w=width, _c=code):
            self._set(_n, value, _w, _c)

        setattr(cls, name, property(getter, setter))
    return cls


def _zeros(fields, n):
    out = {}
    for name, width, code in fields:
        shape = (n, width) if width > 1 else (n,)
        out[name] = np.zeros(shape, dtype=np.dtype("<" + code))
    return out


@_install_fields
class RecordSoA(_DualSoA):
    """Shading-point records (reference: records.py:75-140)."""

    _FIELDS = N.RECORD_FIELDS
    _STRUCT = N.Records
    _EARLY = ("pos", "kind", "class_id")  # all the clustering reads

    def __init__(self, *args, cluster_id=None, _dev=None, _n=None, **kwargs):
        host = {}
        names = [f[0] for f in self._FIELDS]
        for name, value in zip(names, args):
            kwargs[name] = value
        for name, width, code in self._FIELDS:
            if name in kwargs and kwargs[name] is not None:
                host[name] = np.ascontiguousarray(kwargs[name], dtype=np.dtype("<" + code))
        if _dev is None and len(host) != len(names):
            missing = [nm for nm in names if nm not in host]
            raise TypeError(f"RecordSoA missing fields: {missing}")
        super().__init__(host, _dev, _n)
        object.__setattr__(self, "_cluster_id", None)
        object.__setattr__(self, "_cluster_id_fn", None)
        if cluster_id is not None:
            self.cluster_id = cluster_id

    @property
    def cluster_id(self) -> np.ndarray:
        if self._cluster_id is None:
            if self._cluster_id_fn is not None:
                object.__setattr__(self, "_cluster_id", self._cluster_id_fn())
            else:
                object.__setattr__(self, "_cluster_id", np.full(self.n, -1, dtype=np.int64))
        return self._cluster_id

    @cluster_id.setter
    def cluster_id(self, value):
        object.__setattr__(self, "_cluster_id", np.asarray(value, dtype=np.int64))
        object.__setattr__(self, "_cluster_id_fn", None)

    def _set_cluster_provider(self, fn: Callable[[], np.ndarray]):
        object.__setattr__(self, "_cluster_id", None)
        object.__setattr__(self, "_cluster_id_fn", fn)

    @classmethod
    def empty(cls, n: int) -> "RecordSoA":
        return cls(**_zeros(cls._FIELDS, n))

    @classmethod
    def from_device(cls, tensors: dict, n: int) -> "RecordSoA":
        return cls(_dev=tensors, _n=n)

    def kernel_arrays(self):
        return tuple(self._get(name) for name, _, _ in self._FIELDS)

    def next_index(self) -> np.ndarray:
        """Continuation child per record: r + 1 when it is on the same path, else -1."""
        pid = self.path_idx
        nxt = np.full(self.n, -1, dtype=np.int64)
        if self.n > 1:
            rows = np.flatnonzero(pid[1:] == pid[:-1])
            nxt[rows] = rows + 1
        return nxt


@_install_fields
class PathSoA(_DualSoA):
    """Per-path table (reference: records.py:143-176)."""

    _FIELDS = N.PATH_FIELDS
    _STRUCT = N.Paths

    def __init__(self, *args, _dev=None, _n=None, **kwargs):
        host = {}
        names = [f[0] for f in self._FIELDS]
        for name, value in zip(names, args):
            kwargs[name] = value
        for name, width, code in self._FIELDS:
            if name in kwargs and kwargs[name] is not None:
                host[name] = np.ascontiguousarray(kwargs[name], dtype=np.dtype("<" + code))
        if _dev is None and len(host) != len(names):
            missing = [nm for nm in names if nm not in host]
            raise TypeError(f"PathSoA missing fields: {missing}")
        super().__init__(host, _dev, _n)

    @classmethod
    def empty(cls, n: int) -> "PathSoA":
        return cls(**_zeros(cls._FIELDS, n))

    @classmethod
    def from_device(cls, tensors: dict, n: int) -> "PathSoA":
        return cls(_dev=tensors, _n=n)

    def kernel_arrays(self):
        return (self.cam_weight, self.d_cam, self.direct0, self.direct0_nee,
                self.direct0_phase, self.pt_estimate)


class TraceOutput:
    """Everything one instrumented render produces (reference: records.py:179-188).

    `image` (the PT image) may be given or computed on the device on first access.
    """

    def __init__(self, image, records: RecordSoA, paths: PathSoA, width: int, height: int,
                 spp: int):
        self._image = image
        self.records = records
        self.paths = paths
        self.width = int(width)
        self.height = int(height)
        self.spp = int(spp)

    @property
    def image(self) -> np.ndarray:
        if self._image is None:
            self._image = splat_pt_image(self.paths, self.width, self.height, self.spp)
        return self._image

    @image.setter
    def image(self, value):
        self._image = value


# ------------------------------------------------ the reference's own objects
def as_records(obj) -> RecordSoA:
    """A RecordSoA for `obj`: ours as is, or any object carrying the
    reference's record fields as arrays (volpg.transport.records.RecordSoA,
    records.py:75-126) -- copied into a host RecordSoA."""
    if isinstance(obj, RecordSoA):
        return obj
    try:
        return RecordSoA(**{name: np.asarray(getattr(obj, name)) for name, _, _ in N.RECORD_FIELDS})
    except AttributeError as exc:
        raise TypeError(f"not a record set: {type(obj).__name__} lacks {exc}") from None


def as_paths(obj) -> PathSoA:
    """PathSoA for ours or the reference's path table (records.py:143-176)."""
    if isinstance(obj, PathSoA):
        return obj
    try:
        return PathSoA(**{name: np.asarray(getattr(obj, name)) for name, _, _ in N.PATH_FIELDS})
    except AttributeError as exc:
        raise TypeError(f"not a path table: {type(obj).__name__} lacks {exc}") from None


def as_trace(obj) -> TraceOutput:
    """TraceOutput for ours or the reference's (records.py:179-188): a
    volpg TraceOutput is wrapped (its arrays copied once to host SoAs); the
    caller writes results back where the reference mutates it (build_graph
    sets records.cluster_id, graph.py:62)."""
    if isinstance(obj, TraceOutput):
        return obj
    for a in ("records", "paths", "width", "height", "spp"):
        if not hasattr(obj, a):
            raise TypeError(f"not a trace: {type(obj).__name__} has no {a!r}")
    return TraceOutput(getattr(obj, "image", None), as_records(obj.records), as_paths(obj.paths),
                       obj.width, obj.height, obj.spp)


def splat_pt_image(paths: PathSoA, width: int, height: int, spp: int) -> np.ndarray:
    """Per-pixel mean of the PT estimates in sample order, on the device."""
    torch = N.require_cuda()
    st = paths.device()
    img = torch.empty((height, width, 3), dtype=torch.float64, device="cuda")
    N.check(N.lib().vpg_splat_pt(ctypes.byref(st), width, height, spp, img.data_ptr(),
                                 N.stream_handle()))
    return img.cpu().numpy()


_CODEC_CHUNK = 32 << 20  # bytes of packed rows per staged chunk
_STAGING = {}


def _staging(torch, nbytes):
    """Two (pinned host, device, event) staging buffers, cached per device."""
    key = torch.cuda.current_device()
    cur = _STAGING.get(key)
    if cur is None or cur[0][0].numel() < nbytes:
        cur = [(torch.empty(nbytes, dtype=torch.uint8).pin_memory(),
                torch.empty(nbytes, dtype=torch.uint8, device="cuda"), torch.cuda.Event())
               for _ in range(2)]
        for _, _, ev in cur:
            ev.record()
        _STAGING[key] = cur
    return cur


def _codec_table(dtype, dev: dict, r0: int):
    """CodecField array of a packed dtype against device arrays, rows from r0."""
    names = dtype.names
    table = (N.CodecField * len(names))()
    for i, name in enumerate(names):
        off = dtype.fields[name][1]
        nbytes = dtype.fields[name][0].itemsize
        table[i].offset = off
        table[i].bytes = nbytes
        table[i].ptr = dev[name].data_ptr() + r0 * nbytes
    return table


def _block_to_device(f, path, n, dtype, dev, torch, stream, what):
    """Stream n packed rows from the file into the device arrays: chunked
    reads into pinned staging, async upload and vpg_unpack_rows on `stream`,
    double-buffered so the read of chunk k+1 overlaps chunk k on the device."""
    row = dtype.itemsize
    per = max(1, _CODEC_CHUNK // row)
    bufs = _staging(torch, per * row)
    lib = N.lib()
    for c, r0 in enumerate(range(0, n, per)):
        host, devbuf, ev = bufs[c % 2]
        ev.synchronize()
        cnt = min(per, n - r0)
        nb = cnt * row
        got = f.readinto(memoryview(host.numpy())[:nb])
        if got != nb:
            raise IOError(f"{path}: truncated {what} block")
        with torch.cuda.stream(stream):
            devbuf[:nb].copy_(host[:nb], non_blocking=True)
            table = _codec_table(dtype, dev, r0)
            N.check(lib.vpg_unpack_rows(devbuf.data_ptr(), cnt, row, table, len(table),
                                        N.stream_handle()))
            ev.record(stream)


def _block_from_device(f, n, dtype, dev, torch, stream):
    """Write n rows of the device arrays as packed rows: vpg_pack_rows into a
    device staging chunk, async download to pinned memory, file write of the
    previous chunk while the next one packs."""
    row = dtype.itemsize
    per = max(1, _CODEC_CHUNK // row)
    bufs = _staging(torch, per * row)
    lib = N.lib()
    pending = None
    for c, r0 in enumerate(range(0, n, per)):
        host, devbuf, ev = bufs[c % 2]
        ev.synchronize()
        cnt = min(per, n - r0)
        nb = cnt * row
        with torch.cuda.stream(stream):
            table = _codec_table(dtype, dev, r0)
            N.check(lib.vpg_pack_rows(devbuf.data_ptr(), cnt, row, table, len(table),
                                      N.stream_handle()))
            host[:nb].copy_(devbuf[:nb], non_blocking=True)
            ev.record(stream)
        if pending is not None:
            pending[1].synchronize()
            f.write(memoryview(pending[0].numpy())[:pending[2]])
        pending = (host, ev, nb)
    if pending is not None:
        pending[1].synchronize()
        f.write(memoryview(pending[0].numpy())[:pending[2]])


def _write_header(f, out: TraceOutput):
    f.write(VPGR_MAGIC)
    f.write(struct.pack("<IQQIII", VPGR_VERSION, out.records.n, out.paths.n, out.width,
                        out.height, out.spp))


def save_records(path, out: TraceOutput) -> None:
    """Write the versioned VPGR dump (reference: records.py:191-217).

    Device-resident records (a device trace, or a device load) are packed on
    the device (vpg_pack_rows) and streamed to the file in chunks; host
    records are packed with numpy.  Either way the file is byte-identical to
    the reference's dump of the same records."""
    if out.records.on_device() and out.paths.on_device():
        torch = N.require_cuda()
        rdev, pdev = out.records.device_tensors(), out.paths.device_tensors()
        stream = _copy_stream(torch)
        stream.wait_stream(torch.cuda.current_stream())
        with open(path, "wb") as f:
            _write_header(f, out)
            _block_from_device(f, out.records.n, RECORD_DTYPE, rdev, torch, stream)
            _block_from_device(f, out.paths.n, PATH_DTYPE, pdev, torch, stream)
        return
    rec = np.zeros(out.records.n, dtype=RECORD_DTYPE)
    for name, _, _ in N.RECORD_FIELDS:
        rec[name] = out.records._get(name)
    pth = np.zeros(out.paths.n, dtype=PATH_DTYPE)
    for name, _, _ in N.PATH_FIELDS:
        pth[name] = out.paths._get(name)
    with open(path, "wb") as f:
        _write_header(f, out)
        f.write(rec.tobytes())
        f.write(pth.tobytes())


def _read_header(f, path):
    if f.read(4) != VPGR_MAGIC:
        raise IOError(f"{path}: not a VPGR record dump")
    head = f.read(32)
    if len(head) != 32:
        raise IOError(f"{path}: truncated VPGR header")
    version, n_rec, n_path, width, height, spp = struct.unpack("<IQQIII", head)
    if version != VPGR_VERSION:
        raise IOError(f"{path}: unsupported VPGR version {version}")
    return n_rec, n_path, width, height, spp


def _device_empty(torch, fields, n):
    out = {}
    for name, width, code in fields:
        np_dt = np.dtype("<" + code)
        t_dt = {np.dtype("<f8"): torch.float64, np.dtype("<i4"): torch.int32,
                np.dtype("<i8"): torch.int64, np.dtype("<u1"): torch.uint8}[np_dt]
        shape = (n, width) if width > 1 else (n,)
        out[name] = torch.empty(shape, dtype=t_dt, device="cuda")
    return out


def load_records(path, pin: bool = False, device: bool = False) -> TraceOutput:
    """Read a VPGR dump (reference: records.py:220-256).

    Host load (default): numpy SoA arrays; pin=True places them in
    page-locked memory for asynchronous upload.  device=True loads straight
    into HBM: the packed blocks are streamed through pinned staging chunks
    and transposed to SoA on the device (vpg_unpack_rows), so the records
    never exist as host SoA arrays (they materialise on first host read).
    A short or cut block raises IOError either way.
    """
    with open(path, "rb") as f:
        n_rec, n_path, width, height, spp = _read_header(f, path)
        if device:
            torch = N.require_cuda()
            main = torch.cuda.current_stream()
            stream = _copy_stream(torch)
            rdev = _device_empty(torch, N.RECORD_FIELDS, n_rec)
            pdev = _device_empty(torch, N.PATH_FIELDS, n_path)
            stream.wait_stream(main)
            _block_to_device(f, path, n_rec, RECORD_DTYPE, rdev, torch, stream, "record")
            _block_to_device(f, path, n_path, PATH_DTYPE, pdev, torch, stream, "path")
            main.wait_stream(stream)
            return TraceOutput(None, RecordSoA.from_device(rdev, n_rec),
                               PathSoA.from_device(pdev, n_path), width, height, spp)
        # a short block is a truncated dump (IOError, as the reference raises
        # for a block cut at a record boundary) wherever the cut falls
        raw = f.read(RECORD_DTYPE.itemsize * n_rec)
        if len(raw) != RECORD_DTYPE.itemsize * n_rec:
            raise IOError(f"{path}: truncated record block")
        rec = np.frombuffer(raw, dtype=RECORD_DTYPE)
        raw = f.read(PATH_DTYPE.itemsize * n_path)
        if len(raw) != PATH_DTYPE.itemsize * n_path:
            raise IOError(f"{path}: truncated path block")
        pth = np.frombuffer(raw, dtype=PATH_DTYPE)
    records = RecordSoA(**{name: np.ascontiguousarray(rec[name]) for name, _, _ in N.RECORD_FIELDS})
    paths = PathSoA(**{name: np.ascontiguousarray(pth[name]) for name, _, _ in N.PATH_FIELDS})
    if pin:
        records.pin_memory()
        paths.pin_memory()
    return TraceOutput(None, records, paths, width, height, spp)
