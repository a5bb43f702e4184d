"""Portable float map I/O for the harness (the reference declares it at
harness/pfm.py and SPEC.md:390-409): colour "PF" files, little-endian
float32, rows stored bottom to top.  Images in memory are (H, W, 3) with row
0 at the top; a write/read round trip is bit-exact for float32 values."""

from __future__ import annotations

import numpy as np


class PfmError(IOError):
    pass


def write_pfm(image, path) -> None:
    data = np.asarray(image, dtype="<f4")
    if data.ndim != 3 or data.shape[2] != 3:
        raise PfmError(f"a PFM colour image is (height, width, 3), got {data.shape}")
    height, width = data.shape[:2]
    header = b"PF\n%d %d\n-1.0\n" % (width, height)
    with open(path, "wb") as f:
        f.write(header)
        f.write(np.flipud(data).astype("<f4", copy=False).tobytes(order="C"))


def _tokens(f, count):
    out, cur = [], bytearray()
    while len(out) < count:
        ch = f.read(1)
        if not ch:
            raise PfmError("PFM header ends early")
        if ch.isspace():
            if cur:
                out.append(bytes(cur))
                cur = bytearray()
        else:
            cur += ch
    return out


def read_pfm(path) -> np.ndarray:
    with open(path, "rb") as f:
        magic, w, h, scale = _tokens(f, 4)
        if magic == b"Pf":
            raise PfmError(f"{path}: greyscale PFM is not supported")
        if magic != b"PF":
            raise PfmError(f"{path}: not a PFM file")
        width, height, scale = int(w), int(h), float(scale)
        if scale >= 0.0:
            raise PfmError(f"{path}: big-endian PFM is not supported")
        raw = f.read(12 * width * height)
    if len(raw) != 12 * width * height:
        raise PfmError(f"{path}: pixel data is truncated")
    img = np.frombuffer(raw, dtype="<f4").reshape(height, width, 3)
    return np.ascontiguousarray(np.flipud(img))
