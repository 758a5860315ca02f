"""PFM image I/O for parity artefacts (proj/src/image.cpp:20-66, write_pfm / read_pfm).

Planar [C, H, W] float32 images (Image<float>, image.h:16-35) <-> Portable Float Map: header
"PF" (3 channels) / "Pf" (1), "W H", scale -1.0 (little endian); bottom-up scanlines of
interleaved samples.  Host-side only."""
from __future__ import annotations

import sys

import numpy as np

from ._abi import Error


def write_pfm(path, img) -> None:
    """write_pfm (image.cpp:20-35).  `img`: Image or float32 array [C, H, W] / [H, W]."""
    a = getattr(img, "data", img)
    a = np.asarray(a, np.float32)
    if a.ndim == 2:
        a = a[None]
    if a.shape[0] not in (1, 3):
        raise Error("pfm: 1 or 3 channels only")
    c, h, w = a.shape
    le = sys.byteorder == "little"
    hdr = f"{'PF' if c == 3 else 'Pf'}\n{w} {h}\n{'-1.0' if le else '1.0'}\n".encode()
    body = np.ascontiguousarray(a.transpose(1, 2, 0)[::-1])  # bottom-up rows, interleaved
    try:
        with open(path, "wb") as f:
            f.write(hdr)
            f.write(body.astype(np.float32).tobytes())
    except OSError as e:
        raise Error(f"pfm: cannot open for writing: {path}") from e


def read_pfm(path) -> np.ndarray:
    """read_pfm (image.cpp:36-66): returns float32 [C, H, W]."""
    try:
        raw = open(path, "rb").read()
    except OSError as e:
        raise Error(f"pfm: cannot open: {path}") from e
    parts = raw.split(maxsplit=4)
    if len(parts) < 5 or parts[0] not in (b"PF", b"Pf"):
        raise Error(f"pfm: bad magic in {path}")
    w, h, scale = int(parts[1]), int(parts[2]), float(parts[3])
    if w <= 0 or h <= 0:
        raise Error(f"pfm: bad dimensions in {path}")
    c = 3 if parts[0] == b"PF" else 1
    # the header ends with one whitespace byte after the scale token
    off = raw.index(parts[3], len(parts[0]) + len(parts[1]) + len(parts[2])) + len(parts[3]) + 1
    dt = np.dtype("<f4" if scale < 0 else ">f4")
    n = w * h * c
    if len(raw) - off < 4 * n:
        raise Error(f"pfm: truncated file: {path}")
    a = np.frombuffer(raw, dt, n, off).astype(np.float32).reshape(h, w, c)[::-1]
    return np.ascontiguousarray(a.transpose(2, 0, 1))
