"""LGA archive ("layered grid archive") I/O — drop-in for tomogram.py:219-276.

Byte-identical to the reference writer (format README.md:111-121): a 52-byte
little-endian header <4sIIIfdddfI, then per slice a 9-byte <dB header (plane
height, layer mask) and the float32 ground / ceiling / cost layers.

``save_tomogram`` assembles the archive in one page-locked host buffer:
layers that live on the GPU are copied by the DMA engine straight to their
byte offset in the archive (no intermediate numpy arrays, one
synchronisation), host layers are copied in place; the buffer is then
written to the file.  ``load_tomogram`` parses with the reference's checks
and error messages and returns host-resident layers.
"""

from __future__ import annotations

import ctypes as C
import struct
from pathlib import Path

import numpy as np

from . import _lib
from .tomogram import Layer, Tomogram, TomogramSlice

_MAGIC = b"LGA1"
_HEADER = struct.Struct("<4sIIIfdddfI")
_SLICE_HEADER = struct.Struct("<dB")

MASK_GROUND = 1
MASK_CEILING = 2
MASK_COST = 4


def archive_size(tomogram) -> int:
    plane = tomogram.rows * tomogram.cols * 4
    n = _HEADER.size
    for sl in tomogram.slices:
        n += _SLICE_HEADER.size + plane * (3 if sl.cost is not None else 2)
    return n


def archive_bytes(tomogram) -> np.ndarray:
    """The archive as a uint8 numpy array (page-locked when a GPU is used)."""
    total = archive_size(tomogram)
    rows, cols = tomogram.rows, tomogram.cols
    plane = rows * cols * 4
    layers = [l for sl in tomogram.slices for l in (sl.ground, sl.ceiling, sl.cost)
              if l is not None]
    on_dev = [l for l in layers if isinstance(l, Layer) and l._values is None and l._stack]
    ctx = on_dev[0]._stack.ctx if on_dev else None
    buf = _lib.pinned_pool(ctx).array((total,), np.uint8) if ctx else np.empty(total, np.uint8)
    ox, oy = tomogram.origin
    _HEADER.pack_into(buf, 0, _MAGIC, 1, rows, cols, np.float32(tomogram.resolution), float(ox),
                      float(oy), float(tomogram.z_min), np.float32(tomogram.d_s),
                      len(tomogram.slices))
    off = _HEADER.size
    base = buf.ctypes.data
    pending = False
    for sl in tomogram.slices:
        mask = MASK_GROUND | MASK_CEILING | (MASK_COST if sl.cost is not None else 0)
        _SLICE_HEADER.pack_into(buf, off, float(sl.plane_height), mask)
        off += _SLICE_HEADER.size
        for layer in (sl.ground, sl.ceiling, sl.cost):
            if layer is None:
                continue
            if layer.shape != (rows, cols):
                raise ValueError("slice layers have different shapes")
            if isinstance(layer, Layer) and layer._values is None and layer._stack is not None:
                st, k = layer._stack, layer._k
                st.ctx.check(st.ctx.lib.pct_memcpy_d2h_async(st.ctx.h, base + off, st.slice_ptr(k),
                                                             plane), "d2h")
                pending = True
            else:
                v = np.ascontiguousarray(layer.values, dtype="<f4")
                buf[off:off + plane] = v.view(np.uint8).reshape(-1)
            off += plane
    if pending:  # one synchronisation per context with copies in flight
        for c in {id(l._stack.ctx): l._stack.ctx for l in on_dev}.values():
            c.check(c.lib.pct_sync(c.h), "sync")
    assert off == total
    return buf


def save_tomogram(tomogram: Tomogram, path):
    """Serialize to the LGA format (tomogram.py:228-244), byte-identical."""
    buf = archive_bytes(tomogram)
    with open(path, "wb") as f:
        f.write(memoryview(buf))


def load_tomogram(path) -> Tomogram:
    """Parse an LGA archive (tomogram.py:247-276) into host-resident layers."""
    data = Path(path).read_bytes()
    if len(data) < _HEADER.size or data[:4] != _MAGIC:
        raise ValueError(f"{path}: not an LGA archive")
    magic, version, rows, cols, res, ox, oy, z_min, d_s, count = _HEADER.unpack_from(data, 0)
    if version != 1:
        raise ValueError(f"{path}: unsupported LGA version {version}")
    off = _HEADER.size
    plane = rows * cols * 4
    origin = (ox, oy)
    slices = []
    for k in range(count):
        if off + _SLICE_HEADER.size > len(data):
            raise ValueError(f"{path}: truncated archive")
        height, mask = _SLICE_HEADER.unpack_from(data, off)
        off += _SLICE_HEADER.size
        got = {}
        for bit, name in ((MASK_GROUND, "ground"), (MASK_CEILING, "ceiling"), (MASK_COST, "cost")):
            if mask & bit:
                if off + plane > len(data):
                    raise ValueError(f"{path}: truncated archive")
                arr = np.frombuffer(data, dtype="<f4", count=rows * cols, offset=off)
                got[name] = Layer(arr.reshape(rows, cols).copy(), float(res), origin)
                off += plane
        if "ground" not in got or "ceiling" not in got:
            raise ValueError(f"{path}: slice {k} is missing ground or ceiling layer")
        slices.append(TomogramSlice(got["ground"], got["ceiling"], float(height), k,
                                    got.get("cost")))
    if off != len(data):
        raise ValueError(f"{path}: {len(data) - off} trailing bytes")
    return Tomogram(slices=slices, d_s=float(d_s), z_min=float(z_min))
