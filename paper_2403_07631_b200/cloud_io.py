"""Point-cloud file ingest onto the GPU (SURVEY.md §8 f rank 3).

Drop-in for ``tomoplan.cloud_io.load_cloud`` / ``sniff_format``
(cloud_io.py:281-310).  ``pcd_binary`` — the format large maps are stored in —
is read by the native loader (``pct_pcd_load``): the payload goes from the
file into pinned chunks and straight to HBM, where the float32 x/y/z of every
record are gathered and the finite rows compacted in order
(cloud_io.py:123-146 + _keep_finite :53-55).  The result is a
:class:`DeviceCloud`, a ``PointCloud`` whose points stay in HBM;
``build_tomogram`` consumes it in place.  ``.points`` copies the float32
points to the host on first access, ``.xyz`` is their float64 copy (the
reference's type; float32 -> float64 is exact).

Header parsing and validation happen here on the host with the reference's
error types and messages (cloud_io.py:92-141).  The text formats (PCD ascii,
PLY ascii, xyz text) are not on the hot path and are not parsed here:
``load_cloud`` raises ``CloudFormatError`` for them.  ``compat.install``
routes them to the reference's own parsers when it patches ``tomoplan``.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from . import _lib
from .cloud import CloudFormatError, PointCloud

FORMATS = ("pcd_ascii", "pcd_binary", "ply_ascii", "xyz_text")

_PCD_KINDS = {"F": "f", "I": "i", "U": "u"}


def read_pcd_header(fh) -> dict:
    """Header lines up to and including DATA (cloud_io.py:92-104): upper-cased
    keyword -> list of value tokens; blank and '#' lines are skipped."""
    header = {}
    while True:
        raw = fh.readline()
        if not raw:
            raise CloudFormatError("PCD header ended before DATA line")
        text = raw.decode("ascii", errors="replace").strip()
        if not text or text.startswith("#"):
            continue
        tokens = text.split()
        keyword = tokens[0].upper()
        header[keyword] = tokens[1:]
        if keyword == "DATA":
            return header


def pcd_record_dtype(header: dict):
    """(names, sizes, kinds, counts, point count, DATA kind) of a PCD header, with the
    reference's validation order and messages (cloud_io.py:107-141)."""
    try:
        names = [f.lower() for f in header["FIELDS"]]
        sizes = [int(s) for s in header["SIZE"]]
        kinds = [t.upper() for t in header["TYPE"]]
        counts = [int(c) for c in header.get("COUNT", ["1"] * len(names))]
        n_points = int(header["POINTS"][0])
        data = header["DATA"][0].lower()
    except (KeyError, IndexError, ValueError) as exc:
        raise CloudFormatError(f"malformed PCD header: {exc}") from exc
    for axis in ("x", "y", "z"):
        if axis not in names:
            raise CloudFormatError(f"PCD file missing field '{axis}'")
    return names, sizes, kinds, counts, n_points, data


def _binary_layout(names, sizes, kinds, counts) -> np.dtype:
    spec = []
    for name, size, kind, count in zip(names, sizes, kinds, counts):
        if kind not in _PCD_KINDS:
            raise CloudFormatError(f"unsupported PCD TYPE '{kind}'")
        base = f"<{_PCD_KINDS[kind]}{size}"
        spec.append((name, base, (count,)) if count > 1 else (name, base))
    dtype = np.dtype(spec)
    for axis in ("x", "y", "z"):
        if dtype[axis] != np.dtype("<f4"):
            raise CloudFormatError("binary PCD x/y/z must be little-endian float32")
    return dtype


class DeviceCloud(PointCloud):
    """A ``PointCloud`` whose (N, 3) float32 points live in HBM.

    ``len``, ``dropped`` and ``bounds`` (computed on the device) need no host
    copy; ``points`` downloads the float32 points once, ``xyz`` is their
    float64 copy (as the reference stores it)."""

    def __init__(self, ctx, buf, n: int, dropped: int):  # noqa: D107 (no validation pass)
        self._ctx, self._buf, self._n = ctx, buf, int(n)
        self.dropped = int(dropped)
        self._host = None
        self._xyz64 = None
        self._bounds = None

    @property
    def points(self) -> np.ndarray:
        if self._host is None:
            out = np.empty((self._n, 3), np.float32)
            self._buf.to_host(out)
            self._host = out
        return self._host

    def __len__(self):
        return self._n

    def __repr__(self):
        return f"DeviceCloud(n={self._n}, dropped={self.dropped}, device={self._ctx.device})"

    @property
    def bounds(self):
        if self._bounds is None:
            from .tomogram import bounds_on_device
            self._bounds = bounds_on_device(self._ctx, self._buf.ptr, self._n, np.float32)
        return self._bounds

    def device_points(self):
        """(device pointer, N, dtype, device id) of the HBM-resident points."""
        return self._buf.ptr, self._n, np.float32, self._ctx.device


def _ingest(ctx, n_records: int, offsets, call, what: str) -> DeviceCloud:
    buf = _lib.DeviceBuffer(ctx, max(1, n_records) * 12)
    offs = (C.c_int64 * 3)(*offsets)
    n_valid = C.c_int64(0)
    with ctx.lock:
        rc = call(offs, buf.ptr, C.byref(n_valid))
        if rc == _lib.PCT_E_IO:
            raise CloudFormatError(ctx.error())
        ctx.check(rc, "PCD ingest")
    if n_valid.value == 0:
        raise CloudFormatError(f"{what}zero valid points")
    return DeviceCloud(ctx, buf, n_valid.value, n_records - n_valid.value)


def load_pcd_binary(path, *, device=None, chunk_bytes: int = 0) -> DeviceCloud:
    """Binary PCD -> HBM-resident cloud (cloud_io.py:123-146, binary branch)."""
    path = Path(path)
    with path.open("rb") as fh:
        header = read_pcd_header(fh)
        names, sizes, kinds, counts, n_points, data = pcd_record_dtype(header)
        if data != "binary":
            raise CloudFormatError(f"{path}: header DATA is '{data}', expected binary")
        dtype = _binary_layout(names, sizes, kinds, counts)
        data_offset = fh.tell()
        size = os.fstat(fh.fileno()).st_size
    n_points = max(n_points, 0)
    if size - data_offset < dtype.itemsize * n_points:
        raise CloudFormatError(f"{path}: truncated binary payload")
    ctx = _lib.context(device)
    offsets = [dtype.fields[a][1] for a in ("x", "y", "z")]
    return _ingest(ctx, n_points, offsets,
                   lambda offs, out, nv: ctx.lib.pct_pcd_load(
                       ctx.h, os.fsencode(str(path)), int(data_offset), int(n_points),
                       int(dtype.itemsize), offs, int(chunk_bytes), out, nv),
                   f"{path}: ")


def pcd_records_to_device(records: np.ndarray, *, device=None) -> DeviceCloud:
    """Records already in memory (a numpy structured array with float32 x, y,
    z fields, e.g. from a network stream) -> HBM-resident cloud."""
    rec = np.ascontiguousarray(records)
    dt = rec.dtype
    if dt.fields is None or any(a not in dt.fields for a in ("x", "y", "z")):
        raise ValueError("records need x, y and z fields")
    for a in ("x", "y", "z"):
        if dt[a] != np.dtype("<f4"):
            raise CloudFormatError("binary PCD x/y/z must be little-endian float32")
    ctx = _lib.context(device)
    n = rec.shape[0]
    offsets = [dt.fields[a][1] for a in ("x", "y", "z")]
    return _ingest(ctx, n, offsets,
                   lambda offs, out, nv: ctx.lib.pct_pcd_extract(
                       ctx.h, rec.ctypes.data, int(n), int(dt.itemsize), offs, 1, out, nv), "")


def load_cloud(path, fmt: str, *, device=None) -> PointCloud:
    """Read a point cloud (cloud_io.py:281-288); non-finite rows are dropped
    into ``cloud.dropped``.  Only ``pcd_binary`` (the format large maps are
    stored in) is read here, by the device ingest; the text formats are
    file IO before the hot path and raise ``CloudFormatError``."""
    if fmt not in FORMATS:
        raise ValueError(f"unknown format '{fmt}', expected one of {FORMATS}")
    path = Path(path)
    if not path.is_file():
        raise CloudFormatError(f"{path}: no such file")
    if fmt != "pcd_binary":
        raise CloudFormatError(f"{path}: format '{fmt}' has no device ingest; only pcd_binary "
                               "is read by this package")
    return load_pcd_binary(path, device=device)


def sniff_format(path) -> str:
    """Format from the extension and, for .pcd, the DATA line (cloud_io.py:298-310)."""
    path = Path(path)
    ext = path.suffix.lower()
    if ext == ".pcd":
        if not path.is_file():
            return "pcd_binary"
        with path.open("rb") as fh:
            header = read_pcd_header(fh)
        return "pcd_binary" if header["DATA"][0].lower() == "binary" else "pcd_ascii"
    if ext == ".ply":
        return "ply_ascii"
    return "xyz_text"
