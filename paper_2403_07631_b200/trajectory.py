"""Ceiling inflation for the trajectory optimiser on the GPU (SURVEY.md §8 f
rank 4).

The reference's ``_Problem.__init__`` (trajectory.py:366-374) calls
``_inflate_ceiling`` (trajectory.py:277-317) for every slice a path touches,
on every optimisation: a float64 min-filter over the robot radius and up to
60 Jacobi sweeps of a chamfer descent skirt, in numpy.  Here the same two
arrays come out of ``pct_ceiling_inflate`` bit for bit — one call for a single
layer (drop-in, host arrays in and out) or for every slice of a tomogram at
once (:func:`inflate_ceilings`, reading the ceiling stack where it already
lives in HBM), so the optimiser can take them as a precomputed input.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .tomogram import Layer, device_run, upload_stack

CEILING_EROSION = 0.20      # OptConfig.ceiling_erosion (trajectory.py:71)
CEILING_SKIRT_SLOPE = 0.30  # OptConfig.ceiling_skirt_slope (trajectory.py:72)


def _run(ctx, ceil_ptr, S, rows, cols, res, erosion, skirt_slope):
    n = S * rows * cols
    flat = _lib.DeviceBuffer(ctx, n * 8)
    skirt = _lib.DeviceBuffer(ctx, n * 8)
    ctx.check(ctx.lib.pct_ceiling_inflate(ctx.h, ceil_ptr, int(S), int(rows), int(cols),
                                          float(res), float(erosion), float(skirt_slope),
                                          flat.ptr, skirt.ptr), "pct_ceiling_inflate")
    out_f = np.empty((S, rows, cols), np.float64)
    out_s = np.empty((S, rows, cols), np.float64)
    flat.to_host(out_f)
    skirt.to_host(out_s)
    return out_f, out_s


def inflate_ceiling(values: np.ndarray, valid: np.ndarray, res: float, erosion: float,
                    skirt_slope: float, *, device=None):
    """Drop-in for ``trajectory._inflate_ceiling``: (flat, skirted) float64
    arrays for one ceiling layer; cells with no ceiling stay +inf."""
    v = np.asarray(values, dtype=np.float32)
    ok = np.asarray(valid, dtype=bool)
    if v.ndim != 2 or ok.shape != v.shape:
        raise ValueError("ceiling values and valid mask must be matching 2-D arrays")
    if not np.array_equal(ok, np.isfinite(v)):
        v = np.where(ok, v, np.float32(np.nan))
    ctx = _lib.context(device)
    rows, cols = v.shape
    with ctx.lock:
        st = upload_stack(ctx, [v])
        f, s = _run(ctx, st.ptr, 1, rows, cols, res, erosion, skirt_slope)
    return f[0], s[0]


def inflate_ceilings(tomogram, erosion: float = CEILING_EROSION,
                     skirt_slope: float = CEILING_SKIRT_SLOPE, *, device=None):
    """(flat, skirted) float64 stacks (S, rows, cols) for every slice of
    ``tomogram`` — the per-slice results of ``_inflate_ceiling`` with the
    tomogram's resolution, computed in one device call."""
    slices = tomogram.slices
    layers = [s.ceiling for s in slices]
    rows, cols = layers[0].shape
    src = device_run(layers)
    ctx = src[0].ctx if src is not None else _lib.context(device)
    with ctx.lock:
        if src is not None:
            ptr, keep = src[0].slice_ptr(src[1]), None
        else:
            keep = upload_stack(ctx, [l.values if isinstance(l, Layer) else np.asarray(l.values)
                                      for l in layers])
            ptr = keep.ptr
        return _run(ctx, ptr, len(layers), rows, cols, float(tomogram.resolution), erosion,
                    skirt_slope)
