"""Redundant-slice simplification on the GPU (drop-in for tomoplan/simplify.py).

The reference's forward sweep to a fixpoint (simplify.py:56-73) is replayed
exactly by libpct's host runtime (k_simplify.cu: run_simplify) from any()
reductions computed on the device; only the surviving slice indices come
back to the host.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .tomogram import Layer, Tomogram, TomogramSlice, device_run, upload_stack

DEFAULT_EPS_E = 1e-6


def _check_costs(slices):
    if slices[0].cost is None:
        raise ValueError("slice has no cost layer; evaluate the tomogram first")
    if any(s.cost is None for s in slices):
        raise ValueError("neighbor slice has no cost layer")


def _stack_ptr(ctx, layers, keep):
    src = device_run(layers)
    if src is not None and src[0].ctx is ctx:
        return src[0].slice_ptr(src[1])
    shape = layers[0].shape
    if any(l.shape != shape for l in layers):
        raise ValueError("slice layers have different shapes")
    st = upload_stack(ctx, [l.values for l in layers])
    keep.append(st)
    return st.ptr


def _change_info(slices):
    """The slice-change information of the slices' stacks (the build's
    ground masks, the evaluation's tile masks) when the slices are exactly
    the whole ground stack of one device build and the whole cost stack its
    evaluation wrote (values untouched on the host), else None."""
    g = device_run([s.ground for s in slices])
    c = device_run([s.cost for s in slices])
    if g is None or c is None or g[1] != 0 or c[1] != 0:
        return None
    info = c[0].change_info
    if info is None or info["ground"] is not g[0] or g[0].n_slices != len(slices) or \
            c[0].n_slices != len(slices) or c[0].ctx is not g[0].ctx:
        return None
    return info


def _ctx(slices):
    for s in slices:
        d = s.ground.device if isinstance(s.ground, Layer) else None
        if d is not None:
            return d[0].ctx
    return _lib.context()


def simplify_tomogram(tomogram: Tomogram, eps_e: float = DEFAULT_EPS_E,
                      c_barrier: float = 50.0) -> Tomogram:
    """Remove redundant slices; indices are reassigned, plane heights kept."""
    slices = list(tomogram.slices)
    if len(slices) > 1:
        _check_costs(slices)
        ctx = _ctx(slices)
        keepalive = []
        rows, cols = slices[0].ground.shape
        with ctx.lock:
            g = _stack_ptr(ctx, [s.ground for s in slices], keepalive)
            c = _stack_ptr(ctx, [s.cost for s in slices], keepalive)
            idx = np.empty(len(slices), np.int32)
            n = C.c_int32(0)
            info = _change_info(slices)
            if info is not None:  # whole stacks of one build + evaluation
                ctx.check(ctx.lib.pct_simplify_masked(
                    ctx.h, g, c, len(slices), rows, cols, float(eps_e), float(c_barrier),
                    info["masks"], info["tiles"].ptr, info["geom"].ctypes.data,
                    idx.ctypes.data, C.byref(n)), "pct_simplify")
            else:
                ctx.check(ctx.lib.pct_simplify(ctx.h, g, c, len(slices), rows, cols,
                                               float(eps_e), float(c_barrier), idx.ctypes.data,
                                               C.byref(n)), "pct_simplify")
        slices = [slices[i] for i in idx[:n.value]]
    out = [TomogramSlice(s.ground, s.ceiling, s.plane_height, i, s.cost)
           for i, s in enumerate(slices)]
    return Tomogram(slices=out, d_s=tomogram.d_s, z_min=tomogram.z_min)


def unique_cells(tomogram: Tomogram, k: int, eps_e: float = DEFAULT_EPS_E,
                 c_barrier: float = 50.0) -> set:
    """The (i, j) cells of slice k not covered by the adjacent slices."""
    slices = tomogram.slices
    if not 0 <= k < len(slices):
        raise IndexError(f"slice index {k} out of range")
    if slices[k].cost is None:
        raise ValueError("slice has no cost layer; evaluate the tomogram first")
    lo = k - 1 if k > 0 else -1
    hi = k + 1 if k + 1 < len(slices) else -1
    for nb in (lo, hi):
        if nb >= 0 and slices[nb].cost is None:
            raise ValueError("neighbor slice has no cost layer")
    idx = [i for i in (lo, k, hi) if i >= 0]
    sub = [slices[i] for i in idx]
    ctx = _ctx(sub)
    rows, cols = slices[k].ground.shape
    keepalive = []
    with ctx.lock:
        g = _stack_ptr(ctx, [s.ground for s in sub], keepalive)
        c = _stack_ptr(ctx, [s.cost for s in sub], keepalive)
        pos = {i: n for n, i in enumerate(idx)}
        mask = _lib.DeviceBuffer(ctx, rows * cols)
        ctx.check(ctx.lib.pct_unique_mask(ctx.h, g, c, rows, cols, pos[k],
                                          pos[lo] if lo >= 0 else -1,
                                          pos[hi] if hi >= 0 else -1, float(eps_e),
                                          float(c_barrier), mask.ptr), "pct_unique_mask")
        m = np.empty((rows, cols), np.uint8)
        mask.to_host(m)
    ii, jj = np.nonzero(m)
    return set(zip(ii.tolist(), jj.tolist()))
