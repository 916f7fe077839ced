"""Oracle: tomogram construction (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

Restates tomoplan/tomogram.py:127-213 with numpy.  The grid frame
(tomogram.py:134-145), float64 rasterisation (:147-150), stable z-order and
plane split with ties going to the ground group (:152-157), cumulative max
(ground, bottom-up) and cumulative min (ceiling, top-down) reductions
(:162-194) and NaN encoding of empty cells (:199-204) follow the reference
operation for operation, so the outputs are bit-identical to it.
"""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np

GRID_SIDE_LIMIT = 16384


def bounds(xyz):
    """Exact float64 (min, max) corners (cloud_io.py:47-50)."""
    a = np.asarray(xyz)
    return a.min(axis=0).astype(np.float64), a.max(axis=0).astype(np.float64)


def frame(lo, hi, d_s, r_g, max_grid_side=GRID_SIDE_LIMIT):
    """Grid frame of tomogram.py:134-145: origin, rows, cols, plane heights.

    Raises ValueError for non-positive d_s/r_g and OverflowError-free
    ValueError('grid ... exceeds') when a side is above ``max_grid_side``
    (the product raises the reference's GridSizeError subclass)."""
    if d_s <= 0 or r_g <= 0:
        raise ValueError("d_s and r_g must be positive")
    x_min, y_min, z_min = (float(v) for v in lo)
    x_max, y_max, z_max = (float(v) for v in hi)
    rows = math.floor((y_max - y_min) / r_g + 0.5) + 2
    cols = math.floor((x_max - x_min) / r_g + 0.5) + 2
    if rows > max_grid_side or cols > max_grid_side:
        raise ValueError(f"grid {rows}x{cols} exceeds the {max_grid_side} per-side limit")
    n = max(1, math.ceil((z_max - z_min) / d_s - 1e-9))
    heights = z_min + d_s * (np.arange(n, dtype=np.float64) + 1.0)
    return dict(origin=(x_min, y_min), rows=rows, cols=cols, heights=heights,
                z_min=z_min)


def rasterize_index(p, origin, r_g):
    """Nearest-cell-centre index (tomogram.py:99-112), without bounds check."""
    x, y = float(p[0]), float(p[1])
    return (math.floor((y - origin[1]) / r_g + 0.5),
            math.floor((x - origin[0]) / r_g + 0.5))


def _chunked(pool, fn, lo, hi, threads):
    """Apply fn(a, b) over `threads` contiguous pieces of [lo, hi)."""
    n = hi - lo
    pieces = [(lo + n * t // threads, lo + n * (t + 1) // threads) for t in range(threads)]
    pieces = [(a, b) for a, b in pieces if b > a]
    if pool is None or len(pieces) < 2:
        return [fn(a, b) for a, b in pieces]
    return [f.result() for f in [pool.submit(fn, a, b) for a, b in pieces]]


def build(xyz, d_s, r_g, max_grid_side=GRID_SIDE_LIMIT, threads=1):
    """Ground and ceiling stacks for the points ``xyz`` (any float dtype).

    Returns dict(ground, ceiling: (S, rows, cols) float32 with NaN for empty
    cells, heights: (S,) float64, origin, rows, cols, z_min).
    """
    pts = np.asarray(xyz, dtype=np.float64)
    lo, hi = bounds(pts)
    fr = frame(lo, hi, d_s, r_g, max_grid_side)
    rows, cols, heights = fr["rows"], fr["cols"], fr["heights"]
    x0, y0 = fr["origin"]
    n_cells = rows * cols
    S = heights.shape[0]

    # float64 rasterisation (tomogram.py:147-150)
    ii = np.floor((pts[:, 1] - y0) / r_g + 0.5).astype(np.int64)
    jj = np.floor((pts[:, 0] - x0) / r_g + 0.5).astype(np.int64)
    cell = ii * cols + jj

    # stable z order, float32 values, plane split with ties to ground (:152-157)
    perm = np.argsort(pts[:, 2], kind="stable")
    zs = pts[perm, 2]
    cell = cell[perm]
    z32 = zs.astype(np.float32)
    cut = np.searchsorted(zs, heights, side="right")
    bounds_k = np.concatenate([[0], cut, [len(zs)]])  # bin b = (bounds_k[b], bounds_k[b+1])

    threads = max(1, int(threads))
    pool = ThreadPoolExecutor(threads) if threads > 1 else None
    try:
        def sweep(order, ufunc, init):
            # one partial grid per worker; merged snapshot after each bin
            parts = [np.full(n_cells, init, np.float32) for _ in range(threads)]
            snaps = {}
            for b, k in order:
                a, e = int(bounds_k[b]), int(bounds_k[b + 1])
                pieces = _chunked(None, lambda p, q: (p, q), a, e, threads)
                if pool is not None and len(pieces) > 1:
                    futs = [pool.submit(ufunc.at, parts[t], cell[p:q], z32[p:q])
                            for t, (p, q) in enumerate(pieces)]
                    for f in futs:
                        f.result()
                else:
                    for t, (p, q) in enumerate(pieces):
                        ufunc.at(parts[t], cell[p:q], z32[p:q])
                if k is not None:
                    snap = parts[0].copy()
                    for t in range(1, threads):
                        ufunc(snap, parts[t], out=snap)
                    snaps[k] = snap
            return snaps

        # ground[k] = max over bins 0..k; ceiling[k] = min over bins k+1..S
        g = sweep([(b, b) for b in range(S)], np.maximum, np.float32(-np.inf))
        c = sweep([(b, b - 1) for b in range(S, 0, -1)], np.minimum, np.float32(np.inf))
    finally:
        if pool is not None:
            pool.shutdown()

    ground = np.empty((S, rows, cols), np.float32)
    ceiling = np.empty((S, rows, cols), np.float32)
    nan = np.float32(np.nan)
    for k in range(S):
        ground[k] = np.where(np.isfinite(g[k]), g[k], nan).reshape(rows, cols)
        ceiling[k] = np.where(np.isfinite(c[k]), c[k], nan).reshape(rows, cols)
    return dict(ground=ground, ceiling=ceiling, heights=heights, origin=fr["origin"],
                rows=rows, cols=cols, z_min=fr["z_min"], d_s=float(d_s), r_g=float(r_g))
