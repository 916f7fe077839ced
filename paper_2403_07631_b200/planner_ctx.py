"""Planner context precompute on the GPU (SURVEY.md §8 f rank 2).

The reference's A* (planner.py, stays on the CPU) first derives dense
canonical-node arrays from the evaluated tomogram (_PlannerContext,
planner.py:62-129): a run merge of equal ground across adjacent slices and
the run-minimum node cost.  ``PlannerContext`` computes them with one
device kernel (pct_planner_context) and exposes the reference object's
attributes and lookups; ``attach_planner_context`` stores it where the
reference planner looks for its cache (``tomogram._planner_ctx``,
planner.py:132-137), so ``tomoplan.plan_path`` runs unchanged on it.
"""

from __future__ import annotations

import math

import numpy as np

from . import _lib
from .tomogram import Layer, device_run, upload_stack


class PlannerContext:
    def __init__(self, tomogram, eps_e: float = 1e-6, c_barrier: float = 50.0):
        self.tomogram = tomogram
        self.eps_e = float(eps_e)
        self.c_barrier = float(c_barrier)
        self.res = float(tomogram.resolution)
        self.origin = tomogram.origin
        slices = tomogram.slices
        if any(s.cost is None for s in slices):
            raise ValueError("tomogram has no cost layers; run evaluate_tomogram first")
        S = len(slices)
        rows, cols = slices[0].ground.shape
        ctx = None
        for s in slices:
            d = s.ground.device if isinstance(s.ground, Layer) else None
            if d is not None:
                ctx = d[0].ctx
                break
        ctx = ctx or _lib.context()
        keep = []
        with ctx.lock:
            gptr = self._stack_ptr(ctx, [s.ground for s in slices], keep)
            cptr = self._stack_ptr(ctx, [s.cost for s in slices], keep)
            canon = _lib.DeviceBuffer(ctx, S * rows * cols * 4)
            cn = _lib.DeviceBuffer(ctx, S * rows * cols * 4)
            ctx.check(ctx.lib.pct_planner_context(ctx.h, gptr, cptr, S, rows, cols, self.eps_e,
                                                  canon.ptr, cn.ptr), "planner_context")
            self.canon = np.empty((S, rows, cols), np.int32)
            self.cn = np.empty((S, rows, cols), np.float32)
            canon.to_host(self.canon)
            cn.to_host(self.cn)
        self.elev = tomogram.ground_stack()
        self.cost = tomogram.cost_stack()
        self.valid = np.isfinite(self.elev)

    @staticmethod
    def _stack_ptr(ctx, layers, keep):
        src = device_run(layers)
        if src is not None and src[0].ctx is ctx:
            return src[0].slice_ptr(src[1])
        st = upload_stack(ctx, [l.values for l in layers])
        keep.append(st)
        return st.ptr

    # --- the reference object's two lookups (planner.py:95-129), answered
    # from one column of the (K, rows, cols) arrays with vectorised numpy
    def _cell(self, point):
        """Grid cell of a query position (tomogram.rasterize_index rule), or None."""
        K, nr, nc = self.elev.shape
        col = math.floor((float(point[0]) - self.origin[0]) / self.res + 0.5)
        row = math.floor((float(point[1]) - self.origin[1]) / self.res + 0.5)
        return (row, col) if 0 <= row < nr and 0 <= col < nc else None

    def snap(self, point, tol: float):
        """(k0, i, j) of the traversable canonical node nearest a query
        position, or None.  Candidates are the valid slices of the query's
        cell within ``tol`` vertically; the winner is the smallest
        (|dz|, cost, k) triple; it must belong to a node whose run cost is
        below the barrier."""
        cell = self._cell(point)
        if cell is None:
            return None
        i, j = cell
        dz = np.abs(self.elev[:, i, j].astype(np.float64) - float(point[2]))
        ok = np.flatnonzero(self.valid[:, i, j] & (dz <= tol))
        if ok.size == 0:
            return None
        # lexsort: last key is primary -> (dz, cost, k) ascending, first wins
        order = np.lexsort((ok, self.cost[ok, i, j].astype(np.float64), dz[ok]))
        k0 = int(self.canon[ok[order[0]], i, j])
        return (k0, i, j) if self.cn[k0, i, j] < self.c_barrier else None

    def member_with_min_cost(self, k0, i, j):
        """The slice of node (k0, i, j)'s run with the lowest cost (the first
        one on ties): the run is k0 and the slices above it whose canonical
        index is k0."""
        above = self.canon[k0 + 1:, i, j] != k0
        run = int(np.argmax(above)) if above.any() else above.size
        return k0 + int(np.argmin(self.cost[k0:k0 + 1 + run, i, j]))


def attach_planner_context(tomogram, eps_e: float = 1e-6, c_barrier: float = 50.0):
    """Precompute the planner context on the GPU and cache it on the tomogram
    exactly where the reference planner looks for it."""
    ctx = PlannerContext(tomogram, eps_e, c_barrier)
    tomogram._planner_ctx = ctx
    return ctx
