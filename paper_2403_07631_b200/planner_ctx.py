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

    # --- the reference object's lookups (planner.py:95-129), host side
    def snap(self, point, tol: float):
        """Nearest traversable node for a query position, or None."""
        x, y, z = float(point[0]), float(point[1]), float(point[2])
        K, R, C = self.elev.shape
        i = math.floor((y - self.origin[1]) / self.res + 0.5)
        j = math.floor((x - self.origin[0]) / self.res + 0.5)
        if not (0 <= i < R and 0 <= j < C):
            return None
        best = None
        for k in range(K):
            if not self.valid[k, i, j]:
                continue
            dz = abs(float(self.elev[k, i, j]) - z)
            if dz > tol:
                continue
            key = (dz, float(self.cost[k, i, j]), k)
            if best is None or key < best[0]:
                best = (key, k)
        if best is None:
            return None
        k0 = int(self.canon[best[1], i, j])
        if not self.cn[k0, i, j] < self.c_barrier:
            return None
        return k0, i, j

    def member_with_min_cost(self, k0, i, j):
        K = self.elev.shape[0]
        best_k, best_c = k0, float(self.cost[k0, i, j])
        k = k0 + 1
        while k < K and self.canon[k, i, j] == k0:
            c = float(self.cost[k, i, j])
            if c < best_c:
                best_k, best_c = k, c
            k += 1
        return best_k


def attach_planner_context(tomogram, eps_e: float = 1e-6, c_barrier: float = 50.0):
    """Precompute the planner context on the GPU and cache it on the tomogram
    exactly where the reference planner looks for it."""
    ctx = PlannerContext(tomogram, eps_e, c_barrier)
    tomogram._planner_ctx = ctx
    return ctx
