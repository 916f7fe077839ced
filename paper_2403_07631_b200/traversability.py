"""Traversability evaluation on the GPU (drop-in for tomoplan/traversability.py).

``evaluate_tomogram`` runs the fused sm_100a stencil (k_evaluate.cu) over all
slices in one launch; the per-operation functions (interval_cost,
ground_cost, fuse_costs, inflate, ...) keep the reference signatures and
also run on the device.  Parameter objects and the inflation kernel weights
are host-side setup, computed exactly as the reference does
(traversability.py:21-56, 173-202).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, replace

import numpy as np

from . import _lib
from .tomogram import (DeviceTomogram, Layer, Tomogram, TomogramSlice, device_run,
                       new_device_stack, upload_stack)


@dataclass(frozen=True)
class TravParams:
    """Thresholds and weights of the traversability model (Table-defaults)."""

    d_min: float = 0.50
    d_ref: float = 0.65
    theta_b: float = 1.70
    theta_s: float = 0.36
    theta_p: float = 0.20
    c_barrier: float = 50.0
    alpha_d: float = 20.0
    alpha_b: float = 20.0
    alpha_s: float = 15.0
    d_inf: float = 0.20
    d_sm: float = 0.40
    r_c: float = 0.20
    step_patch_radius: int | None = None

    def __post_init__(self):
        if not (0 < self.d_min <= self.d_ref):
            raise ValueError("need 0 < d_min <= d_ref")
        if not (0 < self.theta_s <= self.theta_b):
            raise ValueError("need 0 < theta_s <= theta_b")
        if not (0 <= self.theta_p <= 1):
            raise ValueError("theta_p must lie in [0, 1]")
        if self.c_barrier <= 0:
            raise ValueError("c_barrier must be positive")
        if not (self.d_inf < self.d_sm):
            raise ValueError("need d_inf < d_sm")
        if self.d_inf < self.r_c:
            raise ValueError("inflation radius must cover the collision radius")

    def patch_radius(self, r_g: float) -> int:
        if self.step_patch_radius is not None:
            return int(self.step_patch_radius)
        return int(math.ceil(0.3 / r_g))


@dataclass
class InflationKernel:
    """Radially decaying weights; side = 2*ceil(d_sm/r_g) + 1, float32."""

    weights: np.ndarray
    resolution: float

    @property
    def radius_cells(self) -> int:
        return self.weights.shape[0] // 2

    def weight_classes(self):
        """Distinct positive weights with their cell footprints, largest first."""
        out = []
        for w in np.unique(self.weights)[::-1]:
            if w > 0:
                out.append((np.float32(w), self.weights == w))
        return out


def build_kernel(d_inf: float, d_sm: float, r_g: float) -> InflationKernel:
    """Inflation kernel weights (traversability.py:194-202): 1 inside d_inf,
    then linear falloff; float64 math rounded once to float32."""
    if not (r_g <= d_inf < d_sm):
        raise ValueError("need r_g <= d_inf < d_sm")
    radius = int(math.ceil(d_sm / r_g))
    offs = np.arange(-radius, radius + 1, dtype=np.float64) * r_g
    dist = np.hypot(offs[:, None], offs[None, :])
    w = np.maximum(0.0, np.minimum(1.0 - (dist - d_inf) / (d_sm - r_g), 1.0))
    return InflationKernel(w.astype(np.float32), float(r_g))


# ---------------------------------------------------------------------------
# helpers

def _ctx_for(layers):
    for l in layers:
        d = l.device if isinstance(l, Layer) else None
        if d is not None:
            return d[0].ctx
    return _lib.context()


def _kernel_arg(kernel):
    w = np.ascontiguousarray(np.asarray(kernel.weights, np.float32))
    if w.ndim != 2 or w.shape[0] != w.shape[1] or w.shape[0] % 2 != 1:
        raise ValueError("inflation kernel must be square with an odd side")
    return w


def _layer_values_dev(ctx, layer):
    """(device pointer, keepalive) of one layer's values."""
    d = layer.device if isinstance(layer, Layer) else None
    if d is not None and d[0].ctx is ctx:
        return d[0].slice_ptr(d[1]), d[0]
    vals = layer.values if hasattr(layer, "values") else np.asarray(layer, np.float32)
    buf = _lib.DeviceBuffer.from_host(ctx, np.asarray(vals, np.float32))
    return buf.ptr, buf


def _download(buf, shape, dtype):
    out = np.empty(shape, dtype)
    buf.to_host(out)
    return out


# ---------------------------------------------------------------------------
# per-operation API (traversability.py:59-213)

def interval_cost(ground, ceiling, params) -> np.ndarray:
    """Clearance cost per cell. Open sky costs 0; missing ground is a barrier."""
    if ground.shape != ceiling.shape:
        raise ValueError("ground and ceiling layers are misaligned")
    ctx = _ctx_for([ground, ceiling])
    rows, cols = ground.shape
    with ctx.lock:
        g, kg = _layer_values_dev(ctx, ground)
        c, kc = _layer_values_dev(ctx, ceiling)
        out = _lib.DeviceBuffer(ctx, rows * cols * 4)
        ctx.check(ctx.lib.pct_interval_cost(ctx.h, g, c, rows, cols,
                                            C.byref(_lib.trav_params_c(params, 1.0)), out.ptr),
                  "interval_cost")
        return _download(out, (rows, cols), np.float32)


def slope_magnitudes(ground):
    """Return (m_xy, m_grad, isolated) for the valid cells of a ground layer."""
    ctx = _ctx_for([ground])
    rows, cols = ground.shape
    n = rows * cols
    with ctx.lock:
        g, kg = _layer_values_dev(ctx, ground)
        mx = _lib.DeviceBuffer(ctx, n * 8)
        mg = _lib.DeviceBuffer(ctx, n * 8)
        iso = _lib.DeviceBuffer(ctx, n)
        ctx.check(ctx.lib.pct_slope_magnitudes(ctx.h, g, rows, cols, float(ground.resolution),
                                               mx.ptr, mg.ptr, iso.ptr), "slope_magnitudes")
        return (_download(mx, (rows, cols), np.float64), _download(mg, (rows, cols), np.float64),
                _download(iso, (rows, cols), np.uint8).astype(bool))


def gentle_fraction(gentle: np.ndarray, radius: int) -> np.ndarray:
    """Fraction of gentle cells in the (2r+1)^2 window; outside counts as not gentle."""
    ctx = _lib.context()
    m = np.ascontiguousarray(np.asarray(gentle, dtype=bool).astype(np.uint8))
    rows, cols = m.shape
    with ctx.lock:
        gb = _lib.DeviceBuffer.from_host(ctx, m)
        out = _lib.DeviceBuffer(ctx, rows * cols * 8)
        ctx.check(ctx.lib.pct_gentle_fraction(ctx.h, gb.ptr, rows, cols, int(radius), out.ptr),
                  "gentle_fraction")
        return _download(out, (rows, cols), np.float64)


def terrain_cost_values(m_xy, m_grad, p_s, params) -> np.ndarray:
    """Branch logic of the slope cost; inputs may be scalars or arrays."""
    a, b, c = np.broadcast_arrays(np.asarray(m_xy, np.float64), np.asarray(m_grad, np.float64),
                                  np.asarray(p_s, np.float64))
    shape = a.shape
    a, b, c = (np.ascontiguousarray(v).reshape(-1) for v in (a, b, c))
    ctx = _lib.context()
    with ctx.lock:
        da, db, dc = (_lib.DeviceBuffer.from_host(ctx, v) for v in (a, b, c))
        out = _lib.DeviceBuffer(ctx, max(a.size, 1) * 8)
        ctx.check(ctx.lib.pct_terrain_cost_values(ctx.h, da.ptr, db.ptr, dc.ptr, a.size,
                                                  C.byref(_lib.trav_params_c(params, 1.0)),
                                                  out.ptr), "terrain_cost_values")
        return _download(out, (a.size,), np.float64).reshape(shape)


def ground_cost(ground, params) -> np.ndarray:
    """Terrain condition cost from the ground layer gradients."""
    ctx = _ctx_for([ground])
    rows, cols = ground.shape
    r_g = float(ground.resolution)
    with ctx.lock:
        g, kg = _layer_values_dev(ctx, ground)
        out = _lib.DeviceBuffer(ctx, rows * cols * 4)
        ctx.check(ctx.lib.pct_ground_cost(ctx.h, g, rows, cols, r_g,
                                          C.byref(_lib.trav_params_c(params, r_g)), out.ptr),
                  "ground_cost")
        return _download(out, (rows, cols), np.float32)


def fuse_costs(c_interval, c_ground, ground_valid, params) -> np.ndarray:
    """Clipped sum of the two cost sources; invalid ground stays a barrier."""
    ci = np.ascontiguousarray(np.asarray(c_interval, np.float32))
    cg = np.ascontiguousarray(np.asarray(c_ground, np.float32))
    gv = np.ascontiguousarray(np.asarray(ground_valid, bool).astype(np.uint8))
    ci, cg, gv = np.broadcast_arrays(ci, cg, gv)
    shape = ci.shape
    ci, cg, gv = (np.ascontiguousarray(v).reshape(-1) for v in (ci, cg, gv))
    ctx = _lib.context()
    with ctx.lock:
        d1, d2, d3 = (_lib.DeviceBuffer.from_host(ctx, v) for v in (ci, cg, gv))
        out = _lib.DeviceBuffer(ctx, max(ci.size, 1) * 4)
        ctx.check(ctx.lib.pct_fuse_costs(ctx.h, d1.ptr, d2.ptr, d3.ptr, 1, ci.size,
                                         C.byref(_lib.trav_params_c(params, 1.0)), out.ptr),
                  "fuse_costs")
        return _download(out, (ci.size,), np.float32).reshape(shape)


def inflate(cost: np.ndarray, kernel: InflationKernel) -> np.ndarray:
    """Sliding-window weighted maximum; cells outside the map contribute nothing."""
    c = np.ascontiguousarray(np.asarray(cost, dtype=np.float32))
    w = _kernel_arg(kernel)
    rows, cols = c.shape
    ctx = _lib.context()
    with ctx.lock:
        din = _lib.DeviceBuffer.from_host(ctx, c)
        out = _lib.DeviceBuffer(ctx, max(c.size, 1) * 4)
        ctx.check(ctx.lib.pct_inflate(ctx.h, din.ptr, rows, cols, w.ctypes.data, w.shape[0],
                                      out.ptr), "inflate")
        return _download(out, (rows, cols), np.float32)


# ---------------------------------------------------------------------------
# whole-slice / whole-tomogram evaluation (traversability.py:216-236)

def _evaluate_layers(ctx, grounds, ceilings, r_g, params, w):
    """Cost DeviceStack for lists of ground/ceiling layers (same shape)."""
    rows, cols = grounds[0].shape
    for g, c in zip(grounds, ceilings):
        if g.shape != (rows, cols) or c.shape != (rows, cols):
            raise ValueError("ground and ceiling layers are misaligned")
    S = len(grounds)
    gsrc = device_run(grounds)
    csrc = device_run(ceilings)
    keep = []
    if gsrc is not None and gsrc[0].ctx is ctx:
        gptr = gsrc[0].slice_ptr(gsrc[1])
    else:
        st = upload_stack(ctx, [g.values for g in grounds])
        keep.append(st)
        gptr = st.ptr
    if csrc is not None and csrc[0].ctx is ctx:
        cptr = csrc[0].slice_ptr(csrc[1])
    else:
        st = upload_stack(ctx, [c.values for c in ceilings])
        keep.append(st)
        cptr = st.ptr
    out = new_device_stack(ctx, S, rows, cols)
    # the whole stacks of one device build: its slice-change masks spare the
    # walk a pass over ground + ceiling
    masks = None
    if gsrc is not None and csrc is not None and gsrc[1] == 0 and csrc[1] == 0 and \
            gsrc[0].owner is csrc[0].owner and gsrc[0].n_slices == S and \
            isinstance(gsrc[0].owner, DeviceTomogram) and gsrc[0].ctx is ctx:
        masks = ctx.lib.pct_tomo_masks(gsrc[0].owner.handle)
    if masks:
        # per evaluation tile, the slices whose costs may change: with the
        # build's masks the simplify window then reads only where values
        # change (simplify_tomogram -> pct_simplify_masked)
        tm = _lib.DeviceBuffer(ctx, int(ctx.lib.pct_tile_masks_bytes(rows, cols)))
        geom = np.zeros(2, np.int32)
        ctx.check(ctx.lib.pct_evaluate_tiles(ctx.h, gptr, cptr, S, rows, cols, float(r_g),
                                             C.byref(_lib.trav_params_c(params, r_g)),
                                             w.ctypes.data, w.shape[0], masks, out.ptr, tm.ptr,
                                             geom.ctypes.data), "pct_evaluate")
        if geom[0] > 0:
            # (the ground stack's owner keeps its masks alive as long as this does)
            out.change_info = {"ground": gsrc[0], "masks": masks, "tiles": tm, "geom": geom}
    else:
        ctx.check(ctx.lib.pct_evaluate_masked(ctx.h, gptr, cptr, S, rows, cols, float(r_g),
                                              C.byref(_lib.trav_params_c(params, r_g)),
                                              w.ctypes.data, w.shape[0], masks, out.ptr),
                  "pct_evaluate")
    return out


def evaluate_slice(sl: TomogramSlice, params, kernel: InflationKernel | None = None):
    if kernel is None:
        kernel = build_kernel(params.d_inf, params.d_sm, sl.ground.resolution)
    w = _kernel_arg(kernel)
    ctx = _ctx_for([sl.ground, sl.ceiling])
    with ctx.lock:
        st = _evaluate_layers(ctx, [sl.ground], [sl.ceiling], float(sl.ground.resolution),
                              params, w)
    return replace(sl, cost=Layer.on_device(st, 0, sl.ground.resolution, sl.ground.origin))


def evaluate_tomogram(tomogram: Tomogram, params, threads: int = 1) -> Tomogram:
    """Fill every slice's cost layer (one fused launch over all slices).

    Drop-in for traversability.py:227-236; ``threads`` is ignored."""
    kernel = build_kernel(params.d_inf, params.d_sm, tomogram.resolution)
    w = _kernel_arg(kernel)
    slices = list(tomogram.slices)
    if not slices:
        return Tomogram(slices=[], d_s=tomogram.d_s, z_min=tomogram.z_min)
    ctx = _ctx_for([slices[0].ground])
    # gradients use each slice's own resolution: one launch per run of equal r_g
    out = [None] * len(slices)
    with ctx.lock:
        start = 0
        while start < len(slices):
            r_g = slices[start].ground.resolution
            end = start + 1
            while end < len(slices) and slices[end].ground.resolution == r_g:
                end += 1
            part = slices[start:end]
            st = _evaluate_layers(ctx, [s.ground for s in part], [s.ceiling for s in part],
                                  float(r_g), params, w)
            for n, s in enumerate(part):
                out[start + n] = replace(s, cost=Layer.on_device(st, n, s.ground.resolution,
                                                                 s.ground.origin))
            start = end
    return Tomogram(slices=out, d_s=tomogram.d_s, z_min=tomogram.z_min)
