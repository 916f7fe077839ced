"""Oracle: traversability evaluation (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

numpy restatement of tomoplan/traversability.py:59-236.  Every formula keeps
the reference's float64 operation order and its final float32 rounding:

  interval_cost        traversability.py:59-73
  _axis_gradient       traversability.py:76-103   (central / one-sided / zero)
  slope_magnitudes     traversability.py:106-114  (np.hypot = glibc hypot)
  gentle_fraction      traversability.py:117-128  (fixed (2r+1)^2 divisor)
  terrain_cost_values  traversability.py:131-147
  ground_cost          traversability.py:150-159
  fuse_costs           traversability.py:162-170
  kernel_weights       traversability.py:194-202  (build_kernel)
  inflate              traversability.py:205-213  (per weight class max filter)
  evaluate             traversability.py:216-236

``params`` is any object with the TravParams attribute names.
"""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np
from scipy import ndimage


def patch_radius(params, r_g):
    r = getattr(params, "step_patch_radius", None)
    return int(r) if r is not None else int(math.ceil(0.3 / r_g))


def interval_cost(g, c, params):
    gv = np.isfinite(g)
    cv = np.isfinite(c)
    gap = np.where(gv & cv, c.astype(np.float64) - g.astype(np.float64), np.inf)
    ramp = np.maximum(0.0, params.alpha_d * (params.d_ref - gap))
    out = np.where(gap < params.d_min, params.c_barrier, ramp)
    out = np.where(cv, out, 0.0)
    out = np.where(gv, out, params.c_barrier)
    return out.astype(np.float32)


def _shift(a, axis, step, fill):
    """out[i] = a[i + step] along axis (fill outside)."""
    out = np.full_like(a, fill)
    n = a.shape[axis]
    src = [slice(None)] * a.ndim
    dst = [slice(None)] * a.ndim
    if step > 0:
        src[axis], dst[axis] = slice(step, n), slice(0, n - step)
    else:
        src[axis], dst[axis] = slice(0, n + step), slice(-step, n)
    out[tuple(dst)] = a[tuple(src)]
    return out


def _gradient(e, valid, r_g, axis):
    e64 = np.where(valid, e.astype(np.float64), 0.0)
    nxt, prv = _shift(e64, axis, 1, 0.0), _shift(e64, axis, -1, 0.0)
    vn, vp = _shift(valid, axis, 1, False), _shift(valid, axis, -1, False)
    g = np.zeros_like(e64)
    g = np.where(vn & vp, (nxt - prv) / (2.0 * r_g), g)
    g = np.where(vn & ~vp, (nxt - e64) / r_g, g)
    g = np.where(vp & ~vn, (e64 - prv) / r_g, g)
    return g, vn | vp


def slope_magnitudes(e, r_g):
    valid = np.isfinite(e)
    gx, hx = _gradient(e, valid, r_g, axis=1)
    gy, hy = _gradient(e, valid, r_g, axis=0)
    return (np.maximum(np.abs(gx), np.abs(gy)), np.hypot(gx, gy),
            valid & ~(hx | hy))


def gentle_fraction(mask, radius):
    side = 2 * radius + 1
    rows, cols = mask.shape
    acc = np.zeros((rows + 1, cols + 1), np.int64)
    acc[1:, 1:] = mask.astype(np.int64).cumsum(0).cumsum(1)
    r_lo = np.clip(np.arange(rows) - radius, 0, rows)
    r_hi = np.clip(np.arange(rows) + radius + 1, 0, rows)
    c_lo = np.clip(np.arange(cols) - radius, 0, cols)
    c_hi = np.clip(np.arange(cols) + radius + 1, 0, cols)
    cnt = (acc[r_hi][:, c_hi] - acc[r_hi][:, c_lo] - acc[r_lo][:, c_hi] + acc[r_lo][:, c_lo])
    return cnt / float(side * side)


def terrain_cost_values(m_xy, m_grad, p_s, params):
    m_xy = np.asarray(m_xy, np.float64)
    m_grad = np.asarray(m_grad, np.float64)
    p_s = np.asarray(p_s, np.float64)
    step = np.where(p_s > params.theta_p, params.alpha_b * (m_xy / params.theta_b) ** 2,
                    params.c_barrier)
    gentle = params.alpha_s * (m_grad / params.theta_s) ** 2
    return np.where(m_xy > params.theta_b, params.c_barrier,
                    np.where(m_grad < params.theta_s, gentle, step))


def ground_cost(e, r_g, params):
    valid = np.isfinite(e)
    m_xy, m_grad, isolated = slope_magnitudes(e, r_g)
    p_s = gentle_fraction(valid & (m_grad < params.theta_s), patch_radius(params, r_g))
    out = terrain_cost_values(m_xy, m_grad, p_s, params)
    out = np.where(isolated, params.c_barrier, out)
    return np.where(valid, out, 0.0).astype(np.float32)


def fuse_costs(ci, cg, ground_valid, params):
    tot = np.minimum(np.float64(params.c_barrier),
                     ci.astype(np.float64) + cg.astype(np.float64))
    return np.where(ground_valid, tot, params.c_barrier).astype(np.float32)


def kernel_weights(d_inf, d_sm, r_g):
    if not (r_g <= d_inf < d_sm):
        raise ValueError("need r_g <= d_inf < d_sm")
    R = int(math.ceil(d_sm / r_g))
    o = np.arange(-R, R + 1, dtype=np.float64) * r_g
    d = np.hypot(o[:, None], o[None, :])
    return np.maximum(0.0, np.minimum(1.0 - (d - d_inf) / (d_sm - r_g), 1.0)).astype(np.float32)


def inflate(c, w):
    """max over weight classes of w * (flat max filter, zero padding)."""
    c = np.asarray(c, np.float32)
    out = np.zeros_like(c)
    for val in np.unique(w)[::-1]:
        if val <= 0:
            continue
        m = ndimage.maximum_filter(c, footprint=(w == val), mode="constant", cval=0.0)
        np.maximum(out, np.float32(val) * m, out=out)
    return out


def evaluate_slice(g, c, r_g, params, w=None):
    if w is None:
        w = kernel_weights(params.d_inf, params.d_sm, r_g)
    ci = interval_cost(g, c, params)
    cg = ground_cost(g, r_g, params)
    return inflate(fuse_costs(ci, cg, np.isfinite(g), params), w)


def evaluate(ground, ceiling, r_g, params, threads=1):
    """Cost stack (S, rows, cols) float32 for ground/ceiling stacks."""
    w = kernel_weights(params.d_inf, params.d_sm, r_g)
    S = ground.shape[0]
    if threads > 1:
        with ThreadPoolExecutor(threads) as ex:
            outs = list(ex.map(lambda k: evaluate_slice(ground[k], ceiling[k], r_g, params, w),
                               range(S)))
    else:
        outs = [evaluate_slice(ground[k], ceiling[k], r_g, params, w) for k in range(S)]
    return np.stack(outs) if outs else np.zeros((0,) + ground.shape[1:], np.float32)
