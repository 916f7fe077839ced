"""Oracle: the trajectory optimiser's ceiling inflation.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  numpy restatement of
``_inflate_ceiling`` (tomoplan/trajectory.py:277-317) without scipy:

* flat: +inf where invalid (:288), then the minimum over the disk footprint
  of radius ceil(erosion/res) cells (:291-296), outside the grid = +inf;
  computed as a running minimum over shifted copies of an inf-padded array.
* skirted: Jacobi sweeps (:298-316) — each sweep takes, for every cell, the
  minimum of its previous value and (neighbour + step) / (diagonal
  neighbour + step*sqrt(2)) over the 8 neighbours of the previous sweep;
  at most min(60, ceil(0.8/step)) sweeps, stopping at a fixpoint.
Pinned by tests/golden/golden_traj.json (the reference's own outputs).
"""

from __future__ import annotations

import math

import numpy as np


def _shift_min(a: np.ndarray, offsets, add=None) -> np.ndarray:
    """min over (di, dj) of a[i+di, j+dj] (+ add[k]), inf outside the grid."""
    rows, cols = a.shape
    r = max(max(abs(di), abs(dj)) for di, dj in offsets)
    pad = np.full((rows + 2 * r, cols + 2 * r), np.inf)
    pad[r:r + rows, r:r + cols] = a
    out = np.full_like(a, np.inf)
    for k, (di, dj) in enumerate(offsets):
        v = pad[r + di:r + di + rows, r + dj:r + dj + cols]
        if add is not None:
            v = v + add[k]
        np.minimum(out, v, out=out)
    return out


def inflate_ceiling(values, valid, res, erosion, skirt_slope):
    flat = np.where(valid, np.asarray(values, np.float64), np.inf)
    if not np.isfinite(flat).any():
        return flat, flat
    radius = int(math.ceil(erosion / res))
    if radius > 0:
        disk = [(di, dj) for di in range(-radius, radius + 1)
                for dj in range(-radius, radius + 1) if di * di + dj * dj <= radius * radius]
        flat = _shift_min(flat, disk)
    step = skirt_slope * res
    sweeps = min(60, int(math.ceil(0.8 / max(step, 1e-9))))
    nbrs = [(di, dj) for di in (-1, 0, 1) for dj in (-1, 0, 1) if di or dj]
    w = [step * (math.sqrt(2.0) if di and dj else 1.0) for di, dj in nbrs]
    out = flat.copy()
    for _ in range(sweeps):
        nxt = np.minimum(out, _shift_min(out, nbrs, w))
        if np.array_equal(nxt, out):
            break
        out = nxt
    return flat, out
