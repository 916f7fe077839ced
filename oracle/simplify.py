"""Oracle: redundant-slice simplification (TEST INFRASTRUCTURE ONLY).

numpy restatement of tomoplan/simplify.py:18-73: the per-cell uniqueness
test (paper Eqs. 8-9; _side_condition :18-28, _unique_mask :31-43) and the
forward sweep to a fixpoint that never removes the last remaining slice
(:59-70).  Works on stacks; returns the surviving original slice indices.
"""

from __future__ import annotations

import numpy as np


def _not_covered(e, cost, e_nb, cost_nb, eps_e, lower):
    nv = np.isfinite(e_nb)
    a = np.where(np.isfinite(e), e, 0.0).astype(np.float64)
    b = np.where(nv, e_nb, 0.0).astype(np.float64)
    higher = (a - b > eps_e) if lower else (b - a > eps_e)
    return np.where(nv, higher | (cost < cost_nb), True)


def unique_mask(ground, cost, k, below, above, eps_e=1e-6, c_barrier=50.0):
    """Unique cells of slice k given neighbour slice indices (None = absent)."""
    m = np.isfinite(ground[k]) & (cost[k] < c_barrier)
    if below is not None:
        m &= _not_covered(ground[k], cost[k], ground[below], cost[below], eps_e, True)
    if above is not None:
        m &= _not_covered(ground[k], cost[k], ground[above], cost[above], eps_e, False)
    return m


def simplify(ground, cost, eps_e=1e-6, c_barrier=50.0, trace=None):
    """Surviving slice indices after the reference's forward sweep.

    ``trace`` (a list) receives every (below, k, above, unique_any) check in
    order, which tests use to pin the device sweep step by step."""
    keep = list(range(ground.shape[0]))
    changed = True
    while changed:
        changed = False
        p = 0
        while p < len(keep):
            if len(keep) > 1:
                below = keep[p - 1] if p > 0 else None
                above = keep[p + 1] if p + 1 < len(keep) else None
                anyu = bool(unique_mask(ground, cost, keep[p], below, above,
                                        eps_e, c_barrier).any())
                if trace is not None:
                    trace.append((below, keep[p], above, anyu))
                if not anyu:
                    del keep[p]
                    changed = True
                    continue
            p += 1
    return keep
