"""Oracle: planner context arrays (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

numpy restatement of the canonical-node run merge of planner.py:65-93: runs
of adjacent slices whose ground is valid in both and equal within eps_e are
one node; canon = first slice of the run, cn = run-minimum cost broadcast to
every member (inf where the ground is invalid)."""

import numpy as np


def planner_context(ground, cost, eps_e=1e-6):
    S = ground.shape[0]
    valid = np.isfinite(ground)
    same = np.zeros_like(valid)
    if S > 1:
        e = np.where(valid, ground, 0.0).astype(np.float64)
        same[1:] = valid[1:] & valid[:-1] & (np.abs(e[1:] - e[:-1]) <= eps_e)
    canon = np.zeros(ground.shape, np.int32)
    for k in range(1, S):
        canon[k] = np.where(same[k], canon[k - 1], k)
    cn = np.where(valid, cost, np.float32(np.inf)).astype(np.float32)
    for k in range(1, S):
        cn[k] = np.where(same[k], np.minimum(cn[k], cn[k - 1]), cn[k])
    for k in range(S - 2, -1, -1):
        cn[k] = np.where(same[k + 1], cn[k + 1], cn[k])
    return canon, cn
