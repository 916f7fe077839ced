"""Ceiling layers for the ceiling-inflation parity cases (shared by
tests/golden/make_golden_traj.py and tests/test_trajectory_ceiling.py)."""

from __future__ import annotations

from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"

# (erosion, skirt_slope): defaults (trajectory.py:71-72); no min filter; wider
# disk with the 60-sweep cap; steep slope (4 sweeps); negative slope (60
# sweeps of a decreasing skirt, no fixpoint)
PARAMS = [(0.20, 0.30), (0.0, 0.30), (0.35, 0.10), (0.20, 2.0), (0.15, -0.05)]


def layers():
    """(name, float32 (rows, cols) ceiling with NaN holes, resolution)."""
    out = []
    d = np.load(GOLDEN / "synth_two_storey_small.npz")
    for k in (0, 5, 6, 12):
        out.append((f"two_storey_small_c{k}", d["ceiling"][k], 0.1))
    d = np.load(GOLDEN / "ref_random_multilayer_s9.npz")
    for k in (0, 3):
        out.append((f"random_multilayer_c{k}", d["ceiling"][k], 0.1))
    strip = np.full((90, 70), np.nan, np.float32)
    strip[40:46, :] = np.float32(0.55)          # low overhang strip (test_trajectory.py:273)
    strip[10:12, 5:9] = np.float32(-1.25)       # negative heights
    out.append(("strip", strip, 0.05))
    out.append(("all_nan", np.full((17, 33), np.nan, np.float32), 0.1))
    rng = np.random.default_rng(5)
    speck = np.where(rng.random((64, 129)) < 0.02,
                     rng.uniform(0.3, 3.0, (64, 129)), np.nan).astype(np.float32)
    out.append(("specks", speck, 0.2))
    return out
