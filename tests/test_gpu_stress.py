"""Randomised full-chain parity on the GPU against the C oracle (the CPU
restatement pinned to the reference's golden vectors in test_oracle_c.py):
scene kinds, grid steps, slice counts on both sides of the 64-slice mask
limit and past the histogram build's 100-slice limit, non-default traversal
parameters (full-tap inflation fallback), heavy exact-tie z values, sparse
clouds; every slice of ground / ceiling / cost bitwise, the keep list, and
the host layers of the compacted read-back (Tomogram.materialize)."""
import numpy as np
import pytest

import paper_2403_07631_b200 as pct
from paper_2403_07631_b200 import synth

pytestmark = pytest.mark.gpu

fast = pytest.importorskip("oracle.fast")


def _ties(n, seed):
    rng = np.random.default_rng(seed)
    return np.column_stack([rng.uniform(0, 40, n), rng.uniform(0, 30, n),
                            np.round(rng.uniform(0, 6, n) * 10) / 10]).astype(np.float32)


def _tall(n, seed):  # ~10 m of z over a small footprint: > 64 and > 100 slices
    rng = np.random.default_rng(seed)
    x, y = rng.uniform(0, 12, n), rng.uniform(0, 10, n)
    z = np.where(rng.random(n) < 0.5, 0.02 * x, rng.uniform(0, 10.5, n))
    return np.column_stack([x, y, z]).astype(np.float32)


def _long_thin(n, seed):  # 800 m x 8 m, negative coordinates, a ramp
    rng = np.random.default_rng(seed)
    x, y = rng.uniform(-500, 300, n), rng.uniform(-4, 4, n)
    return np.column_stack([x, y, 0.004 * (x + 500) + rng.uniform(0, 0.05, n)]).astype(np.float32)


def _sparse(n, seed):  # few points over a wide area: mostly empty cells
    rng = np.random.default_rng(seed)
    return np.column_stack([rng.uniform(0, 200, n), rng.uniform(0, 150, n),
                            rng.uniform(0, 3, n)]).astype(np.float32)


CASES = [
    # name, cloud factory, d_s, r_g, TravParams kwargs
    ("campus_box_a", lambda: synth.campus(3_000_000, 11, box=(100, 100, 180, 170)), 0.5, 0.1, {}),
    ("campus_box_b", lambda: synth.campus(2_000_000, 12, box=(0, 0, 120, 90)), 0.4, 0.1, {}),
    ("terrain_r8", lambda: synth.rough_terrain(1_500_000, 21, extent=60.0), 0.3, 0.05, {}),
    ("spiral_d_inf", lambda: synth.spiral_ramp(1_000_000, 31), 0.5, 0.1, {"d_inf": 0.25}),
    ("two_storey_thin", lambda: synth.two_storey(400_000, 41, jitter=True), 0.12, 0.1, {}),
    ("ties", lambda: _ties(600_000, 51), 0.3, 0.1, {}),
    ("tall_80", lambda: _tall(300_000, 61), 0.13, 0.1, {}),
    ("tall_110", lambda: _tall(300_000, 62), 0.095, 0.1, {}),
    ("sparse_wide", lambda: _sparse(200_000, 71), 0.5, 0.1, {}),
    ("long_thin", lambda: _long_thin(1_500_000, 81), 0.4, 0.1, {}),
    ("f64_input", lambda: _ties(300_000, 91).astype(np.float64), 0.3, 0.1, {}),
]


@pytest.mark.parametrize("name,make,d_s,r_g,kw", CASES, ids=[c[0] for c in CASES])
def test_full_chain_matches_c_oracle(name, make, d_s, r_g, kw):
    xyz = make()
    params = pct.TravParams(**kw)
    t, cost, keep = fast.pipeline(xyz, d_s, r_g, params)
    tom = pct.build_tomogram(pct.PointCloud(xyz), d_s, r_g)
    ev = pct.evaluate_tomogram(tom, params)
    g, c, k = ev.ground_stack(), ev.ceiling_stack(), ev.cost_stack()
    assert g.shape == t["ground"].shape, name
    assert np.array_equal(g.view(np.uint32), t["ground"].view(np.uint32)), f"{name}: ground"
    assert np.array_equal(c.view(np.uint32), t["ceiling"].view(np.uint32)), f"{name}: ceiling"
    assert np.array_equal(k.view(np.uint32), cost.view(np.uint32)), f"{name}: cost"
    simp = pct.simplify_tomogram(pct.evaluate_tomogram(
        pct.build_tomogram(pct.PointCloud(xyz), d_s, r_g), params))
    heights = list(t["heights"])
    assert [s.plane_height for s in simp.slices] == [float(heights[i]) for i in keep], name
    simp.materialize()  # compacted where it pays (maps of >= 1M cells)
    for s, i in zip(simp.slices, keep):
        assert np.array_equal(s.ground.values.view(np.uint32), t["ground"][i].view(np.uint32))
        assert np.array_equal(s.ceiling.values.view(np.uint32), t["ceiling"][i].view(np.uint32))
        assert np.array_equal(s.cost.values.view(np.uint32), cost[i].view(np.uint32))
