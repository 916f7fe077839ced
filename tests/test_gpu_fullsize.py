"""Full-size checks: BASELINE config 2 (20M points, 2005 x 2005 cells, 25
slices, the R = 8 inflation kernel) through the GPU path against the CPU
oracle bit for bit, and through size-independent properties (slice
monotonicity, plane bracketing, build / evaluate variants agreeing, point
order and input precision, simplify idempotence).  Config 1 at full size is
pinned to the reference's own outputs in test_gpu_parity (synth_cfg1).
"""

import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

pct = pytest.importorskip("paper_2403_07631_b200")
from paper_2403_07631_b200 import synth  # noqa: E402

CFG = 2
D_S, R_G = synth.CONFIGS[CFG]["d_s"], synth.CONFIGS[CFG]["r_g"]


@pytest.fixture(scope="module")
def cloud():
    return synth.generate(CFG)


@pytest.fixture(scope="module")
def gpu(cloud):
    tom = pct.build_tomogram(pct.PointCloud(cloud), D_S, R_G)
    ev = pct.evaluate_tomogram(tom, pct.TravParams())
    simp = pct.simplify_tomogram(ev)
    return dict(heights=np.array([s.plane_height for s in tom.slices]),
                ground=ev.ground_stack(), ceiling=ev.ceiling_stack(), cost=ev.cost_stack(),
                keep=[s.plane_height for s in simp.slices], simp=simp)


def _same(a, b):
    return a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_full_size_matches_oracle(cloud, gpu):
    threads = os.cpu_count() or 1
    ref = oracle.build(cloud, D_S, R_G, threads=threads)
    assert np.array_equal(gpu["heights"], np.asarray(ref["heights"]))
    assert _same(gpu["ground"], np.asarray(ref["ground"], np.float32))
    assert _same(gpu["ceiling"], np.asarray(ref["ceiling"], np.float32))
    cost = oracle.evaluate(ref["ground"], ref["ceiling"], R_G, pct.TravParams(), threads=threads)
    assert _same(gpu["cost"], cost)
    keep = oracle.simplify(ref["ground"], cost)
    assert gpu["keep"] == [float(ref["heights"][k]) for k in keep]


def test_slices_are_monotone_and_bracket_the_planes(gpu):
    g, c, h = gpu["ground"], gpu["ceiling"], gpu["heights"]
    # ground[k] = max z <= h[k]: once present it stays, and never decreases
    fg = np.isfinite(g)
    assert not (fg[:-1] & ~fg[1:]).any()
    both = fg[:-1] & fg[1:]
    assert (g[1:][both] >= g[:-1][both]).all()
    assert (g.astype(np.float64) <= h[:, None, None])[fg].all()
    # ceiling[k] = min z > h[k]: once gone it stays gone, and never decreases
    fc = np.isfinite(c)
    assert not (~fc[:-1] & fc[1:]).any()
    both = fc[:-1] & fc[1:]
    assert (c[1:][both] >= c[:-1][both]).all()
    assert (c.astype(np.float64) > h[:, None, None])[fc].all()


def test_costs_bounded_and_barrier_where_no_ground(gpu):
    g, cost = gpu["ground"], gpu["cost"]
    p = pct.TravParams()
    assert np.isfinite(cost).all()
    assert (cost >= 0).all() and (cost <= p.c_barrier).all()
    assert (cost[~np.isfinite(g)] == np.float32(p.c_barrier)).all()


@pytest.mark.parametrize("build", ["atomic", "tiled", "hist"])
def test_build_variants_agree(cloud, gpu, monkeypatch, build):
    monkeypatch.setenv("PCT_BUILD", build)
    tom = pct.build_tomogram(pct.PointCloud(cloud), D_S, R_G)
    assert _same(tom.ground_stack(), gpu["ground"])
    assert _same(tom.ceiling_stack(), gpu["ceiling"])


def test_point_order_and_precision(cloud, gpu):
    perm = np.random.default_rng(7).permutation(len(cloud))
    tom = pct.build_tomogram(pct.PointCloud(cloud[perm].astype(np.float64)), D_S, R_G)
    assert _same(tom.ground_stack(), gpu["ground"])
    assert _same(tom.ceiling_stack(), gpu["ceiling"])


@pytest.mark.parametrize("env", [("PCT_BNB_SKIP", "0"), ("PCT_BNB_TILE", "1")])
def test_evaluate_variants_agree(cloud, gpu, monkeypatch, env):
    monkeypatch.setenv(*env)
    tom = pct.build_tomogram(pct.PointCloud(cloud), D_S, R_G)
    assert _same(pct.evaluate_tomogram(tom, pct.TravParams()).cost_stack(), gpu["cost"])


def test_simplify_is_idempotent(gpu):
    again = pct.simplify_tomogram(gpu["simp"])
    assert [s.plane_height for s in again.slices] == gpu["keep"]
