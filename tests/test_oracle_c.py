"""The multi-threaded C oracle (oracle/fast.py) pinned to the reference's
recorded outputs and to the numpy oracle (CPU only).

The C oracle is the checker of the full-size GPU parity tests (config 3 at
200M points) and the CPU baseline / reference arm of bench.py, so it gets
the same golden pins as the numpy oracle plus the config-3 ones
(tests/golden/golden_r2.json, written by make_golden_r2.py from the
reference) and randomised cross-checks against the numpy restatement."""

import json

import numpy as np
import pytest

import oracle
from golden_util import GOLDEN, TABLE_PARAMS, case_input, digest
from oracle import fast

ALL_REF_CASES = ["ref_random_multilayer_s9", "ref_flat_plane_s7", "ref_spiral_s3",
                 "ref_ramp_over_tunnel_s6", "synth_cfg0", "synth_cfg4", "synth_two_storey_small",
                 "synth_cfg1", "synth_cfg2_n2000000"]


@pytest.fixture(scope="module")
def golden_r2():
    return json.loads((GOLDEN / "golden_r2.json").read_text())


def test_library_builds_and_loads():
    fast.build_lib()
    for sym in ("orc_bounds", "orc_build", "orc_evaluate", "orc_unique_any", "orc_simplify"):
        assert hasattr(fast.lib(), sym)


@pytest.mark.parametrize("name", ALL_REF_CASES)
def test_c_oracle_matches_reference(golden, name):
    case = golden["cases"][name]
    xyz = case_input(name, case)
    t, cost, keep = fast.pipeline(xyz, case["d_s"], case["r_g"], TABLE_PARAMS)
    assert list(t["ground"].shape) == case["shape"]
    assert [float(h) for h in t["heights"]] == case["heights"]
    assert list(t["origin"]) == case["origin"]
    assert digest(t["ground"]) == case["ground_sha256"]
    assert digest(t["ceiling"]) == case["ceiling_sha256"]
    assert digest(cost) == case["cost_sha256"]
    assert keep == case["keep"]


def campus_input(case):
    from paper_2403_07631_b200 import synth
    box = tuple(case["box"]) if case["box"] else None
    xyz = synth.campus(case["n_full"], case["seed"], box=box)
    assert digest(xyz) == case["input_sha256"], "campus generator drift"
    return xyz


def check_slices(case, ground, ceiling, cost, keep, heights):
    assert [float(h) for h in heights] == case["heights"]
    assert [digest(g) for g in ground] == case["ground_slice_sha256"]
    assert [digest(c) for c in ceiling] == case["ceiling_slice_sha256"]
    assert [digest(c) for c in cost] == case["cost_slice_sha256"]
    assert list(keep) == case["keep"]


@pytest.mark.parametrize("name", ["campus_crop", "campus_sparse"])
def test_c_oracle_matches_reference_campus(golden_r2, name):
    """Config 3 (campus): a full-density crop of the 200M-point map and the
    full 4004 x 4004 x 44 frame, pinned to the reference's per-slice digests."""
    case = golden_r2["cases"][name]
    xyz = campus_input(case)
    t, cost, keep = fast.pipeline(xyz, case["d_s"], case["r_g"], TABLE_PARAMS)
    assert list(t["ground"].shape) == case["shape"]
    assert list(t["origin"]) == case["origin"]
    check_slices(case, t["ground"], t["ceiling"], cost, keep, t["heights"])


def test_numpy_oracle_matches_reference_campus_crop(golden_r2):
    case = golden_r2["cases"]["campus_crop"]
    xyz = campus_input(case)
    t = oracle.build(xyz, case["d_s"], case["r_g"], threads=4)
    cost = oracle.evaluate(t["ground"], t["ceiling"], case["r_g"], TABLE_PARAMS, threads=4)
    keep = oracle.simplify(t["ground"], cost)
    check_slices(case, t["ground"], t["ceiling"], cost, keep, t["heights"])


def test_campus_crop_is_exact_crop():
    """synth.campus(box=...) yields exactly the full cloud's points in the box."""
    from paper_2403_07631_b200 import synth
    full = synth.campus(3_000_000, 3)
    box = (120.0, 140.0, 180.0, 170.0)
    m = (full[:, 0] >= box[0]) & (full[:, 0] < box[2]) & (full[:, 1] >= box[1]) & \
        (full[:, 1] < box[3])
    assert np.array_equal(full[m], synth.campus(3_000_000, 3, box=box))


def _random_scene(seed, n=40_000, layers=3):
    rng = np.random.default_rng(seed)
    pts = []
    for l in range(layers):
        m = n // layers
        x = rng.uniform(0, 12, m)
        y = rng.uniform(0, 9, m)
        z = 2.2 * l + 0.3 * np.sin(x) + 0.2 * (y > 4) + rng.normal(0, 0.02, m)
        pts.append(np.column_stack([x, y, z]))
    xyz = np.concatenate(pts).astype(np.float32)
    # holes and walls
    keep = ~((xyz[:, 0] > 3) & (xyz[:, 0] < 4) & (xyz[:, 1] > 2) & (xyz[:, 1] < 6))
    wall = np.column_stack([np.full(3000, 7.0), rng.uniform(0, 9, 3000), rng.uniform(0, 6, 3000)])
    return np.concatenate([xyz[keep], wall.astype(np.float32)])


@pytest.mark.parametrize("seed,r_g,d_s", [(1, 0.1, 0.5), (2, 0.05, 0.3), (3, 0.2, 0.4),
                                          (4, 0.1, 0.25)])
def test_c_oracle_matches_numpy_oracle(seed, r_g, d_s):
    xyz = _random_scene(seed)
    a = oracle.build(xyz, d_s, r_g)
    b = fast.build(xyz, d_s, r_g, threads=3)
    assert np.array_equal(a["ground"].view(np.uint32), b["ground"].view(np.uint32))
    assert np.array_equal(a["ceiling"].view(np.uint32), b["ceiling"].view(np.uint32))
    ca = oracle.evaluate(a["ground"], a["ceiling"], r_g, TABLE_PARAMS)
    cb = fast.evaluate(b["ground"], b["ceiling"], r_g, TABLE_PARAMS, threads=3)
    assert np.array_equal(ca.view(np.uint32), cb.view(np.uint32))
    assert oracle.simplify(a["ground"], ca) == fast.simplify(b["ground"], cb, threads=3)


@pytest.mark.parametrize("over", [dict(step_patch_radius=1), dict(theta_s=0.2, theta_p=0.5),
                                  dict(d_min=0.3, d_ref=1.9, alpha_d=3.0),
                                  dict(c_barrier=37.5, alpha_b=30.0)])
def test_c_oracle_parameter_variants(over):
    from types import SimpleNamespace
    p = SimpleNamespace(**dict(vars(TABLE_PARAMS), **over))
    xyz = _random_scene(7)
    t = fast.build(xyz, 0.5, 0.1)
    ca = oracle.evaluate(t["ground"], t["ceiling"], 0.1, p)
    cb = fast.evaluate(t["ground"], t["ceiling"], 0.1, p)
    assert np.array_equal(ca.view(np.uint32), cb.view(np.uint32))
    assert oracle.simplify(t["ground"], ca, c_barrier=p.c_barrier) == \
        fast.simplify(t["ground"], cb, c_barrier=p.c_barrier)


def test_c_oracle_thread_count_independent():
    """The reference's own determinism criterion (test_tomogram.py:123-138)."""
    xyz = _random_scene(11, n=120_000)
    perm = np.random.default_rng(0).permutation(len(xyz))
    outs = []
    for threads, pts in ((1, xyz), (2, xyz), (7, xyz[perm]), (16, xyz.astype(np.float64))):
        t, cost, keep = fast.pipeline(pts, 0.5, 0.1, TABLE_PARAMS, threads=threads)
        outs.append((digest(t["ground"]), digest(t["ceiling"]), digest(cost), keep))
    assert all(o == outs[0] for o in outs)


def test_c_oracle_edge_cases():
    # one point: one slice, one valid cell
    t = fast.build(np.array([[1.0, 2.0, 3.0]], np.float32), 0.5, 0.1)
    assert t["ground"].shape == (1, 2, 2)
    assert np.isfinite(t["ground"]).sum() == 1
    assert np.array_equal(t["ground"].view(np.uint32)[~np.isfinite(t["ground"])],
                          np.full(3, 0x7FC00000, np.uint32))
    # tie at a plane height goes to ground (test_tomogram.py:72-79)
    pts = np.array([[0, 0, 0.0], [0, 0, 0.5], [0.3, 0.3, 1.0]], np.float64)
    a, b = oracle.build(pts, 0.5, 0.1), fast.build(pts, 0.5, 0.1)
    assert np.array_equal(a["ground"], b["ground"], equal_nan=True)
    assert np.array_equal(a["ceiling"], b["ceiling"], equal_nan=True)
    assert b["ground"][0, 0, 0] == np.float32(0.5)
    # grid size limit
    with pytest.raises(ValueError):
        fast.build(np.array([[0, 0, 0], [100.0, 0, 0]]), 0.5, 0.1, max_grid_side=100)
    with pytest.raises(ValueError):
        fast.build(np.zeros((2, 3)), 0.0, 0.1)


def test_unique_any_matches_numpy_mask():
    xyz = _random_scene(5)
    t = fast.build(xyz, 0.5, 0.1)
    cost = fast.evaluate(t["ground"], t["ceiling"], 0.1, TABLE_PARAMS)
    S = t["ground"].shape[0]
    rng = np.random.default_rng(3)
    for _ in range(30):
        k = int(rng.integers(S))
        below = None if rng.random() < 0.3 or k == 0 else int(rng.integers(0, k))
        above = None if rng.random() < 0.3 or k == S - 1 else int(rng.integers(k + 1, S))
        want = oracle.unique_mask(t["ground"], cost, k, below, above).any()
        assert fast.unique_any(t["ground"], cost, k, below, above) == want


# ---------------------------------------------------------------------------
# planner lookups (planner.py:95-129) pinned to the reference's answers

def _host_planner_context(ground, cost, heights_res_origin):
    """A PlannerContext with the oracle's canon / cn arrays (its lookups are
    host-side code; the arrays come from the GPU in the product)."""
    from oracle.planner_ctx import planner_context
    from paper_2403_07631_b200.planner_ctx import PlannerContext
    res, origin = heights_res_origin
    pc = PlannerContext.__new__(PlannerContext)
    pc.eps_e, pc.c_barrier, pc.res, pc.origin = 1e-6, 50.0, res, origin
    pc.canon, pc.cn = planner_context(ground, cost)
    pc.elev, pc.cost, pc.valid = ground, cost, np.isfinite(ground)
    return pc


@pytest.mark.parametrize("name", ["synth_cfg0", "spiral_crop"])
def test_snap_matches_reference(golden_r2, name):
    from paper_2403_07631_b200 import synth
    case = golden_r2["snap"][name]
    cfg = 0 if name == "synth_cfg0" else 1
    xyz = synth.generate(cfg, case["n_points"])
    assert digest(xyz) == case["input_sha256"]
    t, cost, keep = fast.pipeline(xyz, case["d_s"], case["r_g"], TABLE_PARAMS)
    for which, g, c in (("evaluated", t["ground"], cost),
                        ("simplified", t["ground"][keep], cost[keep])):
        pc = _host_planner_context(g, c, (case["r_g"], t["origin"]))
        for q in case[which]:
            got = pc.snap(q["point"], q["tol"])
            assert (None if got is None else list(got)) == q["snap"], (which, q)
            if got is not None:
                assert pc.member_with_min_cost(*got) == q["member"], (which, q)
