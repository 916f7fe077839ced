"""GPU parity: the sm_100a path (through libpct's C ABI) against the reference's
recorded outputs (tests/golden) and the pinned CPU oracle.

Bars (BASELINE.json north_star): ground / ceiling / slice set bit-exact; costs
are compared bit-exact too (stricter than the 1e-5 relative tolerance the
north_star allows) and the traversable classification identical.
"""

import numpy as np
import pytest

import oracle
from golden_util import TABLE_PARAMS, case_arrays, case_input, digest

pytestmark = pytest.mark.gpu

pct = pytest.importorskip("paper_2403_07631_b200")

COST_RTOL = 1e-5  # north_star tolerance; the checks below demand exact equality first


def _run(xyz, d_s, r_g):
    cloud = pct.PointCloud(xyz)
    tom = pct.build_tomogram(cloud, d_s, r_g)
    ev = pct.evaluate_tomogram(tom, pct.TravParams())
    simp = pct.simplify_tomogram(ev)
    return tom, ev, simp


def _assert_layers_equal(got, want, what):
    assert got.shape == want.shape, what
    if not np.array_equal(got, want, equal_nan=True):
        bad = ~((got == want) | (np.isnan(got) & np.isnan(want)))
        k, i, j = np.argwhere(bad)[0]
        raise AssertionError(f"{what}: {bad.sum()} cells differ, first at slice {k} "
                             f"({i},{j}): got {got[k, i, j]!r} want {want[k, i, j]!r}")


GOLDEN_CASES = ["ref_random_multilayer_s9", "ref_flat_plane_s7", "ref_spiral_s3",
                "ref_ramp_over_tunnel_s6", "synth_cfg0", "synth_cfg4", "synth_two_storey_small",
                "synth_cfg1", "synth_cfg2_n2000000"]


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_pipeline_matches_reference_golden(golden, name):
    case = golden["cases"][name]
    xyz = case_input(name, case)
    tom, ev, simp = _run(xyz, case["d_s"], case["r_g"])
    assert [s.plane_height for s in tom.slices] == case["heights"]
    assert list(tom.origin) == case["origin"] and tom.z_min == case["z_min"]
    g, c, cost = ev.ground_stack(), ev.ceiling_stack(), ev.cost_stack()
    assert list(g.shape) == case["shape"]
    arrays = case_arrays(case)
    if arrays is not None and "ground" in arrays:
        _assert_layers_equal(g, arrays["ground"], "ground")
        _assert_layers_equal(c, arrays["ceiling"], "ceiling")
        _assert_layers_equal(cost, arrays["cost"], "cost")
    for k in range(g.shape[0]):
        assert digest(g[k]) == case["ground_slice_sha256"][k], f"ground slice {k}"
        assert digest(c[k]) == case["ceiling_slice_sha256"][k], f"ceiling slice {k}"
        assert digest(cost[k]) == case["cost_slice_sha256"][k], f"cost slice {k}"
    heights = [s.plane_height for s in simp.slices]
    assert heights == [case["heights"][k] for k in case["keep"]]
    assert [s.index for s in simp.slices] == list(range(len(simp.slices)))


@pytest.mark.parametrize("run", ["1", "2", "5", "64"])
def test_incremental_runs_match_full_kernel(golden, monkeypatch, run):
    """The slice-incremental kernel gives the same bytes for any run length
    as the full per-slice kernel (PCT_EVAL_KERNEL=fast)."""
    case = golden["cases"]["synth_cfg0"]
    tom = pct.build_tomogram(pct.PointCloud(case_input("synth_cfg0", case)), 0.5, 0.1)
    monkeypatch.setenv("PCT_EVAL_KERNEL", "fast")
    full = pct.evaluate_tomogram(tom, pct.TravParams()).cost_stack()
    monkeypatch.setenv("PCT_EVAL_KERNEL", "incr")
    monkeypatch.setenv("PCT_EVAL_RUN", run)
    inc = pct.evaluate_tomogram(tom, pct.TravParams()).cost_stack()
    assert np.array_equal(full.view(np.uint32), inc.view(np.uint32))
    for k in range(full.shape[0]):
        assert digest(inc[k]) == case["cost_slice_sha256"][k]


@pytest.mark.parametrize("name,env", [("synth_cfg0", {"PCT_INFL": "sym"}),
                                      ("synth_cfg0", {}),
                                      ("ref_random_multilayer_s9", {}),
                                      ("synth_cfg2_n2000000", {})])
def test_split_paths_match_fused_kernel(golden, monkeypatch, name, env):
    """The two-kernel split (terrain walk + branch-and-bound or full-tap
    inflation) gives the same bytes as the fused per-slice kernel."""
    case = golden["cases"][name]
    tom = pct.build_tomogram(pct.PointCloud(case_input(name, case)), case["d_s"], case["r_g"])
    monkeypatch.setenv("PCT_EVAL_KERNEL", "fast")
    full = pct.evaluate_tomogram(tom, pct.TravParams()).cost_stack()
    monkeypatch.setenv("PCT_EVAL_KERNEL", "split")
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    got = pct.evaluate_tomogram(tom, pct.TravParams()).cost_stack()
    assert np.array_equal(full.view(np.uint32), got.view(np.uint32))


@pytest.mark.parametrize("r_g,d_inf,d_sm,patch", [(0.1, 0.2, 0.4, None), (0.05, 0.2, 0.4, None),
                                                  (0.1, 0.25, 0.4, None), (0.05, 0.25, 0.4, None),
                                                  (0.1, 0.2, 0.4, 4)])
def test_inflation_kernels_vs_oracle_random_costs(r_g, d_inf, d_sm, patch):
    """Branch-and-bound inflation (and its full-tap fallback for kernels
    whose weight-1 disk differs from the compiled one) on random scenes with
    non-default inflation radii, against the oracle."""
    rng = np.random.default_rng(int(r_g * 1000 + d_inf * 100))
    n = 80_000
    xyz = np.column_stack([rng.uniform(0, 9, n), rng.uniform(0, 7, n),
                           rng.uniform(0, 2.5, n)])
    params = pct.TravParams(d_inf=d_inf, d_sm=d_sm, step_patch_radius=patch)
    ref = oracle.build(xyz, 0.5, r_g)
    tom = pct.build_tomogram(pct.PointCloud(xyz), 0.5, r_g)
    got = pct.evaluate_tomogram(tom, params).cost_stack()
    want = oracle.evaluate(ref["ground"], ref["ceiling"], r_g, params)
    _assert_layers_equal(got, want, "cost")


@pytest.mark.parametrize("name", ["synth_cfg0", "ref_random_multilayer_s9", "ref_spiral_s3",
                                  "synth_cfg2_n2000000"])
@pytest.mark.parametrize("mode", ["tiled", "hist"])
def test_tiled_build_matches_reference_golden(golden, monkeypatch, name, mode):
    """The partitioned builds (PCT_BUILD=tiled: bucket by 8x32-cell tile with
    hash-merged passes; PCT_BUILD=hist: per-CTA histograms of 8x64-cell
    buckets; both reduce max / min in shared memory) give the reference's
    layers too."""
    monkeypatch.setenv("PCT_BUILD", mode)
    case = golden["cases"][name]
    xyz = case_input(name, case)
    for arr in (xyz, xyz.astype(np.float64)):
        tom = pct.build_tomogram(pct.PointCloud(arr), case["d_s"], case["r_g"])
        g, c = tom.ground_stack(), tom.ceiling_stack()
        for k in range(g.shape[0]):
            assert digest(g[k]) == case["ground_slice_sha256"][k], f"ground slice {k}"
            assert digest(c[k]) == case["ceiling_slice_sha256"][k], f"ceiling slice {k}"


def test_f32_and_f64_inputs_agree(golden):
    case = golden["cases"]["synth_cfg0"]
    xyz = case_input("synth_cfg0", case)
    a = pct.build_tomogram(pct.PointCloud(xyz), 0.5, 0.1)
    b = pct.build_tomogram(pct.PointCloud(xyz.astype(np.float64)), 0.5, 0.1)
    assert np.array_equal(a.ground_stack(), b.ground_stack(), equal_nan=True)
    assert np.array_equal(a.ceiling_stack(), b.ceiling_stack(), equal_nan=True)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_random_scenes_vs_oracle(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2_000, 60_000))
    xyz = np.column_stack([rng.uniform(-3, 7, n), rng.uniform(-2, 4, n),
                           np.round(rng.uniform(-1, 4, n) * 20) / 20])  # many exact ties
    d_s, r_g = [(0.5, 0.1), (0.3, 0.05), (0.7, 0.2)][seed]
    ref = oracle.build(xyz, d_s, r_g)
    tom, ev, simp = _run(xyz, d_s, r_g)
    _assert_layers_equal(ev.ground_stack(), ref["ground"], "ground")
    _assert_layers_equal(ev.ceiling_stack(), ref["ceiling"], "ceiling")
    cost = oracle.evaluate(ref["ground"], ref["ceiling"], r_g, TABLE_PARAMS)
    _assert_layers_equal(ev.cost_stack(), cost, "cost")
    keep = oracle.simplify(ref["ground"], cost)
    assert [s.plane_height for s in simp.slices] == [float(ref["heights"][k]) for k in keep]


@pytest.mark.parametrize("shape", ["tall", "strip", "column", "wide"])
def test_extreme_shapes_vs_oracle(monkeypatch, shape):
    """Shapes at the kernels' limits: more slices than a bnb work item's
    64-slice skip mask and the tiled build's shared-memory bins (tall), a
    two-column strip (one partial bitmap word per row), a single cell column
    with many slices, and a one-row-of-tiles map wider than the
    32-column tiles; built both ways."""
    rng = np.random.default_rng(11)
    if shape == "tall":  # ~140 slices over a small footprint, stacked floors
        n = 30_000
        xyz = np.column_stack([rng.uniform(0, 3, n), rng.uniform(0, 2, n),
                               np.floor(rng.uniform(0, 70, n)) + rng.normal(0, 0.02, n)])
    elif shape == "strip":
        n = 20_000
        xyz = np.column_stack([rng.uniform(0, 0.1, n), rng.uniform(0, 50, n),
                               rng.uniform(0, 3, n)])
    elif shape == "column":
        n = 5_000
        xyz = np.column_stack([rng.uniform(0, 0.04, n), rng.uniform(0, 0.04, n),
                               rng.uniform(0, 40, n)])
    else:
        n = 40_000
        xyz = np.column_stack([rng.uniform(0, 80, n), rng.uniform(0, 0.5, n),
                               rng.uniform(0, 2, n)])
    d_s, r_g = 0.5, 0.1
    ref = oracle.build(xyz, d_s, r_g)
    cost = oracle.evaluate(ref["ground"], ref["ceiling"], r_g, TABLE_PARAMS)
    keep = oracle.simplify(ref["ground"], cost)
    for build in ("atomic", "tiled", "hist"):
        monkeypatch.setenv("PCT_BUILD", build)
        tom, ev, simp = _run(xyz, d_s, r_g)
        _assert_layers_equal(ev.ground_stack(), ref["ground"], f"ground {build}")
        _assert_layers_equal(ev.ceiling_stack(), ref["ceiling"], f"ceiling {build}")
        _assert_layers_equal(ev.cost_stack(), cost, f"cost {build}")
        assert [s.plane_height for s in simp.slices] == [float(ref["heights"][k]) for k in keep]


@pytest.mark.parametrize("scene", ["plane_tall", "stairs", "random"])
def test_simplify_speculation_matches_host_sweep(monkeypatch, scene):
    """The device-replayed first pass + speculative second-pass triples give
    the same surviving slices as the host-only sweep and the oracle, including
    removal chains longer than the 16-slice window (a plane under a tall
    empty column) and second passes that remove again."""
    rng = np.random.default_rng(3)
    if scene == "plane_tall":
        n = 20_000
        xyz = np.column_stack([rng.uniform(0, 4, n), rng.uniform(0, 4, n), np.zeros(n)])
        xyz = np.vstack([xyz, [[2.0, 2.0, 25.0]]])  # one point far above: ~50 slices
    elif scene == "stairs":
        n = 40_000
        x = rng.uniform(0, 6, n)
        xyz = np.column_stack([x, rng.uniform(0, 3, n), np.floor(x / 0.5) * 0.4])
    else:
        n = 30_000
        xyz = np.column_stack([rng.uniform(0, 5, n), rng.uniform(0, 5, n),
                               np.round(rng.uniform(0, 8, n) * 4) / 4])
    d_s, r_g = 0.5, 0.1
    ref = oracle.build(xyz, d_s, r_g)
    cost = oracle.evaluate(ref["ground"], ref["ceiling"], r_g, TABLE_PARAMS)
    want = [float(ref["heights"][k]) for k in oracle.simplify(ref["ground"], cost)]
    for spec in ("1", "0"):
        monkeypatch.setenv("PCT_SIMPLIFY_SPEC", spec)
        _, _, simp = _run(xyz, d_s, r_g)
        assert [s.plane_height for s in simp.slices] == want, spec


def test_build_speculation_across_layouts(monkeypatch):
    """Consecutive builds on one context with changing grid layouts (smaller,
    larger -> key buffer growth, back, f64 input), with the speculative
    scatter on and off, equal the oracle's stacks."""
    rng = np.random.default_rng(21)

    def cloud(w, h, zmax, n):
        return np.column_stack([rng.uniform(0, w, n), rng.uniform(0, h, n),
                                rng.uniform(0, zmax, n)]).astype(np.float32)

    clouds = [cloud(3, 2, 2, 20_000), cloud(9, 7, 5, 60_000), cloud(3, 2, 2, 20_000),
              cloud(5, 5, 9, 30_000).astype(np.float64), cloud(2, 9, 1, 10_000)]
    for spec in ("1", "0", "1"):
        monkeypatch.setenv("PCT_BUILD_SPEC", spec)
        for xyz in clouds:
            ref = oracle.build(xyz, 0.5, 0.1)
            tom = pct.build_tomogram(pct.PointCloud(xyz), 0.5, 0.1)
            _assert_layers_equal(tom.ground_stack(), ref["ground"], f"ground spec={spec}")
            _assert_layers_equal(tom.ceiling_stack(), ref["ceiling"], f"ceiling spec={spec}")


@pytest.mark.parametrize("chunks", ["1", "3", "7"])
def test_walk_slice_chunks_are_exact(golden, monkeypatch, chunks):
    """The terrain walk split into independent slice chunks (each chunk's
    first slice computed in full) gives the same costs."""
    for name in ("synth_cfg0", "ref_spiral_s3"):
        case = golden["cases"][name]
        tom = pct.build_tomogram(pct.PointCloud(case_input(name, case)), case["d_s"], case["r_g"])
        monkeypatch.delenv("PCT_WALK_CHUNKS", raising=False)
        want = pct.evaluate_tomogram(tom, pct.TravParams()).cost_stack()
        monkeypatch.setenv("PCT_WALK_CHUNKS", chunks)
        got = pct.evaluate_tomogram(tom, pct.TravParams()).cost_stack()
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), name


def test_point_order_independence(golden):
    case = golden["cases"]["synth_cfg0"]
    xyz = case_input("synth_cfg0", case)
    perm = np.random.default_rng(0).permutation(len(xyz))
    a = pct.build_tomogram(pct.PointCloud(xyz), 0.5, 0.1)
    b = pct.build_tomogram(pct.PointCloud(xyz[perm]), 0.5, 0.1)
    assert np.array_equal(a.ground_stack(), b.ground_stack(), equal_nan=True)
    assert np.array_equal(a.ceiling_stack(), b.ceiling_stack(), equal_nan=True)


def test_nan_bits_are_numpy_nan(golden):
    case = golden["cases"]["synth_cfg0"]
    tom = pct.build_tomogram(pct.PointCloud(case_input("synth_cfg0", case)), 0.5, 0.1)
    g = tom.ground_stack().view(np.uint32)
    bad = np.isnan(tom.ground_stack())
    assert bad.any() and np.all(g[bad] == 0x7FC00000)


# --- per-operation API against the oracle -------------------------------------

def _slice_inputs(golden):
    case = golden["cases"]["ref_random_multilayer_s9"]
    arr = case_arrays(case)
    return arr["ground"], arr["ceiling"], arr["cost"]


def test_per_op_functions_match_oracle(golden):
    G, Cc, _ = _slice_inputs(golden)
    P = pct.TravParams()
    for k in range(G.shape[0]):
        g = pct.Layer(G[k], 0.1, (0.0, 0.0))
        c = pct.Layer(Cc[k], 0.1, (0.0, 0.0))
        ci = pct.interval_cost(g, c, P)
        assert np.array_equal(ci, oracle.interval_cost(G[k], Cc[k], P))
        cg = pct.ground_cost(g, P)
        assert np.array_equal(cg, oracle.ground_cost(G[k], 0.1, P))
        mx, mg, iso = pct.slope_magnitudes(g)
        ox, og, oi = oracle.slope_magnitudes(G[k], 0.1)
        assert np.array_equal(mx, ox) and np.array_equal(mg, og) and np.array_equal(iso, oi)
        valid = np.isfinite(G[k])
        f = pct.fuse_costs(ci, cg, valid, P)
        assert np.array_equal(f, oracle.fuse_costs(ci, cg, valid, P))
        gentle = valid & (og < P.theta_s)
        assert np.array_equal(pct.gentle_fraction(gentle, 3), oracle.gentle_fraction(gentle, 3))
        kern = pct.build_kernel(0.2, 0.4, 0.1)
        assert np.array_equal(pct.inflate(f, kern), oracle.inflate(f, kern.weights))


def test_inflation_golden_cases(golden):
    for c in golden["inflation"]:
        kern = pct.build_kernel(0.2, 0.4, c["r_g"])
        assert digest(kern.weights) == c["kernel_sha256"]
        shape = tuple(c["shape"])
        g = np.random.default_rng(c["seed"]).uniform(0.0, 50.0, shape).astype(np.float32)
        g[np.random.default_rng(c["seed"] + 1).uniform(size=shape) < 0.03] = 50.0
        assert digest(pct.inflate(g, kern)) == c["out_sha256"]


def test_terrain_cost_values_kats():
    P = pct.TravParams()
    # test_traversability.py:78-83 / test_acceptance.py:167-170
    assert pct.terrain_cost_values(1.0, 1.2, 0.5, P) == pytest.approx(20.0 * (1.0 / 1.7) ** 2,
                                                                      rel=1e-9)
    assert pct.terrain_cost_values(1.0, 1.2, 0.1, P) == 50.0
    assert pct.terrain_cost_values(2.0, 2.2, 0.9, P) == 50.0
    assert pct.terrain_cost_values(0.18, 0.18, 0.0, P) == pytest.approx(3.75)
    rng = np.random.default_rng(8)
    mx, mg, ps = rng.uniform(0, 3, 4000), rng.uniform(0, 3, 4000), rng.uniform(0, 1, 4000)
    assert np.array_equal(pct.terrain_cost_values(mx, mg, ps, P),
                          oracle.terrain_cost_values(mx, mg, ps, P))


def test_interval_kats():
    P = pct.TravParams()
    g = pct.Layer(np.zeros((1, 5)), 0.1, (0.0, 0.0))
    c = pct.Layer([[0.40, 0.65, 0.55, np.nan, 1.0]], 0.1, (0.0, 0.0))
    out = pct.interval_cost(g, c, P)
    assert out[0, 0] == 50.0 and out[0, 3] == 0.0
    assert out[0, 1] == pytest.approx(0.0, abs=1e-5)
    assert out[0, 2] == pytest.approx(2.0, rel=1e-6)
    out = pct.interval_cost(pct.Layer([[np.nan, 0.0]], 0.1, (0, 0)),
                            pct.Layer([[2.0, 2.0]], 0.1, (0, 0)), P)
    assert out[0, 0] == 50.0 and out[0, 1] == 0.0


def test_inflate_single_barrier_decay():
    kern = pct.build_kernel(0.2, 0.4, 0.1)
    grid = np.zeros((21, 21), np.float32)
    grid[10, 10] = 50.0
    out = pct.inflate(grid, kern)
    assert out[10, 13] == np.float32(np.float32(1 - (0.3 - 0.2) / 0.3) * np.float32(50.0))
    assert out[10, 10] == 50.0 and out[10, 16] == 0.0


def test_unique_cells_matches_oracle(golden):
    G, _, Cost = _slice_inputs(golden)
    from paper_2403_07631_b200.tomogram import Tomogram, TomogramSlice, Layer
    sl = [TomogramSlice(Layer(G[k], 0.1, (0, 0)), Layer(G[k], 0.1, (0, 0)), 0.5 * (k + 1), k,
                        Layer(Cost[k], 0.1, (0, 0))) for k in range(G.shape[0])]
    tom = Tomogram(sl, 0.5, 0.0)
    for k in range(G.shape[0]):
        below = k - 1 if k > 0 else None
        above = k + 1 if k + 1 < G.shape[0] else None
        m = oracle.unique_mask(G, Cost, k, below, above)
        assert pct.unique_cells(tom, k) == set(zip(*[v.tolist() for v in np.nonzero(m)]))
    with pytest.raises(IndexError):
        pct.unique_cells(tom, 99)


def test_simplify_edge_cases():
    from paper_2403_07631_b200.tomogram import Tomogram, TomogramSlice, Layer
    shape = (5, 5)

    def mk(gs, cs):
        return Tomogram([TomogramSlice(Layer(g, 0.1, (0, 0)), Layer(g, 0.1, (0, 0)),
                                       0.5 * (k + 1), k, Layer(c, 0.1, (0, 0)))
                         for k, (g, c) in enumerate(zip(gs, cs))], 0.5, 0.0)
    z = np.zeros(shape, np.float32)
    one = np.ones(shape, np.float32)
    # single slice: unchanged (test_simplify.py:57-61)
    assert len(pct.simplify_tomogram(mk([z], [z])).slices) == 1
    # identical slices collapse to the last one
    out = pct.simplify_tomogram(mk([z, z, z], [one, one, one]))
    assert [s.plane_height for s in out.slices] == [1.5]
    # slope covered above (test_simplify.py:37-51)
    slope = np.tile(np.linspace(0.6, 1.4, 5, dtype=np.float32), (5, 1))
    out = pct.simplify_tomogram(mk([z, slope, slope], [z, one * 2, one * 2]))
    assert [s.plane_height for s in out.slices] == [0.5, 1.5]
    # long removal chains beyond the 32-slice window, checked against the oracle
    rng = np.random.default_rng(3)
    S = 80
    gs = [np.where(rng.uniform(size=shape) < 0.05, np.float32(k // 40), z) for k in range(S)]
    cs = [np.full(shape, 1.0, np.float32) for _ in range(S)]
    G, Cst = np.stack(gs), np.stack(cs)
    keep = oracle.simplify(G, Cst)
    out = pct.simplify_tomogram(mk(gs, cs))
    assert [s.plane_height for s in out.slices] == [0.5 * (k + 1) for k in keep]
    # no cost layer
    t = Tomogram([TomogramSlice(Layer(z, 0.1, (0, 0)), Layer(z, 0.1, (0, 0)), 0.5, 0),
                  TomogramSlice(Layer(z, 0.1, (0, 0)), Layer(z, 0.1, (0, 0)), 1.0, 1)], 0.5, 0.0)
    with pytest.raises(ValueError, match="cost layer"):
        pct.simplify_tomogram(t)


@pytest.mark.parametrize("eps_e", [1e-6, 0.0, -1e-6, 3e-5])
def test_simplify_eps_boundary(eps_e):
    """Elevation differences straddling eps_e at several magnitudes (the
    window kernel's float32 pre-test must defer to the float64 subtraction in
    exactly these cases): surviving slices equal the oracle's."""
    from paper_2403_07631_b200.tomogram import Tomogram, TomogramSlice, Layer
    rng = np.random.default_rng(17)
    shape = (24, 24)
    S = 12
    base = rng.choice(np.array([0.0, 0.37, 3.1, 17.5, 250.0, 4097.0]), size=shape)
    gs, cs = [], []
    for k in range(S):
        # per-cell offsets within a few ulps of +-eps, some exactly representable
        off = eps_e * (1 + rng.integers(-3, 4, size=shape) * 2.0 ** -22) * (k % 3)
        gs.append((base + off).astype(np.float32))
        cs.append(np.ones(shape, np.float32))  # equal costs: elevations decide
    G, Cst = np.stack(gs), np.stack(cs)
    keep = oracle.simplify(G, Cst, eps_e=eps_e)
    tom = Tomogram([TomogramSlice(Layer(g, 0.1, (0, 0)), Layer(g, 0.1, (0, 0)), 0.5 * (k + 1), k,
                                  Layer(c, 0.1, (0, 0))) for k, (g, c) in enumerate(zip(gs, cs))],
                   0.5, 0.0)
    out = pct.simplify_tomogram(tom, eps_e=eps_e)
    assert [s.plane_height for s in out.slices] == [0.5 * (k + 1) for k in keep]


def test_build_errors_and_kats():
    with pytest.raises(ValueError):
        pct.build_tomogram(pct.PointCloud(np.ones((3, 3))), 0.0, 0.1)
    with pytest.raises(pct.GridSizeError):
        pct.build_tomogram(pct.PointCloud(np.array([[0.0, 0, 0], [100.0, 100.0, 1.0]])), 0.5,
                           0.005, max_grid_side=1000)
    # tie at a plane height goes to ground (test_tomogram.py:72-79)
    pts = np.array([[0.0, 0.0, 0.5], [0.02, 0.02, 0.0], [1.0, 1.0, 1.0]])
    tom = pct.build_tomogram(pct.PointCloud(pts), 0.5, 0.1)
    s0 = tom.slices[0]
    i, j = pct.rasterize_index((0.0, 0.0), tom.origin, tom.resolution)
    assert s0.ground.values[i, j] == np.float32(0.5)
    assert not s0.ceiling.valid[i, j]
    # two parallel planes -> six slices with exact heights (test_tomogram.py:57-69)
    xs = np.arange(0.025, 4.0, 0.05)
    gx, gy = np.meshgrid(xs, xs, indexing="ij")
    pts = np.concatenate([np.column_stack([gx.ravel(), gy.ravel(), np.full(gx.size, z)])
                          for z in (0.0, 3.0)])
    tom = pct.build_tomogram(pct.PointCloud(pts), 0.5, 0.1)
    assert len(tom.slices) == 6
    assert [s.plane_height for s in tom.slices] == pytest.approx([0.5, 1.0, 1.5, 2.0, 2.5, 3.0])
    ref = oracle.build(pts, 0.5, 0.1)
    assert np.array_equal(tom.ground_stack(), ref["ground"], equal_nan=True)
    assert np.array_equal(tom.ceiling_stack(), ref["ceiling"], equal_nan=True)


def test_evaluate_accepts_host_tomogram(golden):
    G, Cc, Cost = _slice_inputs(golden)
    from paper_2403_07631_b200.tomogram import Tomogram, TomogramSlice, Layer
    tom = Tomogram([TomogramSlice(Layer(G[k], 0.1, (0, 0)), Layer(Cc[k], 0.1, (0, 0)),
                                  0.5 * (k + 1), k) for k in range(G.shape[0])], 0.5, 0.0)
    ev = pct.evaluate_tomogram(tom, pct.TravParams())
    assert np.array_equal(ev.cost_stack(), Cost)
    # evaluate_slice path
    sl = pct.evaluate_slice(tom.slices[2], pct.TravParams())
    assert np.array_equal(sl.cost.values, Cost[2])


def test_batch_runner_matches_single_maps():
    """evaluate_maps (concurrent contexts, one native call per map) returns the
    same simplified tomograms as the per-map drop-in calls."""
    from paper_2403_07631_b200 import synth
    from paper_2403_07631_b200.batch import evaluate_maps
    clouds = [synth.generate(4, 60_000, 1000 + m) for m in range(12)]
    outs = evaluate_maps(clouds, 0.5, 0.1, pct.TravParams(), workers=4)
    for xyz, got in zip(clouds, outs):
        ev = pct.evaluate_tomogram(pct.build_tomogram(pct.PointCloud(xyz), 0.5, 0.1),
                                   pct.TravParams())
        want = pct.simplify_tomogram(ev)
        assert [s.plane_height for s in got.slices] == [s.plane_height for s in want.slices]
        for a, b in zip(got.slices, want.slices):
            for attr in ("ground", "ceiling", "cost"):
                assert np.array_equal(getattr(a, attr).values.view(np.uint32),
                                      getattr(b, attr).values.view(np.uint32))


def test_batch_of_heterogeneous_maps():
    """One batched native call over maps of very different extents and slice
    counts (a tiny map, a 100+-slice tower, a wide strip, a config-0 map):
    each equals its own per-map drop-in result."""
    from paper_2403_07631_b200 import synth
    from paper_2403_07631_b200.batch import evaluate_maps
    rng = np.random.default_rng(5)
    tower = np.column_stack([rng.uniform(0, 2, 20_000), rng.uniform(0, 2, 20_000),
                             np.floor(rng.uniform(0, 55, 20_000)) + rng.normal(0, 0.02, 20_000)])
    strip = np.column_stack([rng.uniform(0, 60, 30_000), rng.uniform(0, 0.3, 30_000),
                             rng.uniform(0, 2, 30_000)])
    tiny = np.array([[0.0, 0.0, 0.0], [0.05, 0.02, 0.6], [0.1, 0.1, 1.3]])
    clouds = [c.astype(np.float32) for c in (tiny, tower, strip, synth.generate(0, 100_000, 9))]
    outs = evaluate_maps(clouds, 0.5, 0.1, pct.TravParams(), workers=2)
    for xyz, got in zip(clouds, outs):
        ev = pct.evaluate_tomogram(pct.build_tomogram(pct.PointCloud(xyz), 0.5, 0.1),
                                   pct.TravParams())
        want = pct.simplify_tomogram(ev)
        assert [s.plane_height for s in got.slices] == [s.plane_height for s in want.slices]
        for a, b in zip(got.slices, want.slices):
            for attr in ("ground", "ceiling", "cost"):
                assert np.array_equal(getattr(a, attr).values.view(np.uint32),
                                      getattr(b, attr).values.view(np.uint32))


def test_stream_maps_matches_single_maps():
    """stream_maps (maps in flight on two contexts, layers read back in the
    worker) yields, in order, the per-map drop-in results."""
    from paper_2403_07631_b200 import synth
    from paper_2403_07631_b200.batch import stream_maps
    clouds = [synth.generate(4, 60_000, 2000 + m) for m in range(7)]
    clouds[3] = clouds[3].astype(np.float64)
    outs = list(stream_maps(clouds, 0.5, 0.1, pct.TravParams(), workers=2))
    assert len(outs) == len(clouds)
    for xyz, got in zip(clouds, outs):
        ev = pct.evaluate_tomogram(pct.build_tomogram(pct.PointCloud(xyz), 0.5, 0.1),
                                   pct.TravParams())
        want = pct.simplify_tomogram(ev)
        assert [s.plane_height for s in got.slices] == [s.plane_height for s in want.slices]
        for a, b in zip(got.slices, want.slices):
            for attr in ("ground", "ceiling", "cost"):
                la = getattr(a, attr)  # already on the host
                assert la._values is not None or la._k in la._stack._host
                assert np.array_equal(getattr(a, attr).values.view(np.uint32),
                                      getattr(b, attr).values.view(np.uint32))


def test_concurrent_contexts_with_different_parameters():
    """Contexts running at the same time with different TravParams / kernels
    (the __constant__ banks are shared per device) each get their own
    results."""
    import threading
    from paper_2403_07631_b200 import synth
    from paper_2403_07631_b200.batch import BatchRunner, stream_maps
    xyz = synth.generate(4, 80_000, 3000)
    variants = [(pct.TravParams(), 0.1), (pct.TravParams(theta_b=0.9, d_inf=0.25), 0.1),
                (pct.TravParams(c_barrier=30.0), 0.2)]

    def want(params, r_g):
        ev = pct.evaluate_tomogram(pct.build_tomogram(pct.PointCloud(xyz), 0.5, r_g), params)
        return [s.cost.values.copy() for s in pct.simplify_tomogram(ev, c_barrier=params.c_barrier).slices]

    expected = [want(p, r) for p, r in variants]
    got = [[] for _ in variants]

    def worker(i):
        p, r = variants[i]
        run = BatchRunner(0, workers=2)
        for t in stream_maps([xyz] * 6, 0.5, r, p, runner=run, c_barrier=p.c_barrier):
            got[i].append([s.cost.values.copy() for s in t.slices])
        run.close()

    ths = [threading.Thread(target=worker, args=(i,)) for i in range(len(variants))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    for i in range(len(variants)):
        assert len(got[i]) == 6
        for res in got[i]:
            assert len(res) == len(expected[i])
            for a, b in zip(res, expected[i]):
                assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), i


@pytest.mark.parametrize("name", ["ref_random_multilayer_s9", "ref_spiral_s3", "synth_cfg0",
                                  "synth_cfg1"])
def test_lga_archives_byte_identical(golden, tmp_path, name):
    """save_tomogram streams device layers into the archive: the files of the
    built, evaluated and simplified tomograms equal the reference's bytes."""
    import hashlib
    case = golden["cases"][name]
    tom, ev, simp = _run(case_input(name, case), case["d_s"], case["r_g"])
    for key, t in (("built", tom), ("evaluated", ev), ("simplified", simp)):
        f = tmp_path / f"{key}.lga"
        pct.save_tomogram(t, f)
        b = f.read_bytes()
        assert len(b) == case["lga"][key]["bytes"]
        assert hashlib.sha256(b).hexdigest() == case["lga"][key]["sha256"], key
        back = pct.load_tomogram(f)
        g = tmp_path / f"{key}2.lga"
        pct.save_tomogram(back, g)
        assert g.read_bytes() == b


def test_load_tomogram_errors(tmp_path):
    f = tmp_path / "junk.lga"
    f.write_bytes(b"not an archive at all")
    with pytest.raises(ValueError, match="not an LGA archive"):
        pct.load_tomogram(f)


@pytest.mark.parametrize("name", ["ref_random_multilayer_s9", "ref_spiral_s3", "synth_cfg0",
                                  "synth_cfg1"])
def test_planner_context_matches_reference(golden, name):
    """GPU canonical-node arrays == the reference planner's (planner.py:65-93)."""
    from paper_2403_07631_b200.planner_ctx import attach_planner_context
    case = golden["cases"][name]
    _, ev, simp = _run(case_input(name, case), case["d_s"], case["r_g"])
    for key, t in (("evaluated", ev), ("simplified", simp)):
        pc = attach_planner_context(t)
        assert t._planner_ctx is pc and pc.eps_e == 1e-6 and pc.c_barrier == 50.0
        assert digest(pc.canon) == case["planner"][key]["canon_sha256"], key
        assert digest(pc.cn) == case["planner"][key]["cn_sha256"], key


@pytest.mark.parametrize("name,skip", [("synth_cfg1", "1"), ("synth_cfg2_n2000000", "0"),
                                       ("ref_random_multilayer_s9", "1")])
def test_bnb_tile_skipping_is_exact(golden, monkeypatch, name, skip):
    """Skipping unchanged tiles (walk change map; default for R >= 8) and not
    skipping give the reference's cost bytes either way."""
    monkeypatch.setenv("PCT_BNB_SKIP", skip)
    case = golden["cases"][name]
    tom = pct.build_tomogram(pct.PointCloud(case_input(name, case)), case["d_s"], case["r_g"])
    cost = pct.evaluate_tomogram(tom, pct.TravParams()).cost_stack()
    for k in range(cost.shape[0]):
        assert digest(cost[k]) == case["cost_slice_sha256"][k], f"cost slice {k}"


def _np_masks(stack):
    """bit k: slice k differs (bitwise) from slice k-1; bit 0 set."""
    u = np.ascontiguousarray(stack).view(np.uint32)
    m = np.ones(u.shape[1:], np.uint64)
    for k in range(1, u.shape[0]):
        m |= (u[k] != u[k - 1]).astype(np.uint64) << np.uint64(k)
    return m


@pytest.mark.parametrize("mode", ["atomic", "hist", "tiled"])
def test_build_slice_change_masks(monkeypatch, mode):
    """The build's per-cell slice-change masks (read by the terrain walk in
    place of a pass over the stacks) equal the masks of its own layers."""
    from paper_2403_07631_b200 import _lib, synth
    monkeypatch.setenv("PCT_BUILD", mode)
    xyz = synth.two_storey(120_000, seed=3)
    tom = pct.build_tomogram(pct.PointCloud(xyz), 0.5, 0.1)
    g, c = tom.ground_stack(), tom.ceiling_stack()
    owner = tom.slices[0].ground.device[0].owner
    ptr = owner.ctx.lib.pct_tomo_masks(owner.handle)
    if mode == "tiled":  # the hash-merged tile build does not emit them
        assert not ptr
        return
    assert ptr
    cells = g.shape[1] * g.shape[2]
    host = np.empty(2 * cells, np.uint64)
    owner.ctx.check(owner.ctx.lib.pct_memcpy_d2h(owner.ctx.h, host.ctypes.data, ptr, host.nbytes))
    assert np.array_equal(host[:cells].reshape(g.shape[1:]), _np_masks(g))
    assert np.array_equal(host[cells:].reshape(g.shape[1:]), _np_masks(c))
    # the evaluation with and without them is identical
    ev = pct.evaluate_tomogram(tom, pct.TravParams())
    from paper_2403_07631_b200.tomogram import Layer, Tomogram, TomogramSlice
    host_tom = Tomogram([TomogramSlice(Layer(g[k], 0.1, tom.origin), Layer(c[k], 0.1, tom.origin),
                                       s.plane_height, k) for k, s in enumerate(tom.slices)],
                        tom.d_s, tom.z_min)
    ev2 = pct.evaluate_tomogram(host_tom, pct.TravParams())
    assert np.array_equal(ev.cost_stack().view(np.uint32), ev2.cost_stack().view(np.uint32))


@pytest.mark.parametrize("win_skip", ["1", "0"])
def test_fused_run_simplify_matches_oracle(monkeypatch, win_skip):
    """pct_tomo_run (build -> evaluate -> simplify on one device tomogram):
    its simplify window reads only where the build's ground masks and the
    evaluation's per-tile cost masks say values change (PCT_WIN_SKIP=1, the
    default) -- the surviving slices equal the oracle's, as with the full
    window (PCT_WIN_SKIP=0)."""
    from paper_2403_07631_b200 import synth
    from paper_2403_07631_b200.batch import stream_maps
    monkeypatch.setenv("PCT_WIN_SKIP", win_skip)
    rng = np.random.default_rng(17)
    clouds = [synth.generate(4, 80_000, 3000 + m) for m in range(3)]
    clouds.append(synth.spiral_ramp(400_000, seed=9))
    # stacked floors with small height differences around eps_e and equal costs
    n = 60_000
    pts = []
    for lvl, dz in enumerate((0.0, 2.0, 2.0 + 5e-7, 4.0, 4.0 + 2e-6)):
        x, y = rng.uniform(0, 15, n), rng.uniform(0, 12, n)
        pts.append(np.column_stack([x, y, np.full(n, dz) + (x > 7) * 0.3]))
    clouds.append(np.concatenate(pts).astype(np.float32))
    d_s = [0.5, 0.5, 0.5, 0.4, 0.25]
    for xyz, ds in zip(clouds, d_s):
        got = next(stream_maps([xyz], ds, 0.1, pct.TravParams(), workers=1))
        ref = oracle.build(xyz, ds, 0.1)
        cost = oracle.evaluate(ref["ground"], ref["ceiling"], 0.1, TABLE_PARAMS)
        keep = oracle.simplify(ref["ground"], cost)
        assert [s.plane_height for s in got.slices] == [float(ref["heights"][k]) for k in keep]


@pytest.mark.parametrize("sparse,run", [("1", "1"), ("1", "3"), ("1", "64"), ("0", "7")])
@pytest.mark.parametrize("name", ["synth_cfg0", "ref_spiral_s3", "synth_two_storey_small"])
def test_sparse_walk_and_bnb_runs(golden, monkeypatch, name, sparse, run):
    """The walk's sparse output (only recomputed slices + run starts written,
    the inflation kernel merging the rest) at several item run lengths,
    through the fused path and the per-stack path: costs equal the
    reference's."""
    monkeypatch.setenv("PCT_WALK_SPARSE", sparse)
    monkeypatch.setenv("PCT_INFL_RUN", run)
    case = golden["cases"][name]
    xyz = case_input(name, case)
    ev = pct.evaluate_tomogram(pct.build_tomogram(pct.PointCloud(xyz), case["d_s"], case["r_g"]),
                               pct.TravParams())
    assert [digest(s.cost.values) for s in ev.slices] == case["cost_slice_sha256"]
    from paper_2403_07631_b200.batch import stream_maps
    got = next(stream_maps([xyz], case["d_s"], case["r_g"], pct.TravParams(), workers=1))
    assert [s.plane_height for s in got.slices] == [case["heights"][k] for k in case["keep"]]
    assert [digest(s.cost.values) for s in got.slices] == \
        [case["cost_slice_sha256"][k] for k in case["keep"]]


@pytest.mark.parametrize("env", [{"PCT_BUILD_REDUCE": "2"}, {"PCT_BUILD_REDUCE": "3"},
                                 {"PCT_BUILD_TMA": "1"}, {"PCT_HIST_BULK": "0"}])
@pytest.mark.parametrize("name", ["synth_cfg0", "ref_random_multilayer_s9", "synth_cfg2_n2000000"])
def test_hist_build_variants_match_reference_golden(golden, monkeypatch, name, env):
    """The opt-in histogram-build variants (split-scan reduce, one-pass
    1024-thread reduce, TMA box stores of the layers, direct point loads
    instead of bulk-copy staging) give the reference's layers and the same
    slice-change masks as the default reduce."""
    monkeypatch.setenv("PCT_BUILD", "hist")
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    case = golden["cases"][name]
    xyz = case_input(name, case)
    tom = pct.build_tomogram(pct.PointCloud(xyz), case["d_s"], case["r_g"])
    g, c = tom.ground_stack(), tom.ceiling_stack()
    for k in range(g.shape[0]):
        assert digest(g[k]) == case["ground_slice_sha256"][k], f"ground slice {k}"
        assert digest(c[k]) == case["ceiling_slice_sha256"][k], f"ceiling slice {k}"
    owner = tom.slices[0].ground.device[0].owner
    ptr = owner.ctx.lib.pct_tomo_masks(owner.handle)
    if ptr and g.shape[0] <= 64:  # the variants emit the same slice-change masks
        cells = g.shape[1] * g.shape[2]
        host = np.empty(2 * cells, np.uint64)
        owner.ctx.check(owner.ctx.lib.pct_memcpy_d2h(owner.ctx.h, host.ctypes.data, ptr,
                                                     host.nbytes))
        assert np.array_equal(host[:cells].reshape(g.shape[1:]), _np_masks(g))
        assert np.array_equal(host[cells:].reshape(g.shape[1:]), _np_masks(c))


@pytest.mark.parametrize("env", [{"PCT_BNB_DYNAMIC": "0"}, {"PCT_WIN_DYNAMIC": "0"},
                                 {"PCT_BNB_DYNAMIC": "0", "PCT_WIN_DYNAMIC": "0"}])
def test_dynamic_work_claims_match_static(golden, monkeypatch, env):
    """The inflation kernel's dynamic item claims and the simplify window's
    dynamic cell-group claims (the defaults) against their static round-robin
    schedules: the same costs (the reference's) and the same surviving slices,
    on a map large enough for the segment window (> 1M cells)."""
    from paper_2403_07631_b200.batch import stream_maps
    name = "synth_cfg2_n2000000"
    case = golden["cases"][name]
    xyz = case_input(name, case)

    def run():
        ev = pct.evaluate_tomogram(
            pct.build_tomogram(pct.PointCloud(xyz), case["d_s"], case["r_g"]), pct.TravParams())
        got = next(stream_maps([xyz], case["d_s"], case["r_g"], pct.TravParams(), workers=1))
        return ([digest(s.cost.values) for s in ev.slices], [s.plane_height for s in got.slices],
                [digest(s.cost.values) for s in got.slices])

    dyn = run()
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    assert run() == dyn
    assert dyn[0] == case["cost_slice_sha256"]
    assert dyn[1] == [case["heights"][k] for k in case["keep"]]


@pytest.mark.parametrize("offset", [0.0, 12.37, -731.9, 5.0e5])
def test_partitioned_builds_at_cell_borders(monkeypatch, offset):
    """Every build against the oracle on float32 points placed within a few
    ulps of cell borders (v = v0 + (i + 0.5) r_g) and of the plane heights,
    at small and large coordinates (5e5: the float32 grid is 3 cm).  (A
    float32 cell path with a float64 fallback near borders was measured in
    the histogram passes: correct here, but slower -- DESIGN 9.1.)"""
    rng = np.random.default_rng(int(abs(offset)) + 7)
    r_g, d_s = 0.1, 0.5
    x0, y0, z0 = np.float32(offset), np.float32(offset * 0.5 - 3.3), np.float32(offset * 0.01)
    n_i, n_j = 40, 60
    pts = []
    for i in range(n_i):
        for j in range(0, n_j, 3):
            for d in (-2, -1, 0, 1, 2):
                bx = np.float32(np.float64(x0) + (j + 0.5) * r_g)
                by = np.float32(np.float64(y0) + (i + 0.5) * r_g)
                x = bx
                y = by
                for _ in range(abs(d)):
                    x = np.nextafter(x, np.float32(np.inf if d > 0 else -np.inf))
                    y = np.nextafter(y, np.float32(np.inf if d > 0 else -np.inf))
                k = int(rng.integers(0, 6))
                h = np.float32(np.float64(z0) + d_s * (k + 1))
                for dz in (-1, 0, 1):
                    z = h if dz == 0 else np.nextafter(h, np.float32(np.inf * dz))
                    pts.append((x, y, z))
    pts = np.array(pts, np.float32)
    extra = np.column_stack([x0 + rng.uniform(0, n_j * r_g, 20_000),
                             y0 + rng.uniform(0, n_i * r_g, 20_000),
                             z0 + rng.uniform(0, 3.2, 20_000)]).astype(np.float32)
    corner = np.array([[x0, y0, z0]], np.float32)
    xyz = np.concatenate([corner, pts, extra])
    xyz = xyz[rng.permutation(len(xyz))]
    ref = oracle.build(xyz, d_s, r_g)
    for build in ("atomic", "tiled", "hist"):
        monkeypatch.setenv("PCT_BUILD", build)
        tom = pct.build_tomogram(pct.PointCloud(xyz), d_s, r_g)
        _assert_layers_equal(tom.ground_stack(), ref["ground"], f"ground {build}")
        _assert_layers_equal(tom.ceiling_stack(), ref["ceiling"], f"ceiling {build}")


def test_simplify_uses_change_masks_and_matches(golden):
    """The drop-in chain's simplify reads only where values change (the
    build's ground masks + the evaluation's tile masks, pct_simplify_masked)
    and keeps the same slices as the unmasked sweep and the reference."""
    from paper_2403_07631_b200 import simplify as simp_mod
    name = "synth_cfg2_n2000000"
    case = golden["cases"][name]
    xyz = case_input(name, case)
    ev = pct.evaluate_tomogram(pct.build_tomogram(pct.PointCloud(xyz), case["d_s"], case["r_g"]),
                               pct.TravParams())
    info = simp_mod._change_info(list(ev.slices))
    assert info is not None and int(info["geom"][0]) > 0
    got = [s.plane_height for s in pct.simplify_tomogram(ev).slices]
    # the same sweep without the masks: a cost layer replaced on the host
    # (same values) breaks the device run, so the plain path runs
    ev2 = pct.evaluate_tomogram(pct.build_tomogram(pct.PointCloud(xyz), case["d_s"], case["r_g"]),
                                pct.TravParams())
    ev2.slices[0].cost.values = ev2.slices[0].cost.values.copy()
    assert simp_mod._change_info(list(ev2.slices)) is None
    want = [s.plane_height for s in pct.simplify_tomogram(ev2).slices]
    assert got == want == [case["heights"][k] for k in case["keep"]]
