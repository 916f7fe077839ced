"""CPU checks of the per-cell arithmetic the kernels execute (csrc/cellmath.cuh,
host build lib/libpct_hostmath.so) against numpy / the oracle."""

import ctypes as C
from pathlib import Path

import numpy as np
import pytest

import oracle
from golden_util import TABLE_PARAMS, case_arrays

ROOT = Path(__file__).resolve().parent.parent
HOSTLIB = ROOT / "paper_2403_07631_b200" / "lib" / "libpct_hostmath.so"


@pytest.fixture(scope="module")
def hm():
    import __graft_entry__
    __graft_entry__.build()  # incremental
    lib = C.CDLL(str(HOSTLIB))
    P = C.c_void_p
    lib.pcth_hypot.argtypes = [P, P, C.c_int64, P]
    lib.pcth_div_const.argtypes = [P, C.c_int64, C.c_double, P]
    lib.pcth_cinit.argtypes = [P, P, C.c_int, C.c_int, C.c_double, P, C.c_int, C.c_int, P]
    lib.pcth_fast_cells.argtypes = [P, P, C.c_int64, C.c_double, P, P, P]
    lib.pcth_fast_cells.restype = C.c_int64
    lib.pcth_ref_cells.argtypes = [P, P, C.c_int64, C.c_double, P, P, P]
    return lib


def _hypot(hm, x, y):
    out = np.empty_like(x)
    hm.pcth_hypot(x.ctypes.data, y.ctypes.data, x.size, out.ctypes.data)
    return out


def test_glibc_hypot_restatement_matches_numpy(hm):
    rng = np.random.default_rng(1)
    n = 2_000_000
    # gradient-like inputs: differences of float32 values over r_g, 2 r_g
    a = rng.uniform(-5, 5, (3, n)).astype(np.float32).astype(np.float64)
    x = (a[0] - a[1]) / 0.2
    y = (a[2] - a[0]) / 0.1
    assert np.array_equal(_hypot(hm, x, y), np.hypot(x, y))
    # wide dynamic range and edge cases
    x = rng.standard_normal(n) * 10.0 ** rng.integers(-300, 300, n)
    y = rng.standard_normal(n) * 10.0 ** rng.integers(-300, 300, n)
    x[:10] = 0.0
    y[5:15] = 0.0
    assert np.array_equal(_hypot(hm, x, y), np.hypot(x, y))


@pytest.mark.parametrize("d", [0.2, 0.1, 0.05, 0.36, 1.7, 0.4, 0.10000000149011612])
def test_markstein_division_is_correctly_rounded(hm, d):
    rng = np.random.default_rng(2)
    n = 2_000_000
    a = rng.uniform(-20, 20, (2, n)).astype(np.float32).astype(np.float64)
    num = np.concatenate([a[0] - a[1], rng.uniform(0, 3, n), [0.0, -0.0]])
    out = np.empty_like(num)
    hm.pcth_div_const(num.ctypes.data, num.size, d, out.ctypes.data)
    assert np.array_equal(out, num / d)


def _cinit_oracle(G, Cc, r_g, p):
    ci = oracle.interval_cost(G, Cc, p)
    cg = oracle.ground_cost(G, r_g, p)
    return oracle.fuse_costs(ci, cg, np.isfinite(G), p)


def _ps_min_count(theta_p, r):
    side = 2 * r + 1
    for c in range(side * side + 1):
        if c / float(side * side) > theta_p:
            return c
    return side * side + 1


def _cinit_host(hm, G, Cc, r_g, p):
    G = np.ascontiguousarray(G, np.float32)
    Cc = np.ascontiguousarray(Cc, np.float32)
    pv = np.array([p.d_min, p.d_ref, p.theta_b, p.theta_s, p.theta_p, p.c_barrier, p.alpha_d,
                   p.alpha_b, p.alpha_s])
    r = oracle.traversability.patch_radius(p, r_g)
    out = np.empty_like(G)
    hm.pcth_cinit(G.ctypes.data, Cc.ctypes.data, G.shape[0], G.shape[1], r_g, pv.ctypes.data, r,
                  _ps_min_count(p.theta_p, r), out.ctypes.data)
    return out


@pytest.mark.parametrize("name", ["ref_random_multilayer_s9", "synth_two_storey_small"])
def test_cinit_composition_matches_oracle(hm, golden, name):
    arr = case_arrays(golden["cases"][name])
    for k in range(arr["ground"].shape[0]):
        G, Cc = arr["ground"][k], arr["ceiling"][k]
        assert np.array_equal(_cinit_host(hm, G, Cc, 0.1, TABLE_PARAMS),
                              _cinit_oracle(G, Cc, 0.1, TABLE_PARAMS))


def _cells(hm, fn, cross, ceil, r_g):
    P = TABLE_PARAMS
    pv = np.array([P.d_min, P.d_ref, P.theta_b, P.theta_s, P.theta_p, P.c_barrier, P.alpha_d,
                   P.alpha_b, P.alpha_s])
    enc = np.empty(len(ceil), np.float32)
    gen = np.empty(len(ceil), np.uint8)
    r = fn(cross.ctypes.data, ceil.ctypes.data, len(ceil), C.c_double(r_g), pv.ctypes.data,
           enc.ctypes.data, gen.ctypes.data)
    return enc, gen, r


@pytest.mark.parametrize("r_g", [0.1, 0.05, 0.2])
def test_fast_guarded_path_equals_reference_path(hm, r_g):
    """eval_fast_kernel's per-cell arithmetic (sqrt + guard instead of the
    exact glibc hypot) must equal the reference-order path on every cell,
    including cells steered into the theta_s guard band."""
    hm.pcth_fast_cells.restype = C.c_int64
    rng = np.random.default_rng(11)
    n = 3_000_000
    e = rng.uniform(0, 3, n).astype(np.float32)
    scale = np.float32(r_g) * rng.choice(np.array([0.02, 0.2, 0.5, 1.0, 3.0], np.float32), n)
    cross = np.stack([e] + [e + (rng.standard_normal(n).astype(np.float32) * scale)
                            for _ in range(4)], axis=1).astype(np.float32)
    # exact slope theta_s along x on a share of the cells: lands in the guard band
    k = n // 10
    cross[:k, 2] = (cross[:k, 0].astype(np.float64) + 0.36 * r_g).astype(np.float32)
    cross[:k, 1] = np.nan
    cross[:k, 3] = cross[:k, 0]
    cross[:k, 4] = np.nan
    holes = rng.uniform(size=cross.shape) < 0.05
    cross[holes] = np.nan
    ceil = (e + rng.uniform(0.3, 2.0, n)).astype(np.float32)
    ceil[rng.uniform(size=n) < 0.3] = np.nan
    cross = np.ascontiguousarray(cross)
    f_enc, f_gen, exact = _cells(hm, hm.pcth_fast_cells, cross, ceil, r_g)
    r_enc, r_gen, _ = _cells(hm, hm.pcth_ref_cells, cross, ceil, r_g)
    assert np.array_equal(f_gen, r_gen)
    assert np.array_equal(f_enc.view(np.uint32), r_enc.view(np.uint32))
    assert exact > 0  # the guard paths were exercised


def test_cinit_random_rough_terrain(hm):
    """Steep, noisy, holey surfaces exercise every branch (barrier, gentle,
    foothold pass/fail, isolated, one-sided gradients)."""
    rng = np.random.default_rng(7)
    for r_g in (0.1, 0.05, 0.2):
        G = (np.cumsum(rng.normal(0, 0.08, (90, 70)), axis=1)).astype(np.float32)
        G[rng.uniform(size=G.shape) < 0.15] = np.nan
        Cc = (G + rng.uniform(0.3, 1.0, G.shape)).astype(np.float32)
        Cc[rng.uniform(size=G.shape) < 0.3] = np.nan
        assert np.array_equal(_cinit_host(hm, G, Cc, r_g, TABLE_PARAMS),
                              _cinit_oracle(G, Cc, r_g, TABLE_PARAMS))
