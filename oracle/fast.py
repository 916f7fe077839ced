"""Multi-threaded C oracle (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

ctypes front end of ``oracle/c/pct_oracle.c``: the same restatement of
tomogram.py:127-213, traversability.py:59-236 and simplify.py:18-73 as the
numpy modules next to it, in C with a pthread pool, so full-size maps (the
200M-point config 3) can be checked and timed on the host in seconds.  It is
pinned to the same golden fixtures as the numpy oracle
(tests/test_oracle_golden.py) and to the numpy oracle itself.

Built by ``make -C oracle`` (``__graft_entry__.build()`` runs it) into
``oracle/lib/liboracle_c.so``.  Same call signatures and return values as
``oracle.build`` / ``oracle.evaluate`` / ``oracle.simplify`` plus ``threads``
(default: every host thread).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

from .tomography import GRID_SIDE_LIMIT, frame
from .traversability import kernel_weights, patch_radius

HERE = Path(__file__).resolve().parent
LIB = HERE / "lib" / "liboracle_c.so"
SRC = HERE / "c" / "pct_oracle.c"

_lib = None


class _Params(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("d_min", "d_ref", "theta_b", "theta_s", "theta_p",
                                          "c_barrier", "alpha_d", "alpha_b", "alpha_s")] + \
               [("patch_radius", C.c_int32), ("pad_", C.c_int32)]


def build_lib(force: bool = False) -> Path:
    """Compile the C oracle (gcc, no fast-math, no FMA contraction)."""
    if force or not LIB.exists() or LIB.stat().st_mtime < SRC.stat().st_mtime:
        subprocess.run(["make", "-s"] + (["-B"] if force else []) + ["-C", str(HERE)], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build_lib()
        L = C.CDLL(str(LIB))
        p, i64, i32, d = C.c_void_p, C.c_int64, C.c_int, C.c_double
        L.orc_bounds.argtypes = [p, i64, i32, i32, p, p]
        L.orc_bounds.restype = i32
        L.orc_build.argtypes = [p, i64, i32, d, d, d, i64, i64, p, i32, p, p, i32]
        L.orc_build.restype = i64
        L.orc_evaluate.argtypes = [p, p, i32, i64, i64, d, p, p, i32, p, i32]
        L.orc_evaluate.restype = i32
        L.orc_unique_any.argtypes = [p, p, i64, i32, i32, i32, d, d, i32]
        L.orc_unique_any.restype = i32
        L.orc_simplify.argtypes = [p, p, i32, i64, d, d, p, i32]
        L.orc_simplify.restype = i32
        _lib = L
    return _lib


def _threads(threads):
    return int(threads) if threads else (os.cpu_count() or 1)


def _points(xyz):
    a = np.asarray(xyz)
    if a.dtype not in (np.float32, np.float64):
        a = a.astype(np.float64)
    a = np.ascontiguousarray(a)
    if a.ndim != 2 or a.shape[1] != 3:
        raise ValueError(f"expected (N, 3) point array, got shape {a.shape}")
    return a, int(a.dtype == np.float64)


def bounds(xyz, threads=None):
    """Exact float64 (min, max) corners (cloud_io.py:47-50)."""
    a, f64 = _points(xyz)
    lo, hi = np.empty(3), np.empty(3)
    if lib().orc_bounds(a.ctypes.data, a.shape[0], f64, _threads(threads), lo.ctypes.data,
                        hi.ctypes.data) != 0:
        raise ValueError("zero valid points")
    return lo, hi


def build(xyz, d_s, r_g, max_grid_side=GRID_SIDE_LIMIT, threads=None):
    """Same result as ``oracle.build`` (tomogram.py:127-213)."""
    a, f64 = _points(xyz)
    lo, hi = bounds(a, threads)
    fr = frame(lo, hi, d_s, r_g, max_grid_side)
    rows, cols, heights = fr["rows"], fr["cols"], np.ascontiguousarray(fr["heights"])
    S = heights.shape[0]
    ground = np.empty((S, rows, cols), np.float32)
    ceiling = np.empty((S, rows, cols), np.float32)
    bad = lib().orc_build(a.ctypes.data, a.shape[0], f64, fr["origin"][0], fr["origin"][1],
                          float(r_g), rows, cols, heights.ctypes.data, S, ground.ctypes.data,
                          ceiling.ctypes.data, _threads(threads))
    if bad:
        raise RuntimeError(f"{bad} points fell outside the grid")
    return dict(ground=ground, ceiling=ceiling, heights=heights, origin=fr["origin"],
                rows=rows, cols=cols, z_min=fr["z_min"], d_s=float(d_s), r_g=float(r_g))


def _params(params, r_g):
    return _Params(float(params.d_min), float(params.d_ref), float(params.theta_b),
                   float(params.theta_s), float(params.theta_p), float(params.c_barrier),
                   float(params.alpha_d), float(params.alpha_b), float(params.alpha_s),
                   patch_radius(params, r_g), 0)


def evaluate(ground, ceiling, r_g, params, threads=None, w=None):
    """Same result as ``oracle.evaluate`` (traversability.py:216-236)."""
    g = np.ascontiguousarray(ground, np.float32)
    c = np.ascontiguousarray(ceiling, np.float32)
    if g.shape != c.shape:
        raise ValueError("ground and ceiling layers are misaligned")
    if w is None:
        w = kernel_weights(params.d_inf, params.d_sm, r_g)
    w = np.ascontiguousarray(w, np.float32)
    S, rows, cols = g.shape
    out = np.empty_like(g)
    pc = _params(params, r_g)
    if lib().orc_evaluate(g.ctypes.data, c.ctypes.data, S, rows, cols, float(r_g), C.byref(pc),
                          w.ctypes.data, w.shape[0], out.ctypes.data, _threads(threads)) != 0:
        raise MemoryError("oracle evaluate scratch")
    return out


def unique_any(ground, cost, k, below, above, eps_e=1e-6, c_barrier=50.0, threads=None):
    g = np.ascontiguousarray(ground, np.float32)
    c = np.ascontiguousarray(cost, np.float32)
    n = g.shape[1] * g.shape[2]
    return bool(lib().orc_unique_any(g.ctypes.data, c.ctypes.data, n, int(k),
                                     -1 if below is None else int(below),
                                     -1 if above is None else int(above), float(eps_e),
                                     float(c_barrier), _threads(threads)))


def simplify(ground, cost, eps_e=1e-6, c_barrier=50.0, threads=None):
    """Surviving slice indices (simplify.py:56-73), like ``oracle.simplify``."""
    g = np.ascontiguousarray(ground, np.float32)
    c = np.ascontiguousarray(cost, np.float32)
    S = g.shape[0]
    keep = np.empty(max(S, 1), np.int32)
    n = lib().orc_simplify(g.ctypes.data, c.ctypes.data, S, g.shape[1] * g.shape[2],
                           float(eps_e), float(c_barrier), keep.ctypes.data, _threads(threads))
    return [int(k) for k in keep[:n]]


def pipeline(xyz, d_s, r_g, params, eps_e=1e-6, c_barrier=50.0, threads=None):
    """build -> evaluate -> simplify; returns (build dict, cost stack, keep)."""
    t = build(xyz, d_s, r_g, threads=threads)
    cost = evaluate(t["ground"], t["ceiling"], r_g, params, threads=threads)
    keep = simplify(t["ground"], cost, eps_e, c_barrier, threads=threads)
    return t, cost, keep
