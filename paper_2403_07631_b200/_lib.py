"""ctypes binding of libpct.so (include/pct.h) and the per-device contexts.

There is no CPU fallback: importing the hot-path functions works anywhere,
but every call that computes needs libpct.so and a CUDA device and raises
RuntimeError otherwise.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libpct.so"

PCT_OK = 0
PCT_E_INVALID = -1
PCT_E_GRID = -2
PCT_E_CUDA = -3
PCT_E_NOMEM = -4
PCT_E_EMPTY = -5
PCT_E_NONFINITE = -6
PCT_E_NOCOST = -7
PCT_E_RANGE = -8
PCT_E_IO = -9
PCT_F32, PCT_F64 = 0, 1
LAYER_GROUND, LAYER_CEILING, LAYER_COST = 0, 1, 2


class TravParamsC(C.Structure):
    _fields_ = [("d_min", C.c_double), ("d_ref", C.c_double), ("theta_b", C.c_double),
                ("theta_s", C.c_double), ("theta_p", C.c_double), ("c_barrier", C.c_double),
                ("alpha_d", C.c_double), ("alpha_b", C.c_double), ("alpha_s", C.c_double),
                ("patch_radius", C.c_int32), ("_pad", C.c_int32)]


class FrameC(C.Structure):
    _fields_ = [("origin_x", C.c_double), ("origin_y", C.c_double), ("z_min", C.c_double),
                ("d_s", C.c_double), ("r_g", C.c_double), ("rows", C.c_int32),
                ("cols", C.c_int32), ("n_slices", C.c_int32), ("_pad", C.c_int32)]


_vp = C.c_void_p
_i32, _i64, _d = C.c_int32, C.c_int64, C.c_double
_SIGS = {
    "pct_abi_version": ([], C.c_int),
    "pct_ctx_create": ([C.c_int, C.POINTER(_vp)], C.c_int),
    "pct_ctx_destroy": ([_vp], C.c_int),
    "pct_last_error": ([_vp], C.c_char_p),
    "pct_sync": ([_vp], C.c_int),
    "pct_launch_count": ([_vp], C.c_int64),
    "pct_set_stream": ([_vp, _vp], C.c_int),
    "pct_malloc": ([_vp, C.c_size_t, C.POINTER(_vp)], C.c_int),
    "pct_free": ([_vp, _vp], C.c_int),
    "pct_host_alloc": ([_vp, C.c_size_t, C.POINTER(_vp)], C.c_int),
    "pct_host_free": ([_vp, _vp], C.c_int),
    "pct_host_register": ([_vp, _vp, C.c_size_t], C.c_int),
    "pct_host_unregister": ([_vp, _vp], C.c_int),
    "pct_memcpy_h2d": ([_vp, _vp, _vp, C.c_size_t], C.c_int),
    "pct_memcpy_d2h": ([_vp, _vp, _vp, C.c_size_t], C.c_int),
    "pct_memcpy_d2h_async": ([_vp, _vp, _vp, C.c_size_t], C.c_int),
    "pct_bounds": ([_vp, _vp, _i64, C.c_int, _vp, _vp], C.c_int),
    "pct_frame_compute": ([_vp, _vp, _d, _d, _i64, C.POINTER(FrameC), _vp, _i32], C.c_int),
    "pct_build": ([_vp, _vp, _i64, C.c_int, C.POINTER(FrameC), _vp, _vp, _vp], C.c_int),
    "pct_evaluate": ([_vp, _vp, _vp, _i32, _i32, _i32, _d, C.POINTER(TravParamsC), _vp, _i32,
                      _vp], C.c_int),
    "pct_evaluate_masked": ([_vp, _vp, _vp, _i32, _i32, _i32, _d, C.POINTER(TravParamsC), _vp,
                             _i32, _vp, _vp], C.c_int),
    "pct_tomo_masks": ([_vp], _vp),
    "pct_tile_masks_bytes": ([_i32, _i32], C.c_int64),
    "pct_evaluate_tiles": ([_vp, _vp, _vp, _i32, _i32, _i32, _d, C.POINTER(TravParamsC), _vp,
                            _i32, _vp, _vp, _vp, _vp], C.c_int),
    "pct_simplify_masked": ([_vp, _vp, _vp, _i32, _i32, _i32, _d, _d, _vp, _vp, _vp, _vp, _vp],
                            C.c_int),
    "pct_interval_cost": ([_vp, _vp, _vp, _i32, _i32, C.POINTER(TravParamsC), _vp], C.c_int),
    "pct_ground_cost": ([_vp, _vp, _i32, _i32, _d, C.POINTER(TravParamsC), _vp], C.c_int),
    "pct_slope_magnitudes": ([_vp, _vp, _i32, _i32, _d, _vp, _vp, _vp], C.c_int),
    "pct_fuse_costs": ([_vp, _vp, _vp, _vp, _i32, _i32, C.POINTER(TravParamsC), _vp], C.c_int),
    "pct_inflate": ([_vp, _vp, _i32, _i32, _vp, _i32, _vp], C.c_int),
    "pct_gentle_fraction": ([_vp, _vp, _i32, _i32, _i32, _vp], C.c_int),
    "pct_terrain_cost_values": ([_vp, _vp, _vp, _vp, _i64, C.POINTER(TravParamsC), _vp], C.c_int),
    "pct_simplify": ([_vp, _vp, _vp, _i32, _i32, _i32, _d, _d, _vp, _vp], C.c_int),
    "pct_unique_mask": ([_vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _d, _d, _vp], C.c_int),
    "pct_partition_rows": ([_vp, _vp, _i64, C.c_int, C.POINTER(FrameC), _vp, _i32, _vp, _vp],
                           C.c_int),
    "pct_build_band": ([_vp, _vp, _i64, C.c_int, C.POINTER(FrameC), _vp, _i32, _i32, _i64, _vp,
                        _vp], C.c_int),
    "pct_copy_slices": ([_vp, _vp, _i64, _vp, _i64, _vp, _i32, _i64], C.c_int),
    "pct_xfer_count": ([_vp, _vp, _i64, _vp, _i32, _i64, _i32, _vp], C.c_int),
    "pct_xfer_pack": ([_vp, _vp, _i64, _vp, _i32, _i64, _i32, _vp, _vp, _vp, _vp], C.c_int),
    "pct_xfer_chunk_cells": ([], _i64),
    "pct_xfer_count_async": ([_vp, _vp, _i64, _vp, _i32, _i64, _i32, _vp], C.c_int),
    "pct_xfer_fence": ([_vp, _i32], C.c_int),
    "pct_xfer_wait": ([_vp, _i32], C.c_int),
    "pct_xfer_expand": ([_vp, _vp, _vp, _i32, _i64, _i32, _vp, _i32], C.c_int),
    "pct_xfer_expand_from": ([_vp, _vp, _vp, _i32, _i64, _i32, _vp, _i32, _vp], C.c_int),
    "pct_xfer_counts_bytes": ([_i64, _i32], C.c_int64),
    "pct_xfer_count_keep": ([_vp, _vp, _i64, _vp, _i32, _i64, _i32, _vp, _vp], C.c_int),
    "pct_xfer_pack_counted": ([_vp, _vp, _i64, _vp, _i32, _i64, _i32, _vp, _vp, _vp, _vp, _vp],
                              C.c_int),
    "pct_simplify_window": ([_vp, _vp, _vp, _i32, _i64, _i64, _d, _d, _vp], C.c_int),
    "pct_simplify_triples": ([_vp, _vp, _vp, _i32, _i64, _i64, _d, _d, _vp, _i32, _vp], C.c_int),
    "pct_planner_context": ([_vp, _vp, _vp, _i32, _i32, _i32, _d, _vp, _vp], C.c_int),
    "pct_ceiling_inflate": ([_vp, _vp, _i32, _i32, _i32, _d, _d, _d, _vp, _vp], C.c_int),
    "pct_pcd_extract": ([_vp, _vp, _i64, _i64, _vp, C.c_int, _vp, _vp], C.c_int),
    "pct_pcd_load": ([_vp, C.c_char_p, _i64, _i64, _i64, _vp, _i64, _vp, _vp], C.c_int),
    "pct_tomo_build": ([_vp, _vp, _i64, C.c_int, C.c_int, _d, _d, _i64, C.POINTER(_vp)], C.c_int),
    "pct_tomo_upload": ([_vp, C.POINTER(FrameC), _vp, _vp, _vp, C.POINTER(_vp)], C.c_int),
    "pct_tomo_evaluate": ([_vp, _vp, C.POINTER(TravParamsC), _vp, _i32], C.c_int),
    "pct_tomo_simplify": ([_vp, _vp, _d, _d, _vp, _vp], C.c_int),
    "pct_tomo_run": ([_vp, _vp, _i64, C.c_int, C.c_int, _d, _d, _i64, C.POINTER(TravParamsC), _vp,
                      _i32, _d, _d, C.POINTER(_vp), _vp, _vp], C.c_int),
    "pct_tomo_run_batch": ([_vp, _i32, _i32, _vp, _vp, C.c_int, _d, _d, _i64,
                            C.POINTER(TravParamsC), _vp, _i32, _d, _d, _vp, _vp, _i32, _vp],
                           C.c_int),
    "pct_set_timing": ([_vp, C.c_int], C.c_int),
    "pct_last_stage_ms": ([_vp, _vp], C.c_int),
    "pct_tomo_frame": ([_vp, C.POINTER(FrameC), _vp, _i32], C.c_int),
    "pct_tomo_layer": ([_vp, C.c_int], _vp),
    "pct_tomo_download": ([_vp, _vp, C.c_int, _i32, _vp], C.c_int),
    "pct_tomo_free": ([_vp, _vp], C.c_int),
}

_lib = None
_lib_lock = threading.Lock()


def declared_symbols():
    """Every function include/pct.h declares (the ABI the tests check)."""
    return sorted(_SIGS)


def load(path: Path | str | None = None):
    """Load libpct.so (raises RuntimeError if it has not been built)."""
    global _lib
    with _lib_lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path else Path(os.environ.get("PCT_LIB", LIB_PATH))
        if not p.exists():
            raise RuntimeError(f"libpct.so not found at {p}; run `python -c \"import "
                               f"__graft_entry__; __graft_entry__.build()\"` (no CPU fallback)")
        lib = C.CDLL(str(p))
        for name, (args, res) in _SIGS.items():
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = res
        if lib.pct_abi_version() != 1:
            raise RuntimeError("libpct ABI version mismatch")
        if path is None:
            _lib = lib
        return lib


class PctError(RuntimeError):
    pass


class Context:
    """One pct_ctx (device, stream, scratch).  Not re-entrant: calls are
    serialised with a lock."""

    def __init__(self, device: int = 0):
        self.lib = load()
        self.device = device
        h = C.c_void_p()
        rc = self.lib.pct_ctx_create(int(device), C.byref(h))
        if rc != PCT_OK:
            raise RuntimeError(f"libpct: cannot create a context on CUDA device {device} "
                               f"(code {rc}); a Blackwell GPU is required (no CPU fallback)")
        self.h = h
        self.lock = threading.RLock()

    def error(self) -> str:
        return self.lib.pct_last_error(self.h).decode()

    def check(self, rc: int, what: str = ""):
        if rc == PCT_OK:
            return
        msg = self.error()
        if rc == PCT_E_CUDA or rc == PCT_E_NOMEM:
            raise RuntimeError(f"{what}: {msg}")
        raise PctError(rc, msg)

    @property
    def launches(self) -> int:
        return int(self.lib.pct_launch_count(self.h))

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.pct_ctx_destroy(self.h)
                self.h = None
        except Exception:
            pass


_contexts: dict[int, Context] = {}


def default_device() -> int:
    return int(os.environ.get("PCT_DEVICE", "0"))


def context(device: int | None = None) -> Context:
    d = default_device() if device is None else int(device)
    ctx = _contexts.get(d)
    if ctx is None:
        ctx = _contexts[d] = Context(d)
    return ctx


class DeviceBuffer:
    """Stream-ordered device allocation owned by Python (freed on GC)."""

    __slots__ = ("ctx", "ptr", "nbytes", "__weakref__")

    def __init__(self, ctx: Context, nbytes: int):
        self.ctx = ctx
        p = C.c_void_p()
        ctx.check(ctx.lib.pct_malloc(ctx.h, C.c_size_t(int(nbytes)), C.byref(p)), "pct_malloc")
        self.ptr = p.value
        self.nbytes = int(nbytes)

    @classmethod
    def from_host(cls, ctx: Context, arr: np.ndarray) -> "DeviceBuffer":
        a = np.ascontiguousarray(arr)
        b = cls(ctx, a.nbytes)
        ctx.check(ctx.lib.pct_memcpy_h2d(ctx.h, b.ptr, a.ctypes.data, a.nbytes), "h2d")
        return b

    def to_host(self, out: np.ndarray) -> np.ndarray:
        assert out.flags.c_contiguous and out.nbytes <= self.nbytes
        self.ctx.check(self.ctx.lib.pct_memcpy_d2h(self.ctx.h, out.ctypes.data, self.ptr,
                                                   out.nbytes), "d2h")
        return out

    def __del__(self):
        try:
            if self.ptr:
                self.ctx.lib.pct_free(self.ctx.h, self.ptr)
                self.ptr = None
        except Exception:
            pass


class PinnedBuffer:
    """Page-locked host memory (fast H2D/D2H), viewed as a numpy array."""

    def __init__(self, ctx: Context, shape, dtype):
        self.ctx = ctx
        dt = np.dtype(dtype)
        n = int(np.prod(shape)) * dt.itemsize
        p = C.c_void_p()
        ctx.check(ctx.lib.pct_host_alloc(ctx.h, C.c_size_t(max(n, 1)), C.byref(p)), "host_alloc")
        self.ptr = p.value
        buf = (C.c_char * max(n, 1)).from_address(self.ptr)
        self.array = np.frombuffer(buf, dtype=dt, count=int(np.prod(shape))).reshape(shape)

    def __del__(self):
        try:
            if self.ptr:
                self.ctx.lib.pct_host_free(self.ctx.h, self.ptr)
                self.ptr = None
        except Exception:
            pass


class _PinnedBlock:
    """One page-locked block; returned to its pool when the last numpy view dies."""

    def __init__(self, pool, ptr, nbytes):
        self.pool, self.ptr, self.nbytes = pool, ptr, nbytes

    def __del__(self):
        try:
            self.pool._release(self)
        except Exception:
            pass


class PinnedPool:
    """Size-class free lists of page-locked host blocks for device->host copies.

    Arrays handed out stay valid as long as the caller holds them; their
    block goes back to the pool (not to the OS) when they are collected, so
    repeated pipelines do not pay for page locking again."""

    def __init__(self, device: int):
        self.device = device
        self.ctx = None  # the context page-locking new blocks (set per call)
        self.free: dict[int, list[int]] = {}
        self.lock = threading.Lock()

    @staticmethod
    def _class(nbytes: int) -> int:
        q = 1 << 20
        return max(q, (nbytes + q - 1) // q * q)

    def array(self, shape, dtype, ctx: Context | None = None) -> np.ndarray:
        dt = np.dtype(dtype)
        count = int(np.prod(shape))
        size = self._class(count * dt.itemsize)
        with self.lock:
            lst = self.free.get(size)
            ptr = lst.pop() if lst else None
        if ptr is None:
            ctx = ctx or self.ctx
            p = C.c_void_p()
            ctx.check(ctx.lib.pct_host_alloc(ctx.h, C.c_size_t(size), C.byref(p)), "host_alloc")
            ptr = p.value
        raw = (C.c_char * size).from_address(ptr)
        raw._pct_block = _PinnedBlock(self, ptr, size)
        return np.frombuffer(raw, dtype=dt, count=count).reshape(shape)

    def _release(self, block):
        with self.lock:
            self.free.setdefault(block.nbytes, []).append(block.ptr)


_POOLS: dict[int, PinnedPool] = {}
_POOLS_LOCK = threading.Lock()


def pinned_pool(ctx: Context) -> PinnedPool:
    """The process-wide pool of ctx's device: contexts share page-locked
    blocks (any stream can copy into them), so maps read back on alternating
    contexts re-use each other's blocks instead of page-locking new ones."""
    with _POOLS_LOCK:
        pool = _POOLS.get(ctx.device)
        if pool is None:
            pool = _POOLS[ctx.device] = PinnedPool(ctx.device)
    return _BoundPool(pool, ctx)


class _BoundPool:
    """A device pool with the context that page-locks its new blocks."""

    def __init__(self, pool: PinnedPool, ctx: Context):
        self.pool, self.ctx = pool, ctx

    def array(self, shape, dtype) -> np.ndarray:
        return self.pool.array(shape, dtype, self.ctx)


def trav_params_c(params, r_g: float) -> TravParamsC:
    pr = getattr(params, "step_patch_radius", None)
    pr = int(pr) if pr is not None else int(np.ceil(0.3 / r_g))
    return TravParamsC(float(params.d_min), float(params.d_ref), float(params.theta_b),
                       float(params.theta_s), float(params.theta_p), float(params.c_barrier),
                       float(params.alpha_d), float(params.alpha_b), float(params.alpha_s),
                       pr, 0)
