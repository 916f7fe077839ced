"""Many independent maps on one GPU (BASELINE config 4: 256 two-storey maps).

Small maps are latency-bound: one map's pipeline is a handful of short
kernels separated by host round trips (grid frame after the bounds, simplify
sweep).  ``BatchRunner`` owns ``workers`` libpct contexts (a CUDA stream and
scratch each).  Device-resident batches go through one native call,
``pct_tomo_run_batch``, that runs every stage as ONE launch over all maps
(bounds; build; evaluate; simplify tables; triple rounds) with one host
synchronisation per phase; host-resident ones run one ``pct_tomo_run`` per
map on a thread pool (ctypes releases the GIL), so the syncs of one map
overlap the kernels of the others.  Maps never communicate ("batches of independent maps are
distributed without communication"); across GPUs each rank takes its share.

``evaluate_maps`` is the public entry (an extension of the reference API):
clouds in, simplified device-backed ``Tomogram`` objects out, identical to
running build_tomogram -> evaluate_tomogram -> simplify_tomogram per cloud.
"""

from __future__ import annotations

import ctypes as C
import queue
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import _lib
from .cloud import source_points
from .tomogram import GRID_SIDE_LIMIT, DeviceTomogram, Layer, Tomogram, TomogramSlice
from .traversability import build_kernel


class BatchRunner:
    def __init__(self, device: int | None = None, workers: int = 8, streams=None):
        dev = _lib.default_device() if device is None else int(device)
        self.ctxs = [_lib.Context(dev) for _ in range(workers)]
        if streams is not None:  # caller-provided CUDA streams (e.g. for event timing)
            for ctx, s in zip(self.ctxs, streams):
                ctx.check(ctx.lib.pct_set_stream(ctx.h, C.c_void_p(int(s))), "set_stream")
        self.free = queue.Queue()
        for c in self.ctxs:
            self.free.put(c)
        self.pool = ThreadPoolExecutor(workers)

    def _one(self, ptr, n, code, on_host, d_s, r_g, pc, w, eps_e, c_barrier, keep_handle):
        ctx = self.free.get()
        try:
            h = C.c_void_p()
            keep = np.empty(65536, np.int32)
            nk = C.c_int32()
            rc = ctx.lib.pct_tomo_run(ctx.h, ptr, n, code, on_host, d_s, r_g, GRID_SIDE_LIMIT,
                                      C.byref(pc), w.ctypes.data, w.shape[0], eps_e, c_barrier,
                                      C.byref(h), keep.ctypes.data, C.byref(nk))
            ctx.check(rc, "pct_tomo_run")
            if not keep_handle:
                ctx.lib.pct_tomo_free(ctx.h, h)
                return None, keep[:nk.value].tolist()
            return (ctx, h), keep[:nk.value].tolist()
        finally:
            self.free.put(ctx)

    def run(self, maps, d_s, r_g, params, eps_e=1e-6, c_barrier=50.0, keep_handles=True):
        """maps: list of (pointer, n_points, dtype code, on_host).  Returns, in
        order, ((ctx, pct_tomo handle) or None, surviving slice indices).

        Device-resident maps go through pct_tomo_run_batch (one host thread,
        phase by phase over the contexts, one synchronisation per phase);
        host-resident ones through per-map pct_tomo_run calls on the pool."""
        if maps and all(not on_host for _, _, _, on_host in maps) and \
                len({code for _, _, code, _ in maps}) == 1:
            return self._run_batch(maps, d_s, r_g, params, eps_e, c_barrier, keep_handles)
        w = np.ascontiguousarray(build_kernel(params.d_inf, params.d_sm, r_g).weights)
        pc = _lib.trav_params_c(params, r_g)
        futs = [self.pool.submit(self._one, int(p), int(n), code, int(on_host), float(d_s),
                                 float(r_g), pc, w, float(eps_e), float(c_barrier), keep_handles)
                for p, n, code, on_host in maps]
        return [f.result() for f in futs]

    def _run_batch(self, maps, d_s, r_g, params, eps_e, c_barrier, keep_handles):
        """One pct_tomo_run_batch call: one launch per stage for every map."""
        n = len(maps)
        w = np.ascontiguousarray(build_kernel(params.d_inf, params.d_sm, r_g).weights)
        pc = _lib.trav_params_c(params, r_g)
        ctx = self.ctxs[0]
        hs = (C.c_void_p * 1)(ctx.h)
        ptrs = (C.c_void_p * n)(*[int(m[0]) for m in maps])
        npts = np.asarray([int(m[1]) for m in maps], np.int64)
        stride = 4096
        keep = np.empty((n, stride), np.int32)
        nk = np.empty(n, np.int32)
        handles = (C.c_void_p * n)() if keep_handles else None
        rc = ctx.lib.pct_tomo_run_batch(hs, 1, n, ptrs, npts.ctypes.data, maps[0][2], float(d_s),
                                        float(r_g), GRID_SIDE_LIMIT, C.byref(pc), w.ctypes.data,
                                        w.shape[0], float(eps_e), float(c_barrier), handles,
                                        keep.ctypes.data, stride, nk.ctypes.data)
        ctx.check(rc, "pct_tomo_run_batch")
        return [((ctx, C.c_void_p(handles[m])) if keep_handles else None,
                 keep[m, :nk[m]].tolist()) for m in range(n)]

    def close(self):
        self.pool.shutdown()


def _to_tomogram(ctx, handle, keep, d_s, r_g):
    dt = DeviceTomogram(ctx, handle)
    gst, cst = dt.stacks()
    from .tomogram import DeviceStack
    fr = dt.frame
    cost = DeviceStack(ctx, ctx.lib.pct_tomo_layer(handle, _lib.LAYER_COST), fr.n_slices,
                       fr.rows, fr.cols, dt)
    origin = (float(fr.origin_x), float(fr.origin_y))
    slices = [TomogramSlice(Layer.on_device(gst, k, r_g, origin), Layer.on_device(cst, k, r_g, origin),
                            float(dt.heights[k]), i, Layer.on_device(cost, k, r_g, origin))
              for i, k in enumerate(keep)]
    return Tomogram(slices=slices, d_s=float(d_s), z_min=float(fr.z_min))


def evaluate_maps(clouds, d_s, r_g, params, *, workers=8, device=None, eps_e=1e-6,
                  c_barrier=50.0, runner: BatchRunner | None = None):
    """build -> evaluate -> simplify for every cloud; returns the simplified
    tomograms (device-resident, host arrays on access)."""
    if d_s <= 0 or r_g <= 0:
        raise ValueError("d_s and r_g must be positive")
    own = runner is None
    runner = runner or BatchRunner(device, workers)
    arrays = [np.ascontiguousarray(source_points(c)) for c in clouds]
    codes = {a.dtype for a in arrays}
    if len(codes) == 1:
        # one upload per map, then the phase-batched native call
        ctx0 = runner.ctxs[0]
        bufs = [_lib.DeviceBuffer.from_host(ctx0, a) for a in arrays]
        ctx0.check(ctx0.lib.pct_sync(ctx0.h), "sync")
        maps = [(b.ptr, a.shape[0], _lib.PCT_F32 if a.dtype == np.float32 else _lib.PCT_F64, 0)
                for a, b in zip(arrays, bufs)]
    else:
        maps = [(a.ctypes.data, a.shape[0],
                 _lib.PCT_F32 if a.dtype == np.float32 else _lib.PCT_F64, 1) for a in arrays]
    try:
        res = runner.run(maps, d_s, r_g, params, eps_e, c_barrier)
    finally:
        if own:
            runner.close()
    return [_to_tomogram(h[0], h[1], keep, d_s, r_g) for h, keep in res]


def stream_maps(clouds, d_s, r_g, params, *, workers=2, device=None, eps_e=1e-6,
                c_barrier=50.0, runner: BatchRunner | None = None):
    """Generator over ``clouds`` (host arrays or PointClouds, ideally in pinned
    memory): yields, in input order, the simplified tomogram of each cloud
    with every surviving layer already copied to host memory.

    Each map is one native ``pct_tomo_run`` (upload, build, evaluate,
    simplify) plus the read-back of its surviving layers, on one of
    ``workers`` contexts; up to ``workers`` maps are in flight, so the
    host->device upload of one map overlaps the device->host read-back of
    the previous one (the PCIe link is full duplex) and its kernels."""
    if d_s <= 0 or r_g <= 0:
        raise ValueError("d_s and r_g must be positive")
    own = runner is None
    runner = runner or BatchRunner(device, workers)
    w = np.ascontiguousarray(build_kernel(params.d_inf, params.d_sm, r_g).weights)
    pc = _lib.trav_params_c(params, r_g)

    def one(a):
        code = _lib.PCT_F32 if a.dtype == np.float32 else _lib.PCT_F64
        ctx = runner.free.get()  # held until the read-back is done
        try:
            with ctx.lock:
                h = C.c_void_p()
                keep = np.empty(65536, np.int32)
                nk = C.c_int32()
                ctx.check(ctx.lib.pct_tomo_run(ctx.h, a.ctypes.data, a.shape[0], code, 1,
                                               float(d_s), float(r_g), GRID_SIDE_LIMIT,
                                               C.byref(pc), w.ctypes.data, w.shape[0],
                                               float(eps_e), float(c_barrier), C.byref(h),
                                               keep.ctypes.data, C.byref(nk)), "pct_tomo_run")
                return _to_tomogram(ctx, h, keep[:nk.value].tolist(), d_s, r_g).materialize()
        finally:
            runner.free.put(ctx)

    depth = max(1, len(runner.ctxs))
    pending = []
    try:
        for c in clouds:
            a = np.ascontiguousarray(source_points(c))
            if a.dtype not in (np.float32, np.float64) or a.ndim != 2 or a.shape[1] != 3:
                raise ValueError("clouds must be (N, 3) float32/float64 arrays")
            pending.append(runner.pool.submit(one, a))
            if len(pending) >= depth:
                yield pending.pop(0).result()
        while pending:
            yield pending.pop(0).result()
    finally:
        for f in pending:
            f.cancel()
        if own:
            runner.close()
