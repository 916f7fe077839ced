"""Tomogram types and the device build (drop-in for tomoplan/tomogram.py:22-213).

``build_tomogram`` keeps the reference signature (tomogram.py:127-128) and
returns the same object model (Tomogram / TomogramSlice / Layer with
(rows, cols) float32 values, NaN = invalid).  The stacks stay resident on the
GPU; ``Layer.values`` is materialised on the host on first access (one
device-to-host copy of that slice), so a build -> evaluate -> simplify chain
only ever moves the surviving slices to the host.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import time
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib
from .cloud import PointCloud

GRID_SIDE_LIMIT = 16384

# compacted read-back (Tomogram.materialize): slices with at least this share
# of empty-NaN cells, in stacks of at least XFER_MIN_CELLS cells per slice
XFER_MIN_EMPTY = 0.5
XFER_MIN_CELLS = 1 << 20
# a stack's kept slices travel as a delta chain (each against the previous
# kept slice) when at most this share of their cells differ
XFER_DELTA_MAX = 0.25
# the first delta chain crosses PCIe in parts ending at these slices (each
# rebuilt while the next is in flight) so the host starts early
XFER_SPLIT = (4, 12)


class GridSizeError(ValueError):
    """Grid dimensions exceed the configured safety limit."""


# ---------------------------------------------------------------------------
# device-resident layer stacks

class DeviceStack:
    """A (S, rows, cols) float32 stack in device memory.

    ``owner`` keeps the allocation alive (a DeviceTomogram or DeviceBuffer).
    Host copies of individual slices are made on demand and cached.
    """

    def __init__(self, ctx, ptr: int, n_slices: int, rows: int, cols: int, owner):
        self.ctx = ctx
        self.ptr = int(ptr)
        self.n_slices = int(n_slices)
        self.rows = int(rows)
        self.cols = int(cols)
        self.owner = owner
        self._host = {}
        self._kept = None  # (slices, delta, device counts) of the last kept count pass
        # evaluation outputs: the ground stack they came from, its build masks
        # and the tile masks of this (cost) stack (traversability._evaluate_layers)
        self.change_info = None

    @property
    def plane_bytes(self) -> int:
        return self.rows * self.cols * 4

    def slice_ptr(self, k: int) -> int:
        return self.ptr + int(k) * self.plane_bytes

    def host_slice(self, k: int) -> np.ndarray:
        a = self._host.get(k)
        if a is None:
            a = _lib.pinned_pool(self.ctx).array((self.rows, self.cols), np.float32)
            with self.ctx.lock:
                self.ctx.check(self.ctx.lib.pct_memcpy_d2h(self.ctx.h, a.ctypes.data,
                                                           self.slice_ptr(k), a.nbytes), "d2h")
            self._host[k] = a
        return a

    def prefetch(self, ks, sync: bool = True) -> None:
        """Copy several slices to (pinned) host memory: one pinned block, one
        copy per run of consecutive slices, one synchronisation (none with
        ``sync=False``: the caller synchronises the context's stream)."""
        todo = sorted(k for k in set(ks) if k not in self._host)
        if not todo:
            return
        block = _lib.pinned_pool(self.ctx).array((len(todo), self.rows, self.cols), np.float32)
        with self.ctx.lock:
            i = 0
            while i < len(todo):
                j = i
                while j + 1 < len(todo) and todo[j + 1] == todo[j] + 1:
                    j += 1
                self.ctx.check(self.ctx.lib.pct_memcpy_d2h_async(
                    self.ctx.h, block[i].ctypes.data, self.slice_ptr(todo[i]),
                    (j - i + 1) * self.plane_bytes), "d2h")
                i = j + 1
            if sync:
                self.ctx.check(self.ctx.lib.pct_sync(self.ctx.h), "sync")
        for n, k in enumerate(todo):
            self._host[k] = block[n]

    def count_nonempty(self, ks, delta: bool = False) -> np.ndarray:
        """Non-empty cells (not the empty-cell NaN 0x7FC00000) of slices ks;
        with ``delta``, slice m > 0 counts the cells that differ from slice
        m - 1 of the list instead."""
        idx = np.ascontiguousarray(ks, dtype=np.int32)
        tot = np.empty(len(idx), np.int64)
        self._kept = None
        with self.ctx.lock:
            self.ctx.check(self.ctx.lib.pct_xfer_count(
                self.ctx.h, self.ptr, self.rows * self.cols, idx.ctypes.data, len(idx),
                self.rows * self.cols, int(bool(delta)), tot.ctypes.data), "xfer_count")
        return tot

    def count_nonempty_async(self, ks, delta: bool, out: np.ndarray, keep: bool = False) -> None:
        """count_nonempty into ``out`` (page-locked int64), stream-ordered:
        valid once the context's stream has synchronised.  ``keep``: the
        per-chunk counts stay on the device for a compact_start of the same
        slices (pct_xfer_pack_counted: no second count pass)."""
        idx = np.ascontiguousarray(ks, dtype=np.int32)
        cells = self.rows * self.cols
        with self.ctx.lock:
            if keep:
                lib = self.ctx.lib
                buf = _lib.DeviceBuffer(self.ctx, int(lib.pct_xfer_counts_bytes(cells, len(idx))))
                self.ctx.check(lib.pct_xfer_count_keep(
                    self.ctx.h, self.ptr, cells, idx.ctypes.data, len(idx), cells,
                    int(bool(delta)), out.ctypes.data, buf.ptr), "xfer_count")
                self._kept = (tuple(int(k) for k in ks), bool(delta), buf)
            else:
                self.ctx.check(self.ctx.lib.pct_xfer_count_async(
                    self.ctx.h, self.ptr, cells, idx.ctypes.data, len(idx), cells,
                    int(bool(delta)), out.ctypes.data), "xfer_count")

    def compact_start(self, ks, totals, delta: bool = False, split=(), fence=None):
        """Queue the compacted read-back of slices ks (pct_xfer_pack, then
        bitmaps, packed values and chunk offsets to pinned host memory);
        finish with :meth:`compact_finish` once the copies have landed.
        ``split`` = (m1, m2, ..) (delta chains): the copies go in parts
        [0, m1), [m1, m2), .., and ``fence()`` is called after every part but
        the last (so those slices are rebuilt while the rest still crosses
        PCIe; see compact_finish)."""
        cells = self.rows * self.cols
        n = len(ks)
        idx = np.ascontiguousarray(ks, dtype=np.int32)
        off = np.zeros(n, np.int64)
        off[1:] = np.cumsum(np.asarray(totals, np.int64))[:-1]
        n_packed = int(np.sum(totals))
        chunk = int(self.ctx.lib.pct_xfer_chunk_cells())
        nchunk = (cells + chunk - 1) // chunk
        words = (cells + 31) // 32
        pool = _lib.pinned_pool(self.ctx)
        # one 64-byte aligned host slice each (the rebuild streams whole
        # 64-byte lines with non-temporal stores; a slice of cells % 16 != 0
        # cells packed back to back would put every later slice off the lines)
        pc = (cells + 15) // 16 * 16
        raw = pool.array((n, pc), np.float32)
        block = [raw[i, :cells].reshape(self.rows, self.cols) for i in range(n)]
        h_bm = pool.array((n, words), np.uint32)
        h_pk = pool.array((max(n_packed, 1),), np.float32)
        h_co = pool.array((n, nchunk), np.int64)
        d_bm = _lib.DeviceBuffer(self.ctx, h_bm.nbytes)
        d_pk = _lib.DeviceBuffer(self.ctx, h_pk.nbytes)
        d_co = _lib.DeviceBuffer(self.ctx, h_co.nbytes)
        lib, h = self.ctx.lib, self.ctx.h
        prof = os.environ.get("PCT_XFER_TRACE") == "2"  # diagnostic: pack / copy times
        if prof:
            t0 = time.perf_counter()
        kept, self._kept = self._kept, None
        with self.ctx.lock:
            if kept is not None and kept[0] == tuple(int(k) for k in ks) and kept[1] == bool(delta):
                self.ctx.check(lib.pct_xfer_pack_counted(
                    h, self.ptr, cells, idx.ctypes.data, n, cells, int(bool(delta)),
                    off.ctypes.data, kept[2].ptr, d_bm.ptr, d_pk.ptr, d_co.ptr), "xfer_pack")
            else:
                self.ctx.check(lib.pct_xfer_pack(h, self.ptr, cells, idx.ctypes.data, n, cells,
                                                 int(bool(delta)), off.ctypes.data, d_bm.ptr,
                                                 d_pk.ptr, d_co.ptr), "xfer_pack")
            if prof:
                lib.pct_sync(h)
                t1 = time.perf_counter()
            self.ctx.check(lib.pct_memcpy_d2h_async(h, h_co.ctypes.data, d_co.ptr, h_co.nbytes),
                           "d2h")
            cuts = [0] + sorted(m for m in set(split) if 0 < m < n) + [n] if delta else [0, n]
            parts = list(zip(cuts[:-1], cuts[1:]))
            ends = np.concatenate([off, [n_packed]])
            for a, b in parts:
                wb = h_bm.strides[0]
                self.ctx.check(lib.pct_memcpy_d2h_async(h, h_bm.ctypes.data + a * wb,
                                                        d_bm.ptr + a * wb, (b - a) * wb), "d2h")
                p0, p1 = int(ends[a]), int(ends[b])
                if p1 > p0:
                    self.ctx.check(lib.pct_memcpy_d2h_async(h, h_pk.ctypes.data + 4 * p0,
                                                            d_pk.ptr + 4 * p0, 4 * (p1 - p0)),
                                   "d2h")
                if b < n and fence is not None:
                    fence()
            if prof:
                lib.pct_sync(h)
                t2 = time.perf_counter()
                import sys
                sys.stderr.write(f"compact_start: pack {1e3 * (t1 - t0):.2f} ms, copies "
                                 f"{1e3 * (t2 - t1):.2f} ms for {(h_bm.nbytes + h_co.nbytes + 4 * n_packed) / 1e6:.0f} MB\n")
        return (list(ks), block, h_bm, h_pk, h_co, (d_bm, d_pk, d_co), bool(delta))

    def compact_finish(self, pending, threads: int, part=None) -> None:
        """Expand the landed compacted slices into their host arrays
        (``part`` = (a, b): slices [a, b) of the list only; a delta chain's
        part continues from slice a - 1, already rebuilt)."""
        ks, block, h_bm, h_pk, h_co, _dev, delta = pending
        a, b = part if part is not None else (0, len(ks))
        outs = (C.c_void_p * (b - a))(*[block[i].ctypes.data for i in range(a, b)])
        base = block[a - 1].ctypes.data if (delta and a > 0) else None
        self.ctx.check(self.ctx.lib.pct_xfer_expand_from(
            h_bm.ctypes.data + a * h_bm.strides[0], h_pk.ctypes.data,
            h_co.ctypes.data + a * h_co.strides[0], b - a, self.rows * self.cols, int(delta),
            outs, int(threads), base), "xfer_expand")
        for i in range(a, b):
            self._host[ks[i]] = block[i]

    def host_all(self) -> np.ndarray:
        out = np.empty((self.n_slices, self.rows, self.cols), np.float32)
        with self.ctx.lock:
            self.ctx.check(self.ctx.lib.pct_memcpy_d2h(self.ctx.h, out.ctypes.data, self.ptr,
                                                       out.nbytes), "d2h")
        for k in range(self.n_slices):
            self._host.setdefault(k, out[k])
        return out


class DeviceTomogram:
    """Owner of a pct_tomo (ground + ceiling stacks built on the device).

    The stacks reference their owner, never the other way round, so the
    device memory is released by reference counting as soon as the last
    Layer of the tomogram is dropped (no cycle for the GC to find)."""

    def __init__(self, ctx, handle):
        self.ctx = ctx
        self.handle = handle
        fr = _lib.FrameC()
        ctx.check(ctx.lib.pct_tomo_frame(handle, C.byref(fr), None, 0), "frame")
        self.frame = fr
        h = np.empty(max(fr.n_slices, 1), np.float64)
        ctx.check(ctx.lib.pct_tomo_frame(handle, C.byref(fr), h.ctypes.data, fr.n_slices), "frame")
        self.heights = h[:fr.n_slices]
        weakref.finalize(self, ctx.lib.pct_tomo_free, ctx.h, handle)

    def stacks(self):
        fr, ctx = self.frame, self.ctx
        g = DeviceStack(ctx, ctx.lib.pct_tomo_layer(self.handle, _lib.LAYER_GROUND),
                        fr.n_slices, fr.rows, fr.cols, self)
        c = DeviceStack(ctx, ctx.lib.pct_tomo_layer(self.handle, _lib.LAYER_CEILING),
                        fr.n_slices, fr.rows, fr.cols, self)
        return g, c


def new_device_stack(ctx, n_slices, rows, cols) -> DeviceStack:
    buf = _lib.DeviceBuffer(ctx, max(1, n_slices * rows * cols * 4))
    return DeviceStack(ctx, buf.ptr, n_slices, rows, cols, buf)


def upload_stack(ctx, arrays) -> DeviceStack:
    a = np.ascontiguousarray(np.stack([np.asarray(v, np.float32) for v in arrays]))
    buf = _lib.DeviceBuffer.from_host(ctx, a)
    return DeviceStack(ctx, buf.ptr, a.shape[0], a.shape[1], a.shape[2], buf)


# ---------------------------------------------------------------------------
# the reference object model (tomogram.py:29-96)

class Layer:
    """Dense 2D elevation grid; NaN = invalid. Row i follows y, column j follows x.

    ``values`` is a (rows, cols) float32 numpy array; for layers produced on
    the GPU it is copied from device memory on first access.
    """

    __slots__ = ("_values", "_stack", "_k", "resolution", "origin")

    def __init__(self, values, resolution: float, origin):
        self._stack = None
        self._k = -1
        self._values = np.asarray(values, dtype=np.float32)
        if self._values.ndim != 2 or min(self._values.shape) < 1:
            raise ValueError("layer grid must be 2D and non-empty")
        if resolution <= 0:
            raise ValueError("resolution must be positive")
        self.resolution = resolution
        self.origin = origin

    @classmethod
    def on_device(cls, stack: DeviceStack, k: int, resolution: float, origin) -> "Layer":
        self = cls.__new__(cls)
        self._values = None
        self._stack = stack
        self._k = int(k)
        self.resolution = resolution
        self.origin = origin
        return self

    @property
    def values(self) -> np.ndarray:
        if self._values is None:
            self._values = self._stack.host_slice(self._k)
        return self._values

    @values.setter
    def values(self, v):
        self._values = np.asarray(v, dtype=np.float32)
        self._stack = None
        self._k = -1

    @property
    def device(self):
        """(DeviceStack, slice index) when the layer lives on the GPU, else None."""
        return (self._stack, self._k) if self._stack is not None else None

    @property
    def shape(self):
        if self._values is None:
            return (self._stack.rows, self._stack.cols)
        return self._values.shape

    @property
    def valid(self) -> np.ndarray:
        return np.isfinite(self.values)

    def like(self, values: np.ndarray) -> "Layer":
        return Layer(values, self.resolution, self.origin)

    def __repr__(self):
        where = "device" if self._values is None else "host"
        return (f"Layer(shape={self.shape}, resolution={self.resolution!r}, "
                f"origin={self.origin!r}, {where})")


@dataclass
class TomogramSlice:
    ground: Layer
    ceiling: Layer
    plane_height: float
    index: int
    cost: Layer | None = None


@dataclass
class Tomogram:
    slices: list
    d_s: float
    z_min: float

    @property
    def rows(self):
        return self.slices[0].ground.shape[0]

    @property
    def cols(self):
        return self.slices[0].ground.shape[1]

    @property
    def resolution(self):
        return self.slices[0].ground.resolution

    @property
    def origin(self):
        return self.slices[0].ground.origin

    def materialize(self) -> "Tomogram":
        """Copy every device-resident layer to host memory with one
        synchronisation per stack (``Layer.values`` then costs nothing).

        The drop-in chain is bound by this copy (cfg3: 6.7 GB of kept layers
        over PCIe), so the layers travel compacted (k_xfer.cu) and host
        threads rebuild them: a stack whose consecutive kept slices share
        most cells (at most XFER_DELTA_MAX differ; cfg3: 6 %) goes as a delta
        chain -- slice 0 against the empty NaN, every later slice as the cells
        that differ from the previous one; otherwise slices that are mostly
        the empty NaN (at least XFER_MIN_EMPTY of their cells) go as a bitmap
        + their non-empty values, and the rest dense, copied while the
        compacted ones are expanded.  PCT_XFER_COMPACT=0: every slice dense;
        =nan: no delta chains.  cfg3: 127 ms dense, 110 ms NaN-compacted,
        64 ms with delta chains (host-memory bound: 6.7 GB written)."""
        trace = os.environ.get("PCT_XFER_TRACE") == "1"
        t_0 = time.perf_counter()
        marks = []

        def mark(what):
            if trace:
                marks.append((what, time.perf_counter() - t_0))
        groups = {}
        for s in self.slices:
            for l in (s.ground, s.ceiling, s.cost):
                if isinstance(l, Layer) and l._values is None and l._stack is not None:
                    groups.setdefault(id(l._stack), (l._stack, []))[1].append(l._k)
        ctxs = {}
        for stack, _ in groups.values():
            ctxs[id(stack.ctx)] = stack.ctx
        mode = os.environ.get("PCT_XFER_COMPACT", "1")
        compact = mode != "0"
        todo = []
        for stack, ks in groups.values():
            ks = sorted(k for k in set(ks) if k not in stack._host)
            if ks:
                todo.append((stack, ks))

        def counts(cands, delta):
            # every candidate stack's counts queued, one synchronisation (a
            # delta chain's chunk counts stay on the device for its pack)
            outs = []
            for stack, ks in cands:
                out = _lib.pinned_pool(stack.ctx).array((len(ks),), np.int64)
                stack.count_nonempty_async(ks, delta, out, keep=delta)
                outs.append(out)
            for ctx in {id(st.ctx): st.ctx for st, _ in cands}.values():
                with ctx.lock:
                    ctx.check(ctx.lib.pct_sync(ctx.h), "sync")
            return outs

        # plan: stack -> (compacted slices, their counts, delta chain)
        chosen = {}
        min_cells = int(os.environ.get("PCT_XFER_MIN_CELLS", XFER_MIN_CELLS))
        big = [(st, ks) for st, ks in todo if compact and st.rows * st.cols >= min_cells]
        if mode != "nan":
            cands = [(st, ks) for st, ks in big if len(ks) > 1]
            for (st, ks), dt in zip(cands, counts(cands, True)):
                if int(dt[1:].sum()) <= XFER_DELTA_MAX * (len(ks) - 1) * st.rows * st.cols:
                    chosen[id(st)] = (list(ks), [int(t) for t in dt], True)
        mark("delta counts")
        rest = [(st, ks) for st, ks in big if id(st) not in chosen]
        for (st, ks), nt in zip(rest, counts(rest, False)):
            lim = (1.0 - XFER_MIN_EMPTY) * st.rows * st.cols
            ck = [k for k, t in zip(ks, nt) if t <= lim]
            if ck:
                chosen[id(st)] = (ck, [int(t) for t in nt if t <= lim], False)
        # compacted copies first, stack by stack, each followed by an event
        # (slot = its position, up to 8 per context), then the dense copies
        # The first delta chain's first XFER_SPLIT slices cross on their own,
        # so the host starts rebuilding them while the rest is in flight.
        pending, slot_of = [], {}

        def next_slot(ctx):
            slot = slot_of.get(id(ctx), 0) % 8
            slot_of[id(ctx)] = slot + 1
            return slot
        split_done = False
        for st, ks in todo:
            if id(st) in chosen:
                ck, ct, delta = chosen[id(st)]
                split, early = (), []
                if delta and not split_done and len(ck) >= 8:
                    split = tuple(m for m in XFER_SPLIT if m < len(ck) - 2)
                    split_done = True

                def fence(st=st, early=early):
                    early.append(next_slot(st.ctx))
                    st.ctx.check(st.ctx.lib.pct_xfer_fence(st.ctx.h, early[-1]), "xfer_fence")
                with st.ctx.lock:
                    p = st.compact_start(ck, ct, delta, split=split, fence=fence)
                    slot = next_slot(st.ctx)
                    st.ctx.check(st.ctx.lib.pct_xfer_fence(st.ctx.h, slot), "xfer_fence")
                pending.append((st, p, ct, slot, split, early))
        dense = [(st, [k for k in ks if id(st) not in chosen or k not in set(chosen[id(st)][0])])
                 for st, ks in todo]
        # bytes that cross PCIe in this call (dense slices + compacted payloads)
        self.xfer_bytes = sum(len(ks) * st.plane_bytes for st, ks in dense) + \
            sum(p[2].nbytes + 4 * int(sum(ct)) + p[4].nbytes for _, p, ct, *_ in pending)
        mark("packs queued")
        for stack, ks in dense:
            if ks:
                stack.prefetch(ks, sync=False)
        # expand each stack as soon as its compacted data has landed (the later
        # stacks' copies and the dense ones still in flight)
        threads = int(os.environ.get("PCT_XFER_THREADS", 0)) or max(1, (os.cpu_count() or 1))
        for stack, p, _, slot, split, early in pending:
            if early:
                cuts = [0] + list(split) + [len(p[0])]
                for q, ev in enumerate(early + [slot]):
                    stack.ctx.check(stack.ctx.lib.pct_xfer_wait(stack.ctx.h, ev), "xfer_wait")
                    mark(f"part {q} landed")
                    stack.compact_finish(p, threads, part=(cuts[q], cuts[q + 1]))
            else:
                stack.ctx.check(stack.ctx.lib.pct_xfer_wait(stack.ctx.h, slot), "xfer_wait")
                mark("landed")
                stack.compact_finish(p, threads)
            mark("expanded")
        for ctx in ctxs.values():
            with ctx.lock:
                ctx.check(ctx.lib.pct_sync(ctx.h), "sync")
        mark("done")
        if trace:
            import sys
            sys.stderr.write("materialize: " + ", ".join(f"{w} {1e3 * t:.1f}" for w, t in marks) +
                             " ms\n")
        return self

    def _stack(self, attr):
        layers = [getattr(s, attr) for s in self.slices]
        src = device_run(layers)
        if src is not None and src[1] == 0 and src[0].n_slices == len(layers):
            return src[0].host_all()
        return np.stack([l.values for l in layers])

    def ground_stack(self) -> np.ndarray:
        return self._stack("ground")

    def ceiling_stack(self) -> np.ndarray:
        return self._stack("ceiling")

    def cost_stack(self) -> np.ndarray:
        if any(s.cost is None for s in self.slices):
            raise ValueError("tomogram has no cost layers; run evaluate_tomogram first")
        return self._stack("cost")


def device_run(layers):
    """(stack, first) if the layers are consecutive slices first.. of one
    device stack (still un-modified on the host side), else None."""
    if not layers:
        return None
    d0 = layers[0].device if isinstance(layers[0], Layer) else None
    if d0 is None:
        return None
    stack, first = d0
    for n, l in enumerate(layers):
        d = l.device if isinstance(l, Layer) else None
        if d is None or d[0] is not stack or d[1] != first + n:
            return None
    return stack, first


# ---------------------------------------------------------------------------
# build (tomogram.py:99-213)

def rasterize_index(p, origin, r_g: float, shape=None):
    """Map a point to (row, col) with the nearest-cell-center convention.

    i = floor((y - y0) / r_g + 0.5), j = floor((x - x0) / r_g + 0.5)
    (tomogram.py:99-112).  With `shape` given, indices outside the grid raise
    IndexError.  Scalar host helper (not on the hot path).
    """
    if r_g <= 0:
        raise ValueError("r_g must be positive")
    x, y = float(p[0]), float(p[1])
    i = math.floor((y - origin[1]) / r_g + 0.5)
    j = math.floor((x - origin[0]) / r_g + 0.5)
    if shape is not None and not (0 <= i < shape[0] and 0 <= j < shape[1]):
        raise IndexError(f"point ({x}, {y}) rasterizes to ({i}, {j}), outside grid {shape}")
    return i, j


def _dtype_code(arr: np.ndarray) -> int:
    if arr.dtype == np.float32:
        return _lib.PCT_F32
    if arr.dtype == np.float64:
        return _lib.PCT_F64
    raise TypeError(f"unsupported point dtype {arr.dtype}")


def device_bounds(xyz: np.ndarray, device=None):
    """Exact float64 (min, max) corners computed on the GPU (cloud_io.py:47-50)."""
    ctx = _lib.context(device)
    a = np.ascontiguousarray(xyz)
    buf = _lib.DeviceBuffer.from_host(ctx, a)
    return bounds_on_device(ctx, buf.ptr, a.shape[0], a.dtype)


def bounds_on_device(ctx, ptr: int, n: int, dtype):
    """(min, max) of n device-resident points at ``ptr`` (float32/float64)."""
    lo = np.empty(3, np.float64)
    hi = np.empty(3, np.float64)
    with ctx.lock:
        rc = ctx.lib.pct_bounds(ctx.h, ptr, int(n), _dtype_code(np.empty(0, dtype)),
                                lo.ctypes.data, hi.ctypes.data)
        if rc == _lib.PCT_E_NONFINITE:
            raise ValueError("point cloud contains non-finite coordinates")
        ctx.check(rc, "pct_bounds")
    return lo, hi


def build_from_points(xyz, d_s: float, r_g: float, max_grid_side: int = GRID_SIDE_LIMIT,
                      device=None, on_device: bool = False, n_points: int | None = None,
                      dtype=None) -> Tomogram:
    """Build from an (N, 3) float32/float64 array (host numpy, or a raw device
    pointer with ``on_device=True`` plus ``n_points`` and ``dtype``)."""
    if d_s <= 0 or r_g <= 0:
        raise ValueError("d_s and r_g must be positive")
    ctx = _lib.context(device)
    if on_device:
        ptr, n, code = int(xyz), int(n_points), _dtype_code(np.empty(0, dtype))
    else:
        a = np.ascontiguousarray(xyz)
        ptr, n, code = a.ctypes.data, a.shape[0], _dtype_code(a)
    h = C.c_void_p()
    with ctx.lock:
        rc = ctx.lib.pct_tomo_build(ctx.h, ptr, n, code, 0 if on_device else 1, float(d_s),
                                    float(r_g), int(max_grid_side), C.byref(h))
        if rc == _lib.PCT_E_GRID:
            raise GridSizeError(ctx.error())
        if rc == _lib.PCT_E_EMPTY:
            from .cloud import CloudFormatError
            raise CloudFormatError(ctx.error())
        if rc in (_lib.PCT_E_INVALID, _lib.PCT_E_NONFINITE):
            raise ValueError(ctx.error())
        ctx.check(rc, "pct_tomo_build")
    dt = DeviceTomogram(ctx, h)
    fr = dt.frame
    gst, cst = dt.stacks()
    origin = (float(fr.origin_x), float(fr.origin_y))
    slices = [TomogramSlice(ground=Layer.on_device(gst, k, r_g, origin),
                            ceiling=Layer.on_device(cst, k, r_g, origin),
                            plane_height=float(dt.heights[k]), index=k)
              for k in range(fr.n_slices)]
    return Tomogram(slices=slices, d_s=float(d_s), z_min=float(fr.z_min))


def build_tomogram(cloud: PointCloud, d_s: float, r_g: float, threads: int = 1,
                   max_grid_side: int = GRID_SIDE_LIMIT, *, device=None) -> Tomogram:
    """Project the cloud onto planes at z_min + (k+1)*d_s and build all slices.

    Drop-in for tomogram.py:127-213 (same arguments, errors and results,
    bit-identical layers).  ``threads`` is accepted and ignored: the work
    runs on the GPU ``device`` (default: $PCT_DEVICE or 0).
    """
    if d_s <= 0 or r_g <= 0:
        raise ValueError("d_s and r_g must be positive")
    dev = getattr(cloud, "device_points", None)
    if dev is not None:  # HBM-resident cloud (binary PCD ingest): no host round trip
        ptr, n, dtype, dev_id = dev()
        return build_from_points(ptr, d_s, r_g, max_grid_side, device=dev_id, on_device=True,
                                 n_points=n, dtype=dtype)
    from .cloud import source_points
    return build_from_points(source_points(cloud), d_s, r_g, max_grid_side, device=device)
