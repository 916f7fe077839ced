"""Row-band sharding of one large map over several GPUs (SURVEY.md §8 e).

Each rank owns a contiguous band of grid rows.  Per rank (one process per
GPU, NCCL over NVLink via torch.distributed; PyTorch tensors only as
buffers):

  1. bounds of the local point shard -> all-reduce -> the global grid frame
     (tomogram.py:134-145, identical on every rank)
  2. points partitioned by owner band on the device (pct_partition_rows)
     -> all-to-all (NCCL) -> every rank holds the points of its rows
  3. banded build with the GLOBAL frame (pct_build_band) into an extended
     stack that has room for H = R + r + 1 halo rows above and below
  4. halo exchange: the first/last H own rows of ground and ceiling go to the
     neighbour ranks (NCCL send/recv)
  5. fused evaluate on the extended band: the own rows are exact because the
     stencil reaches at most R + r + 1 rows for ground and R for ceiling
  6. simplify: every rank computes the any() table / triple flags over its
     own rows; they are max-reduced and every rank replays the same sweep
     (simplify.py:59-70), so all ranks agree on the surviving slices
  7. gather: the surviving slices of every band (ground, ceiling, cost) go
     to one rank (NCCL send/recv), which assembles the full-grid stacks and
     returns one reference-compatible Tomogram (``tomogram_sharded``).

Every error that depends on the data (a non-finite point on any rank, a band
thinner than the halo) is decided on values all ranks share, before the
first point exchange, so all ranks raise together instead of leaving the
others blocked in a collective.  Strided copies (halo packing, gathering)
are libpct kernels (pct_copy_slices); torch only provides the buffers.

The result is bit-identical to the single-GPU pipeline (tested with
virtual ranks on one GPU, tests/test_gpu_sharded.py, and the collective /
sweep logic with gloo on CPU, tests/test_sharded_host.py).

The pipeline is a generator that yields a request at every collective;
``run_torch`` serves them with torch.distributed, ``run_virtual`` runs P
ranks in lockstep in one process (device copies stand in for NCCL).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib

KWIN = 16   # lower-neighbour window of pct_simplify_window
KNONE = 32  # bit of "no lower neighbour"


# ---------------------------------------------------------------------------
# band geometry

def band_starts(rows: int, size: int) -> list:
    """Balanced contiguous row bands: band b owns rows [s[b], s[b+1])."""
    return [rows * b // size for b in range(size + 1)]


def halo_rows(params, r_g: float, kside: int) -> int:
    """Rows of ground a band needs beyond its own rows: inflation radius R,
    foothold window r and one gradient cell (traversability.py:76-213)."""
    pr = getattr(params, "step_patch_radius", None)
    pr = int(pr) if pr is not None else int(math.ceil(0.3 / r_g))
    return kside // 2 + pr + 1


def owner_band_np(y, y0, r_g, starts):
    """numpy statement of the device owner-band rule (for CPU tests)."""
    i = np.floor((np.asarray(y, np.float64) - y0) / r_g + 0.5)
    return np.searchsorted(np.asarray(starts[1:-1], np.float64), i, side="right")


# ---------------------------------------------------------------------------
# the simplify sweep replayed from (reduced) any() tables

def expand_table(table: np.ndarray) -> np.ndarray:
    """(S,) uint64 bit tables -> (S, 17) uint8: columns 0..15 = bits 0..15 (below =
    k-1-j), column 16 = bit 32 (no lower neighbour); max-reducible across ranks."""
    t = np.asarray(table, np.uint64)
    bits = list(range(KWIN)) + [KNONE]
    return np.stack([((t >> np.uint64(b)) & np.uint64(1)).astype(np.uint8) for b in bits], axis=1)


def replay_sweep(S: int, table_bytes: np.ndarray, triples_any):
    """The forward sweep of simplify.py:59-70 over any()s.

    table_bytes: (S, 17) uint8 from expand_table (already reduced over ranks).
    triples_any(list of (below, k, above)) -> list of bool (reduced over ranks).
    Returns the surviving slice indices."""
    keep = list(range(S))
    if S <= 1:
        return keep
    cache = {}

    def from_window(below, k, above):
        if not (above == k + 1 or (above < 0 and k == S - 1)):
            return None
        if below < 0:
            return bool(table_bytes[k, KWIN])
        if k - 1 - below < KWIN:
            return bool(table_bytes[k, k - 1 - below])
        return None

    while True:
        removed = False
        p = 0
        while p < len(keep):
            if len(keep) > 1:
                k = keep[p]
                below = keep[p - 1] if p > 0 else -1
                above = keep[p + 1] if p + 1 < len(keep) else -1
                u = from_window(below, k, above)
                if u is None:
                    key = (below, k, above)
                    if key not in cache:
                        batch = []
                        for q in range(p, len(keep)):
                            t = (keep[q - 1] if q > 0 else -1, keep[q],
                                 keep[q + 1] if q + 1 < len(keep) else -1)
                            if from_window(*t) is None and t not in cache and len(batch) < 256:
                                batch.append(t)
                        for t, f in zip(batch, triples_any(batch)):
                            cache[t] = bool(f)
                    u = cache[key]
                if not u:
                    del keep[p]
                    removed = True
                    continue
            p += 1
        if not removed:
            return keep


# ---------------------------------------------------------------------------
# the per-rank pipeline

@dataclass
class BandResult:
    rank: int
    size: int
    rows: int
    cols: int
    row0: int
    nrows: int
    heights: np.ndarray
    origin: tuple
    z_min: float
    keep: list
    # device tensors (torch) of the OWN rows, views into the extended stacks
    ground: object = None
    ceiling: object = None
    cost: object = None
    stages_ms: dict = field(default_factory=dict)
    # gather_to=root: the simplified tomogram assembled on the root rank
    tomogram: object = None


def _ptr(t, offset_elems=0):
    return t.data_ptr() + 4 * int(offset_elems)


def _torch_stream(device) -> int:
    """torch's current stream as a cudaStream_t for libpct.  torch's default
    stream is the legacy NULL stream, which pct_set_stream(NULL) would read
    as "the context's own stream" (non-blocking: no ordering with torch's
    work); it is passed as cudaStreamLegacy (0x1) instead."""
    import torch
    return torch.cuda.current_stream(device).cuda_stream or 1


def check_bands(starts, H: int):
    """Every band must be at least as thick as the halo its neighbours read
    from it.  Decided from the shared frame on every rank alike, before any
    point exchange, so either all ranks raise or none does."""
    size = len(starts) - 1
    rows = starts[-1]
    for b in range(size):
        nrows = starts[b + 1] - starts[b]
        need = max(min(H, rows - starts[b]) if b > 0 else 0,          # rank b-1's bottom halo
                   min(H, starts[b + 1]) if b + 1 < size else 0)      # rank b+1's top halo
        if need > nrows:
            raise ValueError(f"row band {b} has {nrows} rows, thinner than the {H}-row halo "
                             f"its neighbours need; use fewer ranks for this {rows}-row grid")


def _copy_slices(ctx, dst, dst_stride, src, src_stride, n, block, idx=None):
    """pct_copy_slices on device pointers (strides / sizes in floats), in
    launches of at most 4096 slices."""
    ix = np.arange(n, dtype=np.int32) if idx is None else np.ascontiguousarray(idx, np.int32)
    for a in range(0, int(n), 4096):
        b = min(int(n), a + 4096)
        sub = None if idx is None else ix[a:b]
        ctx.check(ctx.lib.pct_copy_slices(
            ctx.h, dst + 4 * a * int(dst_stride), int(dst_stride),
            src + (4 * a * int(src_stride) if idx is None else 0), int(src_stride),
            None if sub is None else sub.ctypes.data, b - a, int(block)), "copy_slices")


def band_pipeline(xyz, d_s, r_g, params, rank, size, *, device=None, eps_e=1e-6,
                  c_barrier=50.0, max_grid_side=16384, events=None, gather_to=None):
    """Generator: the row-band pipeline of one rank.

    xyz: this rank's points, a CUDA torch tensor (n, 3) float32/float64.
    Yields collective requests (tuples) and finally returns a BandResult.
    ``events`` (a dict) receives CUDA events recorded on the current stream
    around the evaluate launch ("evaluate" -> (start, end)) and its extent
    ("cell_slices").  ``gather_to`` = a rank: the surviving slices of every
    band are sent to that rank and assembled there into one reference-
    compatible ``Tomogram`` (``BandResult.tomogram``; tomogram.py:65-96)."""
    import torch

    ctx = _lib.context(device if device is not None else xyz.device.index)
    lib, h = ctx.lib, ctx.h
    # libpct and torch share one stream for the whole pipeline (ordering of
    # the NCCL buffers against the kernels); restored at the end
    ctx.check(lib.pct_set_stream(h, C.c_void_p(_torch_stream(xyz.device))), "set_stream")
    dt = torch.float32 if xyz.dtype == torch.float32 else torch.float64
    code = _lib.PCT_F32 if dt == torch.float32 else _lib.PCT_F64
    xyz = xyz.contiguous()
    n = xyz.shape[0]

    # 1. bounds -> global frame; a non-finite point on any rank fails every rank
    lo = np.full(3, np.inf)
    hi = np.full(3, -np.inf)
    bad = 0.0
    if n > 0:
        rc = lib.pct_bounds(h, xyz.data_ptr(), n, code, lo.ctypes.data, hi.ctypes.data)
        if rc == _lib.PCT_E_NONFINITE:
            bad, lo[:], hi[:] = 1.0, np.inf, -np.inf
        else:
            ctx.check(rc, "bounds")
    lo, hi, bad = yield ("bounds", lo, hi, bad)
    if bad:
        raise ValueError("point cloud contains non-finite coordinates")
    if not np.all(np.isfinite(lo)):
        from .cloud import CloudFormatError
        raise CloudFormatError("zero valid points")
    fr = _lib.FrameC()
    heights = np.empty(65536, np.float64)
    rc = lib.pct_frame_compute(lo.ctypes.data, hi.ctypes.data, float(d_s), float(r_g),
                               int(max_grid_side), C.byref(fr), heights.ctypes.data, 65536)
    if rc == _lib.PCT_E_GRID:
        from .tomogram import GridSizeError
        raise GridSizeError(f"grid {fr.rows}x{fr.cols} exceeds the {max_grid_side} per-side limit")
    if rc != 0:
        raise ValueError("d_s and r_g must be positive")
    S, rows, cols = fr.n_slices, fr.rows, fr.cols
    heights = heights[:S].copy()
    starts = band_starts(rows, size)
    row0, row1 = starts[rank], starts[rank + 1]
    nrows = row1 - row0
    from .traversability import build_kernel
    kern = build_kernel(params.d_inf, params.d_sm, r_g)
    w = np.ascontiguousarray(kern.weights)
    H = halo_rows(params, r_g, w.shape[0])
    check_bands(starts, H)

    # 2. partition by owner band, all-to-all (one band owns every point)
    if size == 1:
        mine = xyz
    else:
        part = torch.empty_like(xyz)
        counts = np.zeros(size, np.int64)
        st = np.asarray(starts, np.int32)
        if n > 0:
            ctx.check(lib.pct_partition_rows(h, xyz.data_ptr(), n, code, C.byref(fr),
                                             st.ctypes.data, size, part.data_ptr(),
                                             counts.ctypes.data), "partition")
        mine = yield ("alltoallv", part, counts.tolist())
        mine = mine.contiguous()

    # 3. banded build into the extended stack
    top = min(H, row0)
    bot = min(H, rows - row1)
    ext_rows = top + nrows + bot
    g = torch.empty((S, ext_rows, cols), dtype=torch.float32, device=xyz.device)
    c = torch.empty_like(g)
    stride = ext_rows * cols
    if nrows > 0:
        ctx.check(lib.pct_build_band(h, mine.data_ptr(), mine.shape[0], code, C.byref(fr),
                                     heights.ctypes.data, row0, nrows, stride,
                                     _ptr(g, top * cols), _ptr(c, top * cols)), "build_band")
    # 4. halo exchange: my first rows go up (to rank-1), my last rows go down;
    # packed into / unpacked from contiguous (2, S, rows, cols) buffers by libpct
    up_n = min(H, rows - row0) if rank > 0 else 0   # == rank-1's bottom halo
    down_n = min(H, row1) if rank + 1 < size else 0  # == rank+1's top halo

    def pack(first_row, nr):
        buf = torch.empty((2, S, nr, cols), dtype=torch.float32, device=xyz.device)
        for L, src in enumerate((g, c)):
            _copy_slices(ctx, _ptr(buf, L * S * nr * cols), nr * cols,
                         _ptr(src, first_row * cols), stride, S, nr * cols)
        return buf

    send_up = pack(top, up_n) if rank > 0 else None
    send_down = pack(top + nrows - down_n, down_n) if rank + 1 < size else None
    from_up, from_down = yield ("halo", send_up, send_down, (2, S, top, cols), (2, S, bot, cols))
    for buf, first_row, nr in ((from_up, 0, top), (from_down, top + nrows, bot)):
        if nr:
            buf = buf.contiguous()
            for L, dst in enumerate((g, c)):
                _copy_slices(ctx, _ptr(dst, first_row * cols), stride,
                             _ptr(buf, L * S * nr * cols), nr * cols, S, nr * cols)

    # 5. evaluate the extended band (own rows are exact)
    cost = torch.empty_like(g)
    pc = _lib.trav_params_c(params, r_g)
    if events is not None:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev0.record()
    ctx.check(lib.pct_evaluate(h, g.data_ptr(), c.data_ptr(), S, ext_rows, cols, float(r_g),
                               C.byref(pc), w.ctypes.data, w.shape[0], cost.data_ptr()),
              "evaluate")
    if events is not None:
        ev1 = torch.cuda.Event(enable_timing=True)
        ev1.record()
        events["evaluate"] = (ev0, ev1)
        events["cell_slices"] = S * ext_rows * cols

    # 6. simplify: reduced any() tables, shared sweep
    cells = nrows * cols
    table = np.zeros(S, np.uint64)
    ctx.check(lib.pct_simplify_window(h, _ptr(g, top * cols), _ptr(cost, top * cols), S, cells,
                                      stride, float(eps_e), float(c_barrier), table.ctypes.data),
              "simplify_window")
    tb = yield ("max_u8", expand_table(table))
    pending = {}

    def triples_any(batch):
        tri = np.asarray(batch, np.int32).reshape(-1)
        flags = np.zeros(len(batch), np.int32)
        ctx.check(lib.pct_simplify_triples(h, _ptr(g, top * cols), _ptr(cost, top * cols), S,
                                           cells, stride, float(eps_e), float(c_barrier),
                                           tri.ctypes.data, len(batch), flags.ctypes.data),
                  "simplify_triples")
        pending["local"] = flags.astype(np.uint8)
        return None

    # the sweep is replayed identically on every rank; each triple batch is a
    # collective (local flags -> max over ranks)
    keep_box = {}
    sweep = _sweep_gen(S, tb)
    req = next(sweep)
    while True:
        if req[0] == "done":
            keep_box["keep"] = req[1]
            break
        triples_any(req[1])
        red = yield ("max_u8", pending["local"])
        req = sweep.send([bool(v) for v in red])
    keep = keep_box["keep"]
    res = BandResult(rank=rank, size=size, rows=rows, cols=cols, row0=row0, nrows=nrows,
                     heights=heights, origin=(float(fr.origin_x), float(fr.origin_y)),
                     z_min=float(fr.z_min), keep=keep,
                     ground=g[:, top:top + nrows], ceiling=c[:, top:top + nrows],
                     cost=cost[:, top:top + nrows])

    # 7. gather the surviving slices on one rank
    if gather_to is not None:
        K = len(keep)
        if rank == gather_to:
            from .tomogram import new_device_stack
            stacks = [new_device_stack(ctx, K, rows, cols) for _ in range(3)]
            for L, src in enumerate((g, c, cost)):   # own band, straight from the ext stacks
                _copy_slices(ctx, stacks[L].ptr + 4 * row0 * cols, rows * cols,
                             _ptr(src, top * cols), stride, K, nrows * cols, idx=keep)
            shapes = [(3, K, starts[b + 1] - starts[b], cols) for b in range(size)]
            bands = yield ("gather", None, gather_to, shapes, xyz.device)
            for b, buf in enumerate(bands):
                if b == rank or buf is None:
                    continue
                buf = buf.contiguous()
                nb = starts[b + 1] - starts[b]
                for L in range(3):
                    _copy_slices(ctx, stacks[L].ptr + 4 * starts[b] * cols, rows * cols,
                                 _ptr(buf, L * K * nb * cols), nb * cols, K, nb * cols)
            res.tomogram = _assemble_tomogram(stacks, heights, keep, r_g, res.origin, d_s,
                                              res.z_min)
        else:
            buf = torch.empty((3, K, nrows, cols), dtype=torch.float32, device=xyz.device)
            for L, src in enumerate((g, c, cost)):
                _copy_slices(ctx, _ptr(buf, L * K * nrows * cols), nrows * cols,
                             _ptr(src, top * cols), stride, K, nrows * cols, idx=keep)
            yield ("gather", buf, gather_to, None, xyz.device)
    lib.pct_set_stream(h, None)
    return res


def _assemble_tomogram(stacks, heights, keep, r_g, origin, d_s, z_min):
    """The simplified Tomogram over full-grid device stacks (ground, ceiling,
    cost), as simplify_tomogram returns it (simplify.py:71-73: indices
    0..K-1, plane heights kept); Layer.values materialise on first access."""
    from .tomogram import Layer, Tomogram, TomogramSlice
    g, c, cost = stacks
    slices = [TomogramSlice(Layer.on_device(g, m, r_g, origin), Layer.on_device(c, m, r_g, origin),
                            float(heights[k]), m, Layer.on_device(cost, m, r_g, origin))
              for m, k in enumerate(keep)]
    return Tomogram(slices=slices, d_s=float(d_s), z_min=float(z_min))


# ---------------------------------------------------------------------------
# host gather: every rank DMAs its band of the surviving layers into one
# shared-memory segment on the node (its own PCIe link), the root wraps it

class _Segment:
    """One /dev/shm segment mapped (and page-locked for DMA) in this process."""

    def __init__(self, ctx, name, nbytes, create):
        import mmap
        import os
        path = "/dev/shm/" + name
        fd = os.open(path, (os.O_CREAT | os.O_EXCL | os.O_RDWR) if create else os.O_RDWR, 0o600)
        try:
            if create:
                os.ftruncate(fd, nbytes)
            self.mm = mmap.mmap(fd, nbytes)
        finally:
            os.close(fd)
        self.ctx, self.name, self.nbytes, self.path = ctx, name, nbytes, path
        self._anchor = C.c_char.from_buffer(self.mm)  # exported: the mapping stays put
        self.ptr = C.addressof(self._anchor)
        ctx.check(ctx.lib.pct_host_register(ctx.h, C.c_void_p(self.ptr), C.c_size_t(nbytes)),
                  "host_register")
        self.view = None  # root: weakref to the array handed out

    def free(self):
        return self.view is None or self.view() is None

    def release(self, unlink=False):
        try:
            self.ctx.lib.pct_host_unregister(self.ctx.h, C.c_void_p(self.ptr))
        except Exception:
            pass
        if unlink:
            _unlink(self.path)


def _unlink(path):
    import os
    try:
        os.unlink(path)
    except OSError:
        pass


def _unlink_root_segments():
    for seg in _ROOT_SEGS:
        _unlink(seg.path)


_ROOT_SEGS: list = []   # root: segments it created (reused while free)
_ATTACHED: dict = {}    # other ranks: name -> _Segment (the last few)


def _root_segment(ctx, nbytes):
    import os
    import uuid
    for seg in _ROOT_SEGS:
        if seg.nbytes == nbytes and seg.free() and seg.ctx is ctx:
            return seg, False
    while len(_ROOT_SEGS) >= 2 and any(sg.free() for sg in _ROOT_SEGS):  # drop an idle one
        old = next(sg for sg in _ROOT_SEGS if sg.free())
        _ROOT_SEGS.remove(old)
        old.release(unlink=True)
    if not _ROOT_SEGS:
        import atexit
        atexit.register(_unlink_root_segments)
    seg = _Segment(ctx, f"pct-{os.getpid()}-{uuid.uuid4().hex[:12]}", nbytes, create=True)
    _ROOT_SEGS.append(seg)
    return seg, True


def _attached_segment(ctx, name, nbytes):
    seg = _ATTACHED.get(name)
    if seg is None:
        seg = _Segment(ctx, name, nbytes, create=False)
        _ATTACHED[name] = seg
        while len(_ATTACHED) > 3:  # oldest attachments go (no views on this side)
            old = _ATTACHED.pop(next(iter(_ATTACHED)))
            old.release()
    return seg


def _host_gather(res, ctx, root, group, d_s, r_g):
    """The surviving slices of every band written by their own rank straight
    into one pinned shared-memory segment of the node, wrapped on the root as
    host-resident reference Layers (every rank's D2H runs on its own PCIe
    link; nothing crosses NVLink)."""
    import weakref

    import torch.distributed as dist
    rank = dist.get_rank(group)
    K, R, Cc = len(res.keep), res.rows, res.cols
    nbytes = 3 * K * R * Cc * 4
    box = [None, None]
    if rank == root:
        # a /dev/shm too small for the segment (containers default to 64 MB)
        # would fault on first touch: every rank sends its band to the root
        # instead (NCCL), which reads them back alone
        if _shm_free() >= nbytes + (256 << 20):
            seg, _ = _root_segment(ctx, nbytes)
            box = [seg.name, nbytes]
        else:
            box = ["", nbytes]
    dist.broadcast_object_list(box, src=_global(group, root), group=group)
    name, nb = box
    if not name:
        return _p2p_host_gather(res, ctx, root, group, d_s, r_g)
    seg = seg if rank == root else _attached_segment(ctx, name, nb)
    # this rank's rows of every kept slice of the three layers
    plane = R * Cc * 4
    band = res.nrows * Cc * 4
    with ctx.lock:
        for L, t in enumerate((res.ground, res.ceiling, res.cost)):
            sstride = t.stride(0) * 4
            for m, k in enumerate(res.keep):
                if band == 0:
                    continue
                dst = seg.ptr + (L * K + m) * plane + res.row0 * Cc * 4
                ctx.check(ctx.lib.pct_memcpy_d2h_async(ctx.h, C.c_void_p(dst),
                                                       C.c_void_p(t.data_ptr() + k * sstride),
                                                       C.c_size_t(band)), "d2h")
        ctx.check(ctx.lib.pct_sync(ctx.h), "sync")
    dist.barrier(group=group)  # every band landed; every rank attached the segment
    if rank != root:
        return None
    # (the segment's file stays in /dev/shm while the root may hand it out
    # again -- other ranks re-attach by name -- and is unlinked when dropped
    # from the pool or at exit)
    from .tomogram import Layer, Tomogram, TomogramSlice
    arr = np.frombuffer(seg.mm, np.float32, count=3 * K * R * Cc).reshape(3, K, R, Cc)
    seg.view = weakref.ref(arr)
    origin = res.origin
    slices = [TomogramSlice(Layer(arr[0, m], r_g, origin), Layer(arr[1, m], r_g, origin),
                            float(res.heights[k]), m, Layer(arr[2, m], r_g, origin))
              for m, k in enumerate(res.keep)]
    return Tomogram(slices=slices, d_s=float(d_s), z_min=float(res.z_min))


def _shm_free() -> int:
    import os
    try:
        st = os.statvfs("/dev/shm")
        return int(st.f_bavail) * int(st.f_frsize)
    except OSError:
        return 0


def _p2p_host_gather(res, ctx, root, group, d_s, r_g):
    """_host_gather without a shared segment: every rank packs its band of
    the kept slices (3, K, band rows, cols) on its GPU and sends it to the
    root (NCCL P2P; host-staged for gloo), which copies each band into one
    page-locked host array."""
    import torch
    import torch.distributed as dist
    rank, size = dist.get_rank(group), dist.get_world_size(group)
    nccl = dist.get_backend(group) == "nccl"
    K, R, Cc = len(res.keep), res.rows, res.cols
    dev = res.ground.device
    buf = torch.empty((3, K, res.nrows, Cc), dtype=torch.float32, device=dev)
    with ctx.lock:
        if K and res.nrows:
            for L, t in enumerate((res.ground, res.ceiling, res.cost)):
                _copy_slices(ctx, _ptr(buf, L * K * res.nrows * Cc), res.nrows * Cc, t.data_ptr(),
                             t.stride(0), K, res.nrows * Cc, idx=res.keep)
        ctx.check(ctx.lib.pct_sync(ctx.h), "sync")
    if rank != root:
        if buf.numel():
            dist.send(buf if nccl else buf.cpu(), dst=_global(group, root), group=group)
        return None
    arr = _lib.pinned_pool(ctx).array((3, K, R, Cc), np.float32)
    host = torch.from_numpy(arr)
    starts = band_starts(R, size)
    for b in range(size):
        a0, a1 = starts[b], starts[b + 1]
        if a1 == a0 or K == 0:
            continue
        if b == rank:
            part = buf
        else:
            part = torch.empty((3, K, a1 - a0, Cc), dtype=torch.float32,
                               device=dev if nccl else "cpu")
            dist.recv(part, src=_global(group, b), group=group)
        host[:, :, a0:a1, :].copy_(part)
    from .tomogram import Layer, Tomogram, TomogramSlice
    origin = res.origin
    slices = [TomogramSlice(Layer(arr[0, m], r_g, origin), Layer(arr[1, m], r_g, origin),
                            float(res.heights[k]), m, Layer(arr[2, m], r_g, origin))
              for m, k in enumerate(res.keep)]
    return Tomogram(slices=slices, d_s=float(d_s), z_min=float(res.z_min))


def tomogram_sharded(points, d_s: float, r_g: float, params=None, *, eps_e: float = 1e-6,
                     c_barrier: float = 50.0, root: int = 0, group=None, device=None,
                     max_grid_side: int = 16384, gather: str = "device"):
    """build_tomogram -> evaluate_tomogram -> simplify_tomogram of ONE map
    whose points are spread over the ranks of a torch.distributed group (one
    process per GPU), row-band sharded as in the module docstring.

    ``points``: this rank's share of the cloud -- a PointCloud, an (n, 3)
    float32/float64 host array (pinned memory uploads fastest) or a CUDA
    tensor; any split of the points over the ranks gives the same result.
    Returns on ``root`` the simplified reference-compatible ``Tomogram``
    (tomogram.py:65-96; bit-identical to the one-GPU chain), and None on the
    other ranks.  ``gather="device"``: the bands' surviving slices are sent to
    the root's GPU (NCCL) and its layers stay device-resident until
    ``materialize()`` / ``Layer.values``.  ``gather="host"`` (ranks on one
    node): every rank writes its band straight into one page-locked
    shared-memory segment over its own PCIe link and the root's layers are
    host numpy arrays on return -- the read-back of a large map spreads over
    all the GPUs' links.  With a one-rank group (or no process group) it runs
    the same band pipeline on one GPU."""
    import torch
    import torch.distributed as dist

    from .cloud import source_points
    from .traversability import TravParams
    params = params if params is not None else TravParams()
    single = not (dist.is_available() and dist.is_initialized())
    rank = 0 if single else dist.get_rank(group)
    size = 1 if single else dist.get_world_size(group)
    dev = torch.device("cuda", device if device is not None else torch.cuda.current_device())
    if isinstance(points, torch.Tensor):
        xyz = points.to(dev)
    else:
        arr = np.ascontiguousarray(source_points(points))
        if arr.dtype not in (np.float32, np.float64):
            arr = arr.astype(np.float64)
        ctx = _lib.context(dev.index)
        xyz = torch.empty(arr.shape, dtype=torch.float32 if arr.dtype == np.float32
                          else torch.float64, device=dev)
        stream = _torch_stream(dev)
        with ctx.lock:
            ctx.check(ctx.lib.pct_set_stream(ctx.h, C.c_void_p(stream)), "set_stream")
            ctx.check(ctx.lib.pct_memcpy_h2d(ctx.h, xyz.data_ptr(), arr.ctypes.data, arr.nbytes),
                      "h2d")
    if gather not in ("device", "host"):
        raise ValueError("gather must be 'device' or 'host'")
    host = gather == "host" and size > 1
    gen = band_pipeline(xyz, d_s, r_g, params, rank, size, device=dev.index, eps_e=eps_e,
                        c_barrier=c_barrier, max_grid_side=max_grid_side,
                        gather_to=None if host else (root if size > 1 else 0))
    res = run_virtual([gen])[0] if size == 1 else run_torch(gen, group)
    if host:
        return _host_gather(res, _lib.context(dev.index), root, group, d_s, r_g)
    if rank != root:
        return None
    return res.tomogram.materialize() if gather == "host" else res.tomogram


def _sweep_gen(S, tb):
    """replay_sweep as a generator: yields ("triples", batch) and receives the
    reduced any()s; the (deterministic) replay restarts with the answers
    known so far until it completes, then yields ("done", keep)."""
    answers = {}

    def lookup(batch):
        key = tuple(batch)
        if key not in answers:
            raise _NeedAny(batch)
        return answers[key]

    while True:
        try:
            keep = replay_sweep(S, tb, lookup)
        except _NeedAny as e:
            answers[tuple(e.batch)] = yield ("triples", e.batch)
            continue
        yield ("done", keep)
        return


class _NeedAny(Exception):
    def __init__(self, batch=None):
        super().__init__("any() needed")
        self.batch = batch


# ---------------------------------------------------------------------------
# drivers

def run_torch(gen, group=None):
    """Serve a band_pipeline generator with torch.distributed collectives.

    NCCL: device buffers straight over NVLink.  Gloo (CPU process groups:
    the multi-process tests): the same requests staged through host memory."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    size = dist.get_world_size(group)
    nccl = dist.get_backend(group) == "nccl"
    coll = _collective_device(group)

    def out(t):        # device buffer -> what the backend can send
        return t if (nccl or t is None) else t.cpu()

    def back(t, dev):  # what the backend received -> device buffer
        return t if (nccl or t is None) else t.to(dev)

    req = next(gen)
    while True:
        kind = req[0]
        if kind == "bounds":
            lo, hi, bad = req[1], req[2], req[3]
            t = torch.tensor(np.concatenate([-lo, hi, [bad]]), dtype=torch.float64, device=coll)
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
            v = t.cpu().numpy()
            ans = (-v[:3], v[3:6], float(v[6]))
        elif kind == "alltoallv":
            part, counts = req[1], req[2]
            dev = part.device
            cnt = torch.tensor(counts, dtype=torch.int64, device=coll)
            rcnt = torch.empty_like(cnt)
            dist.all_to_all_single(rcnt, cnt, group=group)
            rc = rcnt.cpu().tolist()
            src = out(part)
            res = torch.empty((int(sum(rc)), 3), dtype=part.dtype, device=src.device)
            dist.all_to_all_single(res, src, output_split_sizes=rc, input_split_sizes=counts,
                                   group=group)
            ans = back(res, dev)
        elif kind == "halo":
            send_up, send_down, up_shape, down_shape = req[1:]
            ref = send_up if send_up is not None else send_down
            dev = ref.device if ref is not None else coll
            bdev = dev if nccl else torch.device("cpu")
            recv_up = torch.empty(up_shape, dtype=torch.float32, device=bdev)
            recv_down = torch.empty(down_shape, dtype=torch.float32, device=bdev)
            ops = []
            if send_up is not None:
                ops.append(dist.P2POp(dist.isend, out(send_up), _global(group, rank - 1), group))
            if send_down is not None:
                ops.append(dist.P2POp(dist.isend, out(send_down), _global(group, rank + 1), group))
            if up_shape[2] > 0:
                ops.append(dist.P2POp(dist.irecv, recv_up, _global(group, rank - 1), group))
            if down_shape[2] > 0:
                ops.append(dist.P2POp(dist.irecv, recv_down, _global(group, rank + 1), group))
            if ops:
                for r in dist.batch_isend_irecv(ops):
                    r.wait()
            ans = (back(recv_up, dev), back(recv_down, dev))
        elif kind == "max_u8":
            t = torch.from_numpy(np.ascontiguousarray(req[1])).to(coll)
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
            ans = t.cpu().numpy()
        elif kind == "gather":
            buf, root, shapes, dev = req[1], req[2], req[3], req[4]
            if rank == root:
                bdev = dev if nccl else torch.device("cpu")
                bufs = [None if b == rank else torch.empty(shapes[b], dtype=torch.float32,
                                                           device=bdev)
                        for b in range(size)]
                ops = [dist.P2POp(dist.irecv, bufs[b], _global(group, b), group)
                       for b in range(size) if b != rank and bufs[b].numel() > 0]
                if ops:
                    for r in dist.batch_isend_irecv(ops):
                        r.wait()
                ans = [back(b, dev) for b in bufs]
            else:
                if buf.numel() > 0:
                    for r in dist.batch_isend_irecv([dist.P2POp(dist.isend, out(buf),
                                                                _global(group, root), group)]):
                        r.wait()
                ans = None
        else:
            raise RuntimeError(f"unknown collective {kind}")
        try:
            req = gen.send(ans)
        except StopIteration as stop:
            return stop.value


def _global(group, r):
    import torch.distributed as dist
    return r if group is None else dist.get_global_rank(group, r)


def _collective_device(group):
    import torch
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def run_virtual(gens):
    """Run P band_pipeline generators in lockstep in one process (one GPU):
    the collectives are performed by direct tensor / array operations."""
    import torch
    if not gens:
        return []

    P = len(gens)
    reqs = [next(g) for g in gens]
    results = [None] * P
    while True:
        kinds = {r[0] for r in reqs}
        assert len(kinds) == 1, f"ranks out of step: {kinds}"
        kind = kinds.pop()
        if kind == "bounds":
            lo = np.min([r[1] for r in reqs], axis=0)
            hi = np.max([r[2] for r in reqs], axis=0)
            bad = max(r[3] for r in reqs)
            answers = [(lo.copy(), hi.copy(), bad) for _ in range(P)]
        elif kind == "alltoallv":
            offs = [np.concatenate([[0], np.cumsum(r[2])]) for r in reqs]
            answers = []
            for dst in range(P):
                pieces = [reqs[src][1][int(offs[src][dst]):int(offs[src][dst + 1])]
                          for src in range(P)]
                answers.append(torch.cat(pieces) if pieces else None)
        elif kind == "halo":
            answers = []
            for r in range(P):
                up = reqs[r - 1][2] if r > 0 else None          # rank-1's send_down
                down = reqs[r + 1][1] if r + 1 < P else None    # rank+1's send_up
                answers.append((up, down))
        elif kind == "max_u8":
            m = np.max([r[1] for r in reqs], axis=0)
            answers = [m.copy() for _ in range(P)]
        elif kind == "gather":
            root = reqs[0][2]
            bufs = [r[1] for r in reqs]
            answers = [bufs if i == root else None for i in range(P)]
        else:
            raise RuntimeError(kind)
        done = 0
        for i, g in enumerate(gens):
            if results[i] is not None:
                done += 1
                continue
            try:
                reqs[i] = g.send(answers[i])
            except StopIteration as stop:
                results[i] = stop.value
                done += 1
        if done == P:
            return results
