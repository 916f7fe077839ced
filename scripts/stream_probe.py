"""ms per map of stream_maps for several worker counts, with pinned-pool
misses and the per-map split between pct_tomo_run and the read-back."""
import sys, threading, time
import numpy as np
import paper_2403_07631_b200 as pct
from paper_2403_07631_b200 import _lib, synth, batch, tomogram
from paper_2403_07631_b200.batch import BatchRunner, stream_maps

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
xyz = synth.generate(cfg)
d_s, r_g = synth.CONFIGS[cfg]["d_s"], synth.CONFIGS[cfg]["r_g"]
r = BatchRunner(0, workers=1)
pin = _lib.PinnedBuffer(r.ctxs[0], xyz.shape, np.float32)
pin.array[...] = xyz

misses = [0]
orig_alloc = _lib.Context.check
orig_array = _lib.PinnedPool.array
def array(self, shape, dtype, ctx=None):
    size = self._class(int(np.prod(shape)) * np.dtype(dtype).itemsize)
    with self.lock:
        if not self.free.get(size):
            misses[0] += 1
    return orig_array(self, shape, dtype, ctx)
_lib.PinnedPool.array = array
phase = []
orig_mat = tomogram.Tomogram.materialize
def mat(self):
    t0 = time.perf_counter()
    out = orig_mat(self)
    phase.append(("mat", threading.get_ident() % 1000, t0, time.perf_counter()))
    return out
tomogram.Tomogram.materialize = mat

T0 = time.perf_counter()
for w in (1, 2, 3):
    run = BatchRunner(0, workers=w)
    for t in stream_maps([pin.array] * 6, d_s, r_g, pct.TravParams(), runner=run):
        pass
    K = 12
    misses[0] = 0
    phase.clear()
    t0 = time.perf_counter()
    tl = []
    for t in stream_maps([pin.array] * K, d_s, r_g, pct.TravParams(), runner=run):
        tl.append(time.perf_counter() - t0)
    dt = (time.perf_counter() - t0) / K
    print(f"workers {w}: {dt*1e3:.3f} ms/map; pool misses {misses[0]}; yields at",
          " ".join(f"{x*1e3:.1f}" for x in tl))
    print("   materialize (thread, start, end ms):",
          " ".join(f"{p[1]}:{(p[2]-t0)*1e3:.1f}-{(p[3]-t0)*1e3:.1f}" for p in phase))
    run.close()
