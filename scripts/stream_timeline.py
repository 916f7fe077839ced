"""Timeline of stream_maps on one config: per map, host timestamps of
pct_tomo_run start/end and read-back start/end (workers=2)."""
import sys, threading, time
import numpy as np
import paper_2403_07631_b200 as pct
from paper_2403_07631_b200 import _lib, synth, batch, tomogram
from paper_2403_07631_b200.batch import BatchRunner, stream_maps

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
xyz = synth.generate(cfg)
d_s, r_g = synth.CONFIGS[cfg]["d_s"], synth.CONFIGS[cfg]["r_g"]
r0 = BatchRunner(0, workers=1)
pin = _lib.PinnedBuffer(r0.ctxs[0], xyz.shape, np.float32)
pin.array[...] = xyz
T = []
orig_mat = tomogram.Tomogram.materialize
def mat(self):
    t0 = time.perf_counter(); out = orig_mat(self); T.append(("mat", threading.get_ident() % 997, t0, time.perf_counter())); return out
tomogram.Tomogram.materialize = mat
orig_run = _lib.Context.check
run = BatchRunner(0, workers=2)
lib = run.ctxs[0].lib
real = lib.pct_tomo_run
def timed(*a):
    t0 = time.perf_counter(); rc = real(*a); T.append(("run", threading.get_ident() % 997, t0, time.perf_counter())); return rc
class L:  # proxy so the worker's ctx.lib.pct_tomo_run is timed
    def __init__(s, l): s.l = l
    def __getattr__(s, n): return timed if n == "pct_tomo_run" else getattr(s.l, n)
for c in run.ctxs:
    c.lib = L(c.lib)
for t in stream_maps([pin.array] * 8, d_s, r_g, pct.TravParams(), runner=run):
    pass
T.clear()
t0 = time.perf_counter()
K = 10
for t in stream_maps([pin.array] * K, d_s, r_g, pct.TravParams(), runner=run):
    T.append(("yield", 0, time.perf_counter(), time.perf_counter()))
dt = (time.perf_counter() - t0) / K * 1e3
print(f"{dt:.3f} ms/map")
for kind, th, a, b in sorted(T, key=lambda x: x[2]):
    print(f"{kind:5s} {th:4d} {(a - t0) * 1e3:8.3f} {(b - t0) * 1e3:8.3f} {(b - a) * 1e3:7.3f}")
