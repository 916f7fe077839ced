"""Probe the cfg3 end-to-end path: NaN share of the surviving layers, and the
host-side costs of the copies (pinned D2H rate, a pageable copy, a masked
expand).  Diagnostic only (not part of the bench)."""
import os
import time

import numpy as np

import paper_2403_07631_b200 as pct
from paper_2403_07631_b200 import _lib, synth

xyz = synth.generate(3)
pin = _lib.PinnedBuffer(_lib.context(0), xyz.shape, np.float32)
pin.array[...] = xyz
cloud = pct.PointCloud(pin.array)
for rep in range(3):
    t0 = time.perf_counter()
    tom = pct.build_tomogram(cloud, 0.5, 0.1, device=0)
    t1 = time.perf_counter()
    ev = pct.evaluate_tomogram(tom, pct.TravParams())
    simp = pct.simplify_tomogram(ev)
    t2 = time.perf_counter()
    simp.materialize()
    t3 = time.perf_counter()
    nb = sum(l.values.nbytes for s in simp.slices for l in (s.ground, s.ceiling, s.cost))
    print(f"rep {rep}: build(+upload) {1e3*(t1-t0):.1f} ms, eval+simplify {1e3*(t2-t1):.1f} ms, "
          f"materialize {1e3*(t3-t2):.1f} ms for {nb/1e9:.2f} GB = {nb/(t3-t2)/1e9:.1f} GB/s", flush=True)
for name in ("ground", "ceiling", "cost"):
    fr = [float(np.isnan(getattr(s, name).values).mean()) for s in simp.slices]
    print(name, "NaN share per kept slice: mean %.3f min %.3f max %.3f" % (np.mean(fr), min(fr), max(fr)))
# equal-to-previous-kept-slice share
for name in ("ground", "ceiling", "cost"):
    v = [getattr(s, name).values.view(np.uint32) for s in simp.slices]
    eq = [float((v[i] == v[i - 1]).mean()) for i in range(1, len(v))]
    print(name, "share equal to the previous kept slice: mean %.3f" % np.mean(eq))
a = simp.slices[5].ceiling.values
m = ~np.isnan(a)
vals = a[m]
t0 = time.perf_counter()
for _ in range(5):
    out = np.full(a.shape, np.nan, np.float32)
    out[m] = vals
t1 = time.perf_counter()
print(f"numpy masked expand of one slice: {(t1-t0)/5*1e3:.1f} ms ({a.nbytes/((t1-t0)/5)/1e9:.1f} GB/s)")
t0 = time.perf_counter()
for _ in range(5):
    b = a.copy()
t1 = time.perf_counter()
print(f"numpy copy of one slice: {(t1-t0)/5*1e3:.1f} ms ({a.nbytes/((t1-t0)/5)/1e9:.1f} GB/s)")
print("cpus", os.cpu_count())
