"""materialize() time of the cfg3 drop-in chain per read-back mode
(PCT_XFER_COMPACT = 0 dense, 1 NaN-compacted, last = delta chain for the
cost stack, delta = delta chains for every stack).  Diagnostic only."""
import os
import time

import numpy as np

import paper_2403_07631_b200 as pct
from paper_2403_07631_b200 import _lib, synth

xyz = synth.generate(3)
pin = _lib.PinnedBuffer(_lib.context(0), xyz.shape, np.float32)
pin.array[...] = xyz
cloud = pct.PointCloud(pin.array)
for mode in ("1", "nan", "1", "0"):
    os.environ["PCT_XFER_COMPACT"] = mode
    ts = []
    for rep in range(3):
        tom = pct.simplify_tomogram(pct.evaluate_tomogram(
            pct.build_tomogram(cloud, 0.5, 0.1, device=0), pct.TravParams()))
        ctx = _lib.context(0)
        ctx.check(ctx.lib.pct_sync(ctx.h), "sync")
        t0 = time.perf_counter()
        tom.materialize()
        ts.append(time.perf_counter() - t0)
        xb = getattr(tom, "xfer_bytes", 0)
        del tom
    print(f"mode {mode}: materialize {1e3*min(ts):.1f} ms (reps {[round(1e3*t,1) for t in ts]}), "
          f"PCIe bytes {xb/1e9:.2f} GB", flush=True)
