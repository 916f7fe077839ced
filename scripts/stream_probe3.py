"""stream_maps over the cfg3 cloud (diagnostic): ms per map with two maps in flight."""
import os
import time

import numpy as np
import torch

import paper_2403_07631_b200 as pct
from paper_2403_07631_b200 import _lib, synth
from paper_2403_07631_b200.batch import BatchRunner, stream_maps

print("host MemTotal/MemAvailable:", [l.strip() for l in open("/proc/meminfo") if l.startswith(("MemTotal", "MemAvailable"))])
xyz = synth.generate(3)
ctx = _lib.context(0)
pin = _lib.PinnedBuffer(ctx, xyz.shape, np.float32)
pin.array[...] = xyz
params = pct.TravParams()
run = BatchRunner(0, workers=int(os.environ.get("W", "2")))
for rep in range(3):
    n = 6
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for tom in stream_maps([pin.array] * n, 0.5, 0.1, params, runner=run):
        for s in tom.slices:
            _ = s.ground.values, s.ceiling.values, s.cost.values
        del tom
    t = (time.perf_counter() - t0) / n
    print(f"rep {rep}: {1e3 * t:.1f} ms / map streamed", flush=True)
run.close()
