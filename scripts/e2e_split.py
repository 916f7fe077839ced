"""Where the cfg3 drop-in e2e step spends its time (diagnostic): raw pinned
H2D of the points, build (upload + device build), evaluate, simplify,
materialize; each stage synchronised and wall-clocked, 5 repetitions."""
import os
import time

import numpy as np
import torch

import paper_2403_07631_b200 as pct
from paper_2403_07631_b200 import _lib, synth

ctx = _lib.context(0)
CFG = int(os.environ.get("CFG", "3"))
xyz = synth.generate(CFG)
d_s, r_g = synth.CONFIGS[CFG]["d_s"], synth.CONFIGS[CFG]["r_g"]
pin = _lib.PinnedBuffer(ctx, xyz.shape, np.float32)
pin.array[...] = xyz
cloud = pct.PointCloud(pin.array)
dev = torch.empty(xyz.nbytes, dtype=torch.uint8, device="cuda")
src = torch.from_numpy(pin.array.view(np.uint8).reshape(-1))
params = pct.TravParams()
for rep in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dev.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    tom = pct.build_tomogram(cloud, d_s, r_g, device=0)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    ev = pct.evaluate_tomogram(tom, params)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    simp = pct.simplify_tomogram(ev)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    simp.materialize()
    t5 = time.perf_counter()
    print(f"rep {rep}: raw H2D {1e3*(t1-t0):.1f} ms ({xyz.nbytes/(t1-t0)/1e9:.1f} GB/s) | build {1e3*(t2-t1):.1f} "
          f"evaluate {1e3*(t3-t2):.1f} simplify {1e3*(t4-t3):.1f} materialize {1e3*(t5-t4):.1f} | "
          f"chain {1e3*(t5-t1):.1f} ms", flush=True)
    del tom, ev, simp
