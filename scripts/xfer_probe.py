"""Phase timing of the compacted materialize on cfg3 (diagnostic)."""
import os
import time

import numpy as np

import paper_2403_07631_b200 as pct
from paper_2403_07631_b200 import _lib, synth
from paper_2403_07631_b200.tomogram import XFER_MIN_EMPTY

xyz = synth.generate(3)
pin = _lib.PinnedBuffer(_lib.context(0), xyz.shape, np.float32)
pin.array[...] = xyz
cloud = pct.PointCloud(pin.array)
for rep in range(4):
    tom = pct.simplify_tomogram(pct.evaluate_tomogram(pct.build_tomogram(cloud, 0.5, 0.1, device=0),
                                                      pct.TravParams()))
    ctx = _lib.context(0)
    ctx.check(ctx.lib.pct_sync(ctx.h), "sync")
    t0 = time.perf_counter()
    groups = {}
    for s in tom.slices:
        for l in (s.ground, s.ceiling, s.cost):
            groups.setdefault(id(l._stack), (l._stack, []))[1].append(l._k)
    plan = []
    for stack, ks in groups.values():
        ks = sorted(set(ks))
        cells = stack.rows * stack.cols
        tot = stack.count_nonempty(ks)
        ck = [k for k, t in zip(ks, tot) if t <= (1 - XFER_MIN_EMPTY) * cells]
        ct = [int(t) for k, t in zip(ks, tot) if t <= (1 - XFER_MIN_EMPTY) * cells]
        plan.append((stack, [k for k in ks if k not in set(ck)], ck, ct))
    t1 = time.perf_counter()
    pending = [(st, st.compact_start(ck, ct)) for st, _, ck, ct in plan if ck]
    ctx.check(ctx.lib.pct_xfer_fence(ctx.h), "f")
    for st, ks, _, _ in plan:
        if ks:
            st.prefetch(ks, sync=False)
    t2 = time.perf_counter()
    ctx.check(ctx.lib.pct_xfer_wait(ctx.h), "w")
    t3 = time.perf_counter()
    for st, p in pending:
        st.compact_finish(p, int(os.environ.get("PCT_XFER_THREADS", os.cpu_count())))
    t4 = time.perf_counter()
    ctx.check(ctx.lib.pct_sync(ctx.h), "sync")
    t5 = time.perf_counter()
    nc = sum(len(ck) for _, _, ck, _ in plan)
    nd = sum(len(ks) for _, ks, _, _ in plan)
    packed = sum(sum(ct) for _, _, _, ct in plan) * 4
    print(f"rep {rep}: count {1e3*(t1-t0):.1f} ms, issue {1e3*(t2-t1):.1f}, wait compact "
          f"{1e3*(t3-t2):.1f}, expand {1e3*(t4-t3):.1f}, rest dense {1e3*(t5-t4):.1f}, total "
          f"{1e3*(t5-t0):.1f} ms; compacted slices {nc} ({packed/1e9:.2f} GB packed), dense {nd}",
          flush=True)
