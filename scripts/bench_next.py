"""Measurement of the SURVEY.md §8 f rows (the callers / formats either side of
the hot path) on the cfg1 map, one JSON line per row:

  lga       archive_bytes (device layers DMA'd into the LGA image)   tomogram.py:219-276
  planner   pct_planner_context (canonical-node run merge)           planner.py:62-93
  pcd       binary PCD file -> HBM points (pct_pcd_load)             cloud_io.py:123-146
  ceiling   pct_ceiling_inflate for every slice                       trajectory.py:277-317

Device times: CUDA events on the library stream after warm-up (median of
--steps).  Wall times: time.perf_counter around the public call.  The CPU
column is the oracle restatement (numpy, test infrastructure) on the same
input; the pcd CPU figure is the reference loader's own steps (read + record
view + stack + float64 + finite filter).  Usage:

    python scripts/bench_next.py [--steps 10] [--rows lga,planner,pcd,ceiling]
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def med(xs):
    return float(statistics.median(xs))


def peak_gbs():
    p = ROOT / "MEASURED_PEAKS.json"
    return float(json.loads(p.read_text())["hbm_gbs"]) if p.exists() else 6650.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--rows", default="lga,planner,pcd,ceiling")
    args = ap.parse_args()
    rows = args.rows.split(",")

    import torch
    import paper_2403_07631_b200 as pct
    from paper_2403_07631_b200 import _lib, synth
    torch.cuda.set_device(0)
    ctx = _lib.context(0)
    stream = torch.cuda.Stream()  # a real stream: the legacy default (handle 0) would
    torch.cuda.set_stream(stream)  # reset the library to its own stream
    ctx.check(ctx.lib.pct_set_stream(ctx.h, C.c_void_p(stream.cuda_stream)), "set_stream")
    peak = peak_gbs()

    def dev_time(fn, steps=args.steps):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            b.synchronize()
            ts.append(a.elapsed_time(b))
        return med(ts)

    def wall_time(fn, steps=args.steps):
        fn()
        ts = []
        for _ in range(steps):
            t = time.perf_counter()
            fn()
            ts.append((time.perf_counter() - t) * 1e3)
        return med(ts)

    cfg = synth.CONFIGS[1]
    xyz = synth.generate(1)
    tom = pct.build_tomogram(pct.PointCloud(xyz), cfg["d_s"], cfg["r_g"])
    ev = pct.evaluate_tomogram(tom, pct.TravParams())
    simp = pct.simplify_tomogram(ev)
    S, R, Cc = len(ev.slices), ev.rows, ev.cols
    base = dict(workload=f"cfg1 spiral_ramp: {len(xyz)} pts, grid {R}x{Cc}, {S} slices "
                f"({len(simp.slices)} after simplify)", data="synthetic (seeded)")
    out = []

    if "lga" in rows:
        from paper_2403_07631_b200.archive import archive_bytes
        from oracle.archive import lga_bytes
        nbytes = archive_bytes(simp).nbytes
        w = wall_time(lambda: archive_bytes(simp))
        gs, cs, ks = simp.ground_stack(), simp.ceiling_stack(), simp.cost_stack()
        hts = [s.plane_height for s in simp.slices]
        t = time.perf_counter()
        lga_bytes(gs, cs, ks, hts, simp.origin, simp.resolution, simp.z_min, simp.d_s)
        cpu = (time.perf_counter() - t) * 1e3
        out.append(dict(row="lga", metric="LGA archive image of the simplified map",
                        value=nbytes / w / 1e6, unit="GB/s", wall_ms=w, bytes=nbytes,
                        note="D2H of the surviving layers into the pinned archive buffer "
                             "(PCIe bound)", cpu_baseline=dict(ms=cpu, kind="port", cores=1)))

    if "planner" in rows:
        from paper_2403_07631_b200.planner_ctx import attach_planner_context
        from oracle.planner_ctx import planner_context
        gst = simp.ground_stack()
        kst = simp.cost_stack()
        Sk = gst.shape[0]
        g_dev = _lib.DeviceBuffer.from_host(ctx, gst)
        k_dev = _lib.DeviceBuffer.from_host(ctx, kst)
        canon = _lib.DeviceBuffer(ctx, gst.size * 4)
        cn = _lib.DeviceBuffer(ctx, gst.size * 4)
        d = dev_time(lambda: ctx.check(ctx.lib.pct_planner_context(
            ctx.h, g_dev.ptr, k_dev.ptr, Sk, R, Cc, 1e-6, canon.ptr, cn.ptr), "planner"))
        w = wall_time(lambda: attach_planner_context(simp), steps=3)
        t = time.perf_counter()
        planner_context(gst, kst)
        cpu = (time.perf_counter() - t) * 1e3
        alg = gst.size * 16  # read ground + cost, write canon + cn
        out.append(dict(row="planner", metric="planner context precompute", value=d,
                        unit="ms (device)", wall_ms=w, algorithmic_bytes=alg,
                        roofline=dict(bound="hbm", achieved=alg / d / 1e6, peak=peak,
                                      unit="GB/s", frac=alg / d / 1e6 / peak),
                        cpu_baseline=dict(ms=cpu, kind="port", cores=1)))

    if "pcd" in rows:
        from paper_2403_07631_b200 import cloud_io
        from oracle import cloud_io as ocio
        n = len(xyz)
        rec = np.zeros(n, [("x", "<f4"), ("y", "<f4"), ("z", "<f4"), ("intensity", "<f4")])
        rec["x"], rec["y"], rec["z"] = xyz[:, 0], xyz[:, 1], xyz[:, 2]
        rec["intensity"] = 1.0
        rec["z"][::1000] = np.nan
        head = ("VERSION 0.7\nFIELDS x y z intensity\nSIZE 4 4 4 4\nTYPE F F F F\n"
                f"COUNT 1 1 1 1\nWIDTH {n}\nHEIGHT 1\nPOINTS {n}\nDATA binary\n").encode()
        d = Path(tempfile.mkdtemp())
        path = d / "cfg1.pcd"
        path.write_bytes(head + rec.tobytes())
        w = wall_time(lambda: cloud_io.load_cloud(path, "pcd_binary"))
        r_dev = _lib.DeviceBuffer.from_host(ctx, rec)
        o_dev = _lib.DeviceBuffer(ctx, n * 12)
        offs = (C.c_int64 * 3)(0, 4, 8)
        nv = C.c_int64()
        dk = dev_time(lambda: ctx.check(ctx.lib.pct_pcd_extract(
            ctx.h, r_dev.ptr, n, 16, offs, 0, o_dev.ptr, C.byref(nv)), "pcd_extract"))
        t = time.perf_counter()
        raw = path.read_bytes()
        ocio.extract(raw[len(head):], n, 16, (0, 4, 8))
        cpu = (time.perf_counter() - t) * 1e3
        alg = n * 16 + nv.value * 12
        out.append(dict(row="pcd", metric="binary PCD ingest (file -> HBM points)",
                        value=n / w / 1e3, unit="Mpts/s (wall, file in page cache)", wall_ms=w,
                        file_bytes=len(head) + rec.nbytes, device_extract_ms=dk,
                        roofline=dict(bound="hbm", kernel="pcd extract (count+offsets+write)",
                                      achieved=alg / dk / 1e6, peak=peak, unit="GB/s",
                                      frac=alg / dk / 1e6 / peak),
                        cpu_baseline=dict(ms=cpu, kind="port", cores=1,
                                          sample="read + record view + float64 + finite filter")))
        os.remove(path)

    if "ceiling" in rows:
        from oracle import trajectory as otraj
        from paper_2403_07631_b200.tomogram import device_run
        st, first = device_run([s.ceiling for s in tom.slices])
        n = S * R * Cc
        f_dev = _lib.DeviceBuffer(ctx, n * 8)
        s_dev = _lib.DeviceBuffer(ctx, n * 8)
        dk = dev_time(lambda: ctx.check(ctx.lib.pct_ceiling_inflate(
            ctx.h, st.slice_ptr(first), S, R, Cc, 0.1, 0.20, 0.30, f_dev.ptr, s_dev.ptr),
            "ceiling_inflate"))
        sample = list(range(0, S, max(1, S // 4)))[:4]
        t = time.perf_counter()
        for k in sample:
            c = tom.slices[k].ceiling.values
            otraj.inflate_ceiling(c, np.isfinite(c), 0.1, 0.20, 0.30)
        cpu = (time.perf_counter() - t) * 1e3 / len(sample) * S
        alg = n * (4 + 8 + 8)  # read ceiling, write flat + skirted
        out.append(dict(row="ceiling", metric="ceiling inflation, all slices",
                        value=dk, unit="ms (device)", slices=S, sweeps=27,
                        algorithmic_bytes=alg,
                        roofline=dict(bound="hbm", achieved=alg / dk / 1e6, peak=peak,
                                      unit="GB/s", frac=alg / dk / 1e6 / peak),
                        cpu_baseline=dict(ms=cpu, kind="port", cores=1,
                                          sample=f"{len(sample)} slices, scaled to {S}")))

    for o in out:
        o.update(base)
        print(json.dumps(o))


if __name__ == "__main__":
    main()
