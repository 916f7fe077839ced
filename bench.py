"""Benchmark of the B200 tomogram hot path: bounds -> build -> evaluate -> simplify.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl b200|reference]

One "step" = one pass of the hot path over one synthetic map (BASELINE.json
config C, default 1: 5M points, 0.1 m, d_s 0.4), inputs resident in HBM.
Prints ONE JSON line (rank 0).  Under torchrun each rank processes its own
independently seeded map (weak scaling, no data-path collective: batches of
independent maps are distributed without communication, BASELINE config 4);
time = max over ranks of the device time of K steps.

--impl reference times the reference algorithm's CPU implementation (the
pinned numpy port in oracle/, the reference package cannot travel to the box)
on the same map with all host threads; rank 0 only.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from paper_2403_07631_b200 import synth  # noqa: E402

METRIC = "tomogram build+eval ms/map & Mpts/s at 1/2/4/8 B200; % HBM peak; vs CPU ref"
L2_FLUSH_BYTES = 256 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--points", type=int, default=None, help="override the config's N")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--profile", action="store_true", help="1 warm-up + 1 step, no extras (ncu)")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def workload(args, rank):
    cfg = synth.CONFIGS[args.config]
    n = args.points or cfg["n_points"]
    seed = cfg["seed"] + rank
    xyz = synth.generate(args.config, n, seed)
    return cfg, xyz, seed


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth)"
    return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


class ClockSampler:
    """SM clock + clock-event (throttle) reasons polled through NVML (the
    library nvidia-smi reads) every ~0.5 ms while the timed region runs —
    the region lasts only milliseconds, too short for nvidia-smi -lms."""

    def __init__(self, device):
        self.device = device
        self.samples = []
        self.stop = threading.Event()
        self.ok = False

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.hd = N.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.hd, N.NVML_CLOCK_SM)
            self.ok = True
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
        except Exception as e:  # no NVML: report unsampled
            self.err = repr(e)
        return self

    def _poll(self):
        N = self.N
        while not self.stop.is_set():
            try:
                sm = N.nvmlDeviceGetClockInfo(self.hd, N.NVML_CLOCK_SM)
                rs = N.nvmlDeviceGetCurrentClocksEventReasons(self.hd)
                self.samples.append((sm, rs))
            except Exception:
                pass
            time.sleep(0.0005)

    def __exit__(self, *a):
        self.stop.set()
        if self.ok:
            self.t.join(1.0)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        N = self.N
        names = {N.nvmlClocksEventReasonHwSlowdown: "hw_slowdown",
                 N.nvmlClocksEventReasonHwThermalSlowdown: "hw_thermal_slowdown",
                 N.nvmlClocksEventReasonSwThermalSlowdown: "sw_thermal_slowdown",
                 N.nvmlClocksEventReasonSwPowerCap: "sw_power_cap"}
        reasons = sorted({nm for _, rs in self.samples for bit, nm in names.items() if rs & bit})
        return {"sm_mhz": statistics.median(s for s, _ in self.samples),
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.samples),
                "source": "NVML polled during the timed region"}


# ---------------------------------------------------------------------------
# reference arm / CPU baseline (the pinned numpy port of the reference)

def cpu_pipeline(xyz, cfg, threads):
    import oracle
    from paper_2403_07631_b200.traversability import TravParams
    TABLE_PARAMS = TravParams()
    t0 = time.perf_counter()
    t = oracle.build(xyz, cfg["d_s"], cfg["r_g"], threads=threads)
    t1 = time.perf_counter()
    cost = oracle.evaluate(t["ground"], t["ceiling"], cfg["r_g"], TABLE_PARAMS, threads=threads)
    t2 = time.perf_counter()
    keep = oracle.simplify(t["ground"], cost)
    t3 = time.perf_counter()
    return (t3 - t0), dict(build=t1 - t0, evaluate=t2 - t1, simplify=t3 - t2), len(keep)


def cpu_model():
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    cfg, xyz, seed = workload(args, 0)
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_pipeline(xyz, cfg, threads)
    times, stages = [], []
    for _ in range(args.steps):
        t, st, keep = cpu_pipeline(xyz, cfg, threads)
        times.append(t)
        stages.append(st)
    ms = 1e3 * statistics.mean(times)
    mpts = len(xyz) / (ms * 1e3)
    line = {
        "impl": "reference", "metric": METRIC, "value": mpts, "unit": "Mpts/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"cfg{args.config} {cfg['name']}", "n_points": len(xyz),
                   "seed": seed, "r_g": cfg["r_g"], "d_s": cfg["d_s"]},
        "stages_ms": {k: 1e3 * statistics.mean(s[k] for s in stages) for k in stages[0]},
        "cpu_baseline": {"value": mpts, "unit": "Mpts/s", "cores": threads, "kind": "port",
                         "sample": f"full cfg{args.config} map per step (build+evaluate+simplify),"
                                   f" {cpu_model()}"},
        "e2e": {"value": mpts, "unit": "Mpts/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# B200 arm

def run_b200(args):
    import torch

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2403_07631_b200 as pct
    from paper_2403_07631_b200 import _lib
    from paper_2403_07631_b200.tomogram import DeviceStack, new_device_stack

    cfg, xyz, seed = workload(args, rank)
    d_s, r_g = cfg["d_s"], cfg["r_g"]
    n = len(xyz)
    ctx = _lib.context(local)
    stream = torch.cuda.Stream(device=local)
    ctx.check(ctx.lib.pct_set_stream(ctx.h, C.c_void_p(stream.cuda_stream)), "set_stream")
    params = pct.TravParams()
    pc = _lib.trav_params_c(params, r_g)
    w = np.ascontiguousarray(pct.build_kernel(params.d_inf, params.d_sm, r_g).weights)
    dxyz = _lib.DeviceBuffer.from_host(ctx, xyz)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=f"cuda:{local}")
    lib, h = ctx.lib, ctx.h

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        return e

    state = {}

    def step():
        """One device-resident pass; returns the 5 stage events."""
        e0 = ev()
        lo = np.empty(3)
        hi = np.empty(3)
        ctx.check(lib.pct_bounds(h, dxyz.ptr, n, _lib.PCT_F32, lo.ctypes.data, hi.ctypes.data),
                  "bounds")
        fr = _lib.FrameC()
        hts = np.empty(4096)
        rc = lib.pct_frame_compute(lo.ctypes.data, hi.ctypes.data, d_s, r_g, 16384, C.byref(fr),
                                   hts.ctypes.data, 4096)
        assert rc == 0
        S, R, Cc = fr.n_slices, fr.rows, fr.cols
        g = new_device_stack(ctx, S, R, Cc)
        c = new_device_stack(ctx, S, R, Cc)
        cost = new_device_stack(ctx, S, R, Cc)
        e1 = ev()
        ctx.check(lib.pct_build(h, dxyz.ptr, n, _lib.PCT_F32, C.byref(fr), hts.ctypes.data,
                                g.ptr, c.ptr), "build")
        e2 = ev()
        ctx.check(lib.pct_evaluate(h, g.ptr, c.ptr, S, R, Cc, r_g, C.byref(pc), w.ctypes.data,
                                   w.shape[0], cost.ptr), "evaluate")
        e3 = ev()
        keep = np.empty(S, np.int32)
        nk = C.c_int32()
        ctx.check(lib.pct_simplify(h, g.ptr, cost.ptr, S, R, Cc, 1e-6, 50.0, keep.ctypes.data,
                                   C.byref(nk)), "simplify")
        e4 = ev()
        state.update(S=S, R=R, C=Cc, keep=int(nk.value), stacks=(g, c, cost))
        return (e0, e1, e2, e3, e4)

    def flush_l2():
        with torch.cuda.stream(stream):
            flush.zero_()

    # warm-up: at least W steps and at least 0.5 s so the SM clock has ramped
    t_w = time.perf_counter()
    done = 0
    while done < args.warmup or (time.perf_counter() - t_w < 0.5 and not args.profile):
        step()
        flush_l2()
        done += 1
        if done % 8 == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    launches0 = ctx.launches
    evs = []
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        t_start = time.perf_counter()
        for _ in range(args.steps):
            evs.append(step())
            flush_l2()   # between steps, outside the per-step events
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_start
    launches = ctx.launches - launches0
    stage_names = ["bounds", "build", "evaluate", "simplify"]
    per = {k: [] for k in stage_names}
    totals = []
    for e in evs:
        for i, k in enumerate(stage_names):
            per[k].append(e[i].elapsed_time(e[i + 1]))
        totals.append(e[0].elapsed_time(e[4]))
    step_ms = sum(totals)  # device time of the K steps (L2 flushes excluded)
    if world > 1:
        t = torch.tensor([step_ms], device=f"cuda:{local}", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        step_ms = float(t.item())
        cnt = torch.tensor([float(n)], device=f"cuda:{local}", dtype=torch.float64)
        torch.distributed.all_reduce(cnt)
        total_pts = float(cnt.item())
    else:
        total_pts = float(n)
    ms = step_ms / args.steps
    value = total_pts * args.steps / (step_ms * 1e3)  # Mpts/s whole job
    S, R, Cc = state["S"], state["R"], state["C"]
    cs = S * R * Cc
    ev_ms = statistics.mean(per["evaluate"])
    peak, peak_src = peaks()
    achieved = 12.0 * cs / (ev_ms * 1e-3) / 1e9
    traffic = None
    prof = ROOT / "profiles" / "ncu_traffic.json"
    if prof.exists():
        try:
            tr = json.loads(prof.read_text())
            key = f"cfg{args.config}"
            if key in tr:
                traffic = tr[key].get("eval_dram_bytes")
        except Exception:
            traffic = None

    line = {
        "metric": METRIC, "value": value, "unit": "Mpts/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"cfg{args.config} {cfg['name']}: {n} float32 pts/rank, "
                               f"grid {R}x{Cc}, {S} slices, r_g {r_g}, d_s {d_s}",
                   "n_points_per_rank": n, "seed": seed, "rows": R, "cols": Cc, "slices": S,
                   "slices_kept": state["keep"], "r_g": r_g, "d_s": d_s,
                   "step": "bounds+build+evaluate+simplify, device-resident points",
                   "l2": f"flushed between steps ({L2_FLUSH_BYTES >> 20} MiB write), "
                         "flush excluded from step time",
                   "parallelism": f"{world} independent maps (one per GPU)"},
        "stages_ms": {k: statistics.mean(v) for k, v in per.items()},
        "wall_s_timed_region": t_wall,
        "algorithmic_bytes_per_step": 12 * n + 28 * cs,
        "pipeline_gbs": (12 * n + 28 * cs) / (ms * 1e-3) / 1e9,
        "roofline": {"kernel": "eval_sym_kernel<4> (fused K4+K5)", "bound": "hbm",
                     "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "algorithmic": f"12 B per cell-slice x {cs} cell-slices per launch",
                     "peak_source": peak_src},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }

    # ---- e2e through the public API with host buffers
    if not args.no_e2e and not args.profile:
        pin = _lib.PinnedBuffer(ctx, xyz.shape, np.float32)
        pin.array[...] = xyz
        cloud = pct.PointCloud(pin.array)
        e2e_times = []
        d2h = 0
        for i in range(args.warmup + args.steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            tom = pct.build_tomogram(cloud, d_s, r_g)
            evt = pct.evaluate_tomogram(tom, params)
            simp = pct.simplify_tomogram(evt).materialize()
            chk = 0.0
            for s in simp.slices:  # the caller reads every surviving layer
                chk += float(s.ground.values[0, 0] if np.isfinite(s.ground.values[0, 0]) else 0)
                _ = s.ceiling.values
                _ = s.cost.values
            t1 = time.perf_counter()
            if i >= args.warmup:
                e2e_times.append(t1 - t0)
            d2h = 3 * 4 * R * Cc * len(simp.slices)
            del tom, evt, simp
        e2e_s = statistics.mean(e2e_times)
        if world > 1:
            t = torch.tensor([e2e_s], device=f"cuda:{local}", dtype=torch.float64)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            e2e_s = float(t.item())
        line["e2e"] = {"value": total_pts / (e2e_s * 1e6), "unit": "Mpts/s",
                       "ms_per_step": 1e3 * e2e_s, "h2d_bytes_per_step": 12 * n,
                       "d2h_bytes_per_step": d2h,
                       "path": "PointCloud(pinned f32) -> build_tomogram -> evaluate_tomogram -> "
                               "simplify_tomogram -> host arrays of surviving slices"}

    # ---- CPU baseline (rank 0, N=1 only): the pinned numpy port, all host threads
    if rank == 0 and world == 1 and not args.no_cpu and not args.profile:
        threads = os.cpu_count() or 1
        t, st, _ = cpu_pipeline(xyz, cfg, threads)
        line["cpu_baseline"] = {"value": n / (t * 1e6), "unit": "Mpts/s", "cores": threads,
                                "kind": "port",
                                "sample": f"1 full cfg{args.config} map (build+evaluate+simplify,"
                                          f" {t:.1f} s), {cpu_model()}",
                                "stages_s": st}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.profile:
        args.warmup, args.steps = 1, 1
    sys.path.insert(0, str(ROOT / "tests"))
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
