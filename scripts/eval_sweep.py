"""Time the evaluate launch on a config map for several kernel settings
(PCT_EVAL_KERNEL / PCT_EVAL_RUN env overrides); prints one line per setting."""
import ctypes as C, os, sys, time, json
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2403_07631_b200 as pct
from paper_2403_07631_b200 import _lib, synth
from paper_2403_07631_b200.tomogram import new_device_stack

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
settings = sys.argv[2:] or ["fast", "incr:4", "incr:8", "incr:12", "incr:37"]
c = synth.CONFIGS[cfg]
xyz = synth.generate(cfg)
tom = pct.build_tomogram(pct.PointCloud(xyz), c["d_s"], c["r_g"])
g, _ = tom.slices[0].ground.device
cst, _ = tom.slices[0].ceiling.device
ctx = g.ctx
S, R, Cc = g.n_slices, g.rows, g.cols
out = new_device_stack(ctx, S, R, Cc)
p = pct.TravParams()
pc = _lib.trav_params_c(p, c["r_g"])
w = np.ascontiguousarray(pct.build_kernel(p.d_inf, p.d_sm, c["r_g"]).weights)
stream = torch.cuda.Stream()
ctx.lib.pct_set_stream(ctx.h, C.c_void_p(stream.cuda_stream))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ref = None
for s in settings:
    kern, _, run = s.partition(":")
    os.environ["PCT_EVAL_KERNEL"] = kern
    if run: os.environ["PCT_EVAL_RUN"] = run
    else: os.environ.pop("PCT_EVAL_RUN", None)
    ts = []
    for i in range(12):
        with torch.cuda.stream(stream): flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ctx.check(ctx.lib.pct_evaluate(ctx.h, g.ptr, cst.ptr, S, R, Cc, c["r_g"], C.byref(pc),
                                       w.ctypes.data, w.shape[0], out.ptr), "eval")
        e1.record(stream); e1.synchronize()
        if i >= 2: ts.append(e0.elapsed_time(e1))
    res = out.host_all().view(np.uint32)
    same = None if ref is None else bool(np.array_equal(ref, res))
    ref = res if ref is None else ref
    print(json.dumps({"cfg": cfg, "setting": s, "eval_us_median": 1e3 * float(np.median(ts)),
                      "eval_us_min": 1e3 * min(ts), "cs": S * R * Cc, "same_as_first": same}), flush=True)
