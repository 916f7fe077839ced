"""Quick GPU check of the evaluate kernels: every PCT_EVAL_KERNEL / PCT_INFL
variant against the fused per-slice kernel on golden inputs, with the
evaluate-stage device time of each.  Usage (on the GPU box):
    python scripts/eval_check.py [case ...]
"""

import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import paper_2403_07631_b200 as pct  # noqa: E402
from golden_util import case_input, digest, load_golden  # noqa: E402

VARIANTS = [("fast", {"PCT_EVAL_KERNEL": "fast"}),
            ("split-sym", {"PCT_EVAL_KERNEL": "split", "PCT_INFL": "sym"}),
            ("split-bnb", {"PCT_EVAL_KERNEL": "split", "PCT_INFL": "bnb"}),
            ("bnb-alt", {"PCT_EVAL_KERNEL": "split", "PCT_INFL": "bnb", "PCT_BNB_TILE": "1"}),
            ("bnb-run1", {"PCT_EVAL_KERNEL": "split", "PCT_INFL": "bnb", "PCT_INFL_RUN": "1"}),
            ("bnb-run3", {"PCT_EVAL_KERNEL": "split", "PCT_INFL": "bnb", "PCT_INFL_RUN": "3"})]
KEYS = ("PCT_EVAL_KERNEL", "PCT_INFL", "PCT_BNB_TILE", "PCT_INFL_RUN")


def run(tom, env, reps=5):
    old = {k: os.environ.get(k) for k in KEYS}
    for k in KEYS:
        os.environ.pop(k, None)
    os.environ.update(env)
    try:
        import torch
        ev = pct.evaluate_tomogram(tom, pct.TravParams())  # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            ev = pct.evaluate_tomogram(tom, pct.TravParams())
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / reps
        return ev.cost_stack(), dt
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def main():
    g = load_golden()
    names = sys.argv[1:] or ["synth_cfg0", "ref_random_multilayer_s9", "synth_cfg1",
                             "synth_cfg2_n2000000"]
    for name in names:
        case = g["cases"][name]
        tom = pct.build_tomogram(pct.PointCloud(case_input(name, case)), case["d_s"], case["r_g"])
        ref = None
        for vname, env in VARIANTS:
            if vname == "split-sym" and case["r_g"] < 0.1:
                continue
            cost, dt = run(tom, env)
            ok_gold = all(digest(cost[k]) == case["cost_slice_sha256"][k]
                          for k in range(cost.shape[0]))
            same = ref is None or np.array_equal(ref.view(np.uint32), cost.view(np.uint32))
            if ref is None:
                ref = cost
            print(f"{name:28s} {vname:10s} wall {dt * 1e3:8.3f} ms  golden={ok_gold} "
                  f"same_as_fast={same}", flush=True)


if __name__ == "__main__":
    main()
