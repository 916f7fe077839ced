"""Golden fixtures added in round 2: config 3 (campus) pins and planner lookups.

Run ONLY in the build container, where the read-only reference package lives:

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden_r2.py

Writes tests/golden/golden_r2.json with

* ``campus_crop``: the reference's build -> evaluate -> simplify on the exact
  crop of the full 200M-point config-3 cloud (``synth.campus(box=...)``, one
  building with its ramps, stair, plant room and walkway stub at full point
  density): per-slice sha256 digests of ground / ceiling / cost, plane
  heights, keep list, origin.
* ``campus_sparse``: the same on the full 400 x 400 m config-3 frame (the
  4004 x 4004 x 44 grid of the headline map) drawn at 8M points: the frame,
  the slice count and the large-map code paths at the headline's grid size.
* ``snap``: the reference planner's ``_PlannerContext.snap`` and
  ``member_with_min_cost`` (planner.py:95-129) on sampled queries over two
  evaluated / simplified tomograms.

Inputs are regenerated from ``paper_2403_07631_b200.synth`` (their sha256 is
recorded, so generator drift fails loudly).  Nothing on the GPU box reads
/root/reference; it only reads the JSON.
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(HERE))

import tomoplan as tp  # noqa: E402  (reference, build container only)
from tomoplan.planner import _PlannerContext  # noqa: E402

from make_golden import digest  # noqa: E402
from paper_2403_07631_b200 import synth  # noqa: E402

CAMPUS_CROP_BOX = (126.0, 126.0, 174.0, 174.0)
CAMPUS_SPARSE_N = 8_000_000


def run_case(xyz, d_s, r_g, threads=8):
    t0 = time.perf_counter()
    tom = tp.build_tomogram(tp.PointCloud(xyz), d_s, r_g, threads=threads)
    t1 = time.perf_counter()
    ev = tp.evaluate_tomogram(tom, tp.TravParams(), threads=threads)
    t2 = time.perf_counter()
    simp = tp.simplify_tomogram(ev)
    t3 = time.perf_counter()
    heights = [s.plane_height for s in ev.slices]
    keep = [heights.index(s.plane_height) for s in simp.slices]
    entry = dict(
        d_s=d_s, r_g=r_g, n_points=int(xyz.shape[0]), input_dtype=str(xyz.dtype),
        input_sha256=digest(xyz), shape=[len(ev.slices), ev.rows, ev.cols],
        heights=[float(h) for h in heights], keep=keep,
        origin=[float(v) for v in ev.origin], z_min=float(ev.z_min),
        ground_slice_sha256=[digest(s.ground.values) for s in ev.slices],
        ceiling_slice_sha256=[digest(s.ceiling.values) for s in ev.slices],
        cost_slice_sha256=[digest(s.cost.values) for s in ev.slices],
        ref_seconds=dict(build=t1 - t0, evaluate=t2 - t1, simplify=t3 - t2, threads=threads),
    )
    return entry, ev, simp


def snap_queries(tom, rng, n=400):
    """Queries near real surfaces (and some far from any), several tolerances."""
    pc = _PlannerContext(tom, 1e-6, 50.0)
    K, R, C = pc.elev.shape
    out = []
    for q in range(n):
        i, j = int(rng.integers(0, R)), int(rng.integers(0, C))
        col = pc.elev[:, i, j]
        ok = np.flatnonzero(np.isfinite(col))
        if ok.size and q % 5:
            z = float(col[rng.choice(ok)]) + float(rng.normal(0.0, 0.3))
        else:
            z = float(rng.uniform(-2.0, 20.0))
        x = pc.origin[0] + (j + rng.uniform(-0.49, 0.49)) * pc.res
        y = pc.origin[1] + (i + rng.uniform(-0.49, 0.49)) * pc.res
        if q % 17 == 0:  # outside the grid
            x -= 5.0 * pc.res * C
        tol = float(rng.choice([0.05, 0.25, 0.5, 1.0, 3.0]))
        res = pc.snap((x, y, z), tol)
        member = None if res is None else int(pc.member_with_min_cost(*res))
        out.append(dict(point=[x, y, z], tol=tol,
                        snap=None if res is None else [int(v) for v in res], member=member))
    return out


def main():
    golden = dict(generator="tests/golden/make_golden_r2.py", reference="tomoplan 0.1.0",
                  numpy=np.__version__, cases={}, snap={})
    c3 = synth.CONFIGS[3]

    xyz = synth.campus(c3["n_points"], c3["seed"], box=CAMPUS_CROP_BOX)
    e, _, _ = run_case(xyz, c3["d_s"], c3["r_g"])
    e.update(source="paper_2403_07631_b200.synth.campus", n_full=c3["n_points"],
             seed=c3["seed"], box=list(CAMPUS_CROP_BOX))
    golden["cases"]["campus_crop"] = e
    print("campus_crop", e["shape"], "keep", len(e["keep"]), e["ref_seconds"], flush=True)
    del xyz

    xyz = synth.campus(CAMPUS_SPARSE_N, c3["seed"])
    e, _, _ = run_case(xyz, c3["d_s"], c3["r_g"])
    e.update(source="paper_2403_07631_b200.synth.campus", n_full=CAMPUS_SPARSE_N,
             seed=c3["seed"], box=None)
    golden["cases"]["campus_sparse"] = e
    print("campus_sparse", e["shape"], "keep", len(e["keep"]), e["ref_seconds"], flush=True)
    del xyz

    rng = np.random.default_rng(2403)
    for name, xyz, d_s in (("synth_cfg0", synth.generate(0), 0.5),
                           ("spiral_crop", synth.generate(1, 600_000), 0.4)):
        _, ev, simp = run_case(xyz, d_s, 0.1)
        golden["snap"][name] = dict(input_sha256=digest(xyz), n_points=int(xyz.shape[0]),
                                    d_s=d_s, r_g=0.1,
                                    evaluated=snap_queries(ev, rng),
                                    simplified=snap_queries(simp, rng))
        print("snap", name, flush=True)

    (HERE / "golden_r2.json").write_text(json.dumps(golden, indent=1))
    print("wrote", HERE / "golden_r2.json")


if __name__ == "__main__":
    main()
