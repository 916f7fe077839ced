"""Generate the golden fixtures that pin the oracle (and through it the GPU path)
to the reference implementation.

Run ONLY in the build container, where the read-only reference package lives:

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

It imports `tomoplan` from /root/reference/pkg/src, runs the reference's own
build_tomogram -> evaluate_tomogram -> simplify_tomogram on seeded inputs and
records (a) small inputs + full outputs as compressed .npz, and (b) sha256
digests of every output stack for large inputs that are regenerated from
`paper_2403_07631_b200.synth` (their input digest is recorded too, so a
generator drift is detected instead of silently changing the case).
Nothing on the GPU box reads /root/reference; it only reads these files.
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(REPO))

import tomoplan as tp  # noqa: E402  (reference, build container only)

from paper_2403_07631_b200 import synth  # noqa: E402


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes()).hexdigest()


def run_reference(xyz, d_s, r_g, threads=8):
    cloud = tp.PointCloud(xyz)
    t0 = time.perf_counter()
    tom = tp.build_tomogram(cloud, d_s, r_g, threads=threads)
    t1 = time.perf_counter()
    ev = tp.evaluate_tomogram(tom, tp.TravParams(), threads=threads)
    t2 = time.perf_counter()
    simp = tp.simplify_tomogram(ev)
    t3 = time.perf_counter()
    heights = np.array([s.plane_height for s in ev.slices])
    keep_h = [s.plane_height for s in simp.slices]
    keep = [int(np.flatnonzero(heights == h)[0]) for h in keep_h]
    # the reference's LGA archives (tomogram.py:228-244) of the built, evaluated
    # and simplified tomograms: the byte-exact target of save_tomogram
    import tempfile
    lga = {}
    with tempfile.TemporaryDirectory() as d:
        for key, t in (("built", tom), ("evaluated", ev), ("simplified", simp)):
            p = Path(d) / f"{key}.lga"
            tp.save_tomogram(t, p)
            b = p.read_bytes()
            lga[key] = dict(sha256=hashlib.sha256(b).hexdigest(), bytes=len(b))
    # the A* planner's canonical-node arrays (planner.py:65-93) of the
    # evaluated and the simplified tomogram: the target of the §8 f precompute
    from tomoplan.planner import _PlannerContext
    planner = {}
    for key, t in (("evaluated", ev), ("simplified", simp)):
        pc = _PlannerContext(t, 1e-6, 50.0)
        planner[key] = dict(canon_sha256=digest(pc.canon), cn_sha256=digest(pc.cn))
    out = dict(
        ground=ev.ground_stack(), ceiling=ev.ceiling_stack(), cost=ev.cost_stack(),
        heights=heights, keep=np.array(keep, np.int64),
        origin=np.array(ev.origin, np.float64), z_min=float(ev.z_min), lga=lga,
        planner=planner,
    )
    return out, (t1 - t0, t2 - t1, t3 - t2)


def record(name, xyz, d_s, r_g, meta, store_arrays, store_input):
    out, times = run_reference(xyz, d_s, r_g)
    entry = dict(meta)
    entry.update(
        d_s=d_s, r_g=r_g, n_points=int(xyz.shape[0]),
        input_dtype=str(xyz.dtype), input_sha256=digest(xyz),
        shape=[int(v) for v in out["ground"].shape],
        heights=[float(h) for h in out["heights"]],
        keep=[int(k) for k in out["keep"]],
        origin=[float(v) for v in out["origin"]], z_min=out["z_min"],
        ground_sha256=digest(out["ground"]), ceiling_sha256=digest(out["ceiling"]),
        cost_sha256=digest(out["cost"]),
        ground_slice_sha256=[digest(g) for g in out["ground"]],
        ceiling_slice_sha256=[digest(g) for g in out["ceiling"]],
        cost_slice_sha256=[digest(g) for g in out["cost"]],
        lga=out["lga"],
        planner=out["planner"],
        ref_seconds=dict(build=times[0], evaluate=times[1], simplify=times[2], threads=8),
    )
    if store_arrays or store_input:
        arrays = {}
        if store_input:
            arrays["xyz"] = xyz
        if store_arrays:
            arrays.update(ground=out["ground"], ceiling=out["ceiling"], cost=out["cost"])
        np.savez_compressed(HERE / f"{name}.npz", **arrays)
        entry["npz"] = f"{name}.npz"
    print(f"{name}: {entry['shape']} keep={entry['keep']} times={times}", flush=True)
    return entry


def inflation_cases():
    """Reference inflate() on random maps (test_acceptance.py:141-150 style)."""
    rng = np.random.default_rng(4242)
    cases = []
    for r_g in (0.1, 0.05, 0.2):
        kern = tp.build_kernel(0.2, 0.4, r_g)
        for t in range(3):
            shape = (int(rng.integers(40, 140)), int(rng.integers(40, 140)))
            seed = int(rng.integers(1 << 30))
            g = np.random.default_rng(seed).uniform(0.0, 50.0, shape).astype(np.float32)
            g[np.random.default_rng(seed + 1).uniform(size=shape) < 0.03] = 50.0
            cases.append(dict(r_g=r_g, shape=list(shape), seed=seed,
                              kernel_sha256=digest(kern.weights),
                              out_sha256=digest(tp.inflate(g, kern))))
    return cases


def main():
    golden = dict(generator="tests/golden/make_golden.py", reference="tomoplan 0.1.0",
                  numpy=np.__version__, cases={})
    C = golden["cases"]

    # reference scenes (inputs stored: only the reference can regenerate them)
    ref_scenes = [
        ("ref_random_multilayer_s9", dict(kind="random_multilayer", dimensions=(6, 6, 3.0),
                                          density=300.0, seed=9), 0.5, 0.1, True),
        ("ref_flat_plane_s7", dict(kind="flat_plane", dimensions=(10, 10), density=100.0,
                                   seed=7), 0.5, 0.1, True),
        ("ref_spiral_s3", dict(kind="spiral_stair", density=300.0, seed=3, turns=5.0,
                               rise_per_turn=4.6), 0.5, 0.1, False),
        ("ref_ramp_over_tunnel_s6", dict(kind="ramp_over_tunnel", density=300.0, seed=6,
                                         noise_sigma=0.01), 0.5, 0.1, False),
    ]
    for name, kw, d_s, r_g, arrays in ref_scenes:
        xyz = tp.generate_scene(tp.SceneSpec(**kw)).xyz
        C[name] = record(name, xyz, d_s, r_g, dict(source="tomoplan.generate_scene",
                                                   spec={k: (list(v) if isinstance(v, tuple) else v)
                                                         for k, v in kw.items()}),
                         store_arrays=arrays, store_input=True)

    # BASELINE configs regenerated from synth (digests only)
    for cfg, n in ((0, None), (1, None), (4, None), (2, 2_000_000)):
        c = synth.CONFIGS[cfg]
        xyz = synth.generate(cfg, n)
        name = f"synth_cfg{cfg}" + ("" if n is None else f"_n{n}")
        C[name] = record(name, xyz, c["d_s"], c["r_g"],
                         dict(source="paper_2403_07631_b200.synth", config=cfg,
                              n_override=n), store_arrays=False, store_input=False)

    # a reduced cfg0 map with full arrays (exact per-cell diagnosis on failure)
    xyz = synth.two_storey(30_000, seed=11)
    C["synth_two_storey_small"] = record("synth_two_storey_small", xyz, 0.5, 0.1,
                                         dict(source="paper_2403_07631_b200.synth.two_storey",
                                              n=30_000, seed=11),
                                         store_arrays=True, store_input=False)

    golden["inflation"] = inflation_cases()
    (HERE / "golden.json").write_text(json.dumps(golden, indent=1))
    print("wrote", HERE / "golden.json")


if __name__ == "__main__":
    main()
