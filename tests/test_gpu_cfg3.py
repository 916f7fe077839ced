"""Config 3 (the headline campus map) and config 4 (batched maps) on the GPU.

* A full-density crop of the 200M-point campus and the full 4004 x 4004 x 44
  frame at 8M points, pinned to the reference's own per-slice digests
  (tests/golden/golden_r2.json, written by make_golden_r2.py).
* The FULL 200M-point map through the library's default path (the tiled
  build, which the library picks above 1.5 GB of key planes), against the C
  oracle run on the box's host cores: every slice bitwise, keep list.
* The same map row-band sharded over 4 virtual ranks with the gather: the
  assembled Tomogram equals the one-GPU one.
* The batched native call (pct_tomo_run_batch) against the reference's
  config-4 digests (map 0 of the batch).
"""

import json
import os

import numpy as np
import pytest

from golden_util import GOLDEN, TABLE_PARAMS, digest, load_golden

pytestmark = pytest.mark.gpu

pct = pytest.importorskip("paper_2403_07631_b200")
from paper_2403_07631_b200 import synth  # noqa: E402

C3 = synth.CONFIGS[3]


@pytest.fixture(scope="module")
def golden_r2():
    return json.loads((GOLDEN / "golden_r2.json").read_text())


def _stacks(xyz, d_s, r_g):
    """Full ground / ceiling / cost stacks and keep list of the drop-in chain."""
    tom = pct.build_tomogram(pct.PointCloud(xyz), d_s, r_g)
    ev = pct.evaluate_tomogram(tom, pct.TravParams())
    simp = pct.simplify_tomogram(ev)
    heights = [s.plane_height for s in ev.slices]
    keep = [heights.index(s.plane_height) for s in simp.slices]
    return ev, simp, keep


@pytest.mark.parametrize("name", ["campus_crop", "campus_sparse"])
def test_campus_matches_reference(golden_r2, name):
    case = golden_r2["cases"][name]
    box = tuple(case["box"]) if case["box"] else None
    xyz = synth.campus(case["n_full"], case["seed"], box=box)
    assert digest(xyz) == case["input_sha256"]
    ev, simp, keep = _stacks(xyz, case["d_s"], case["r_g"])
    assert [ev.rows, ev.cols] == case["shape"][1:] and len(ev.slices) == case["shape"][0]
    assert list(ev.origin) == case["origin"] and ev.z_min == case["z_min"]
    assert [s.plane_height for s in ev.slices] == case["heights"]
    assert [digest(s.ground.values) for s in ev.slices] == case["ground_slice_sha256"]
    assert [digest(s.ceiling.values) for s in ev.slices] == case["ceiling_slice_sha256"]
    assert [digest(s.cost.values) for s in ev.slices] == case["cost_slice_sha256"]
    assert keep == case["keep"]


@pytest.fixture(scope="module")
def full_map():
    return synth.generate(3)


@pytest.fixture(scope="module")
def full_cpu(full_map):
    from oracle import fast
    return fast.pipeline(full_map, C3["d_s"], C3["r_g"], TABLE_PARAMS,
                         threads=os.cpu_count() or 1)


@pytest.mark.slow
def test_cfg3_full_map_matches_c_oracle(full_map, full_cpu):
    """200M points, 4004 x 4004 x 44, default (tiled) build: bit for bit."""
    t, cost, keep = full_cpu
    ev, simp, gkeep = _stacks(full_map, C3["d_s"], C3["r_g"])
    assert len(ev.slices) == t["ground"].shape[0] == 44
    assert np.array_equal(np.asarray([s.plane_height for s in ev.slices]), t["heights"])
    for k, s in enumerate(ev.slices):
        assert np.array_equal(s.ground.values.view(np.uint32), t["ground"][k].view(np.uint32)), k
        assert np.array_equal(s.ceiling.values.view(np.uint32), t["ceiling"][k].view(np.uint32)), k
        assert np.array_equal(s.cost.values.view(np.uint32), cost[k].view(np.uint32)), k
    assert gkeep == keep


@pytest.mark.slow
def test_cfg3_full_map_four_virtual_bands(full_map, full_cpu):
    """The row-band pipeline (4 bands, each fed an arbitrary quarter of the
    surfaces, partitioned on the device, halos exchanged, any()-tables
    reduced, kept slices gathered) returns the one-GPU simplified map."""
    import torch
    from paper_2403_07631_b200 import sharded
    t, cost, keep = full_cpu
    P = 4
    shares = [torch.from_numpy(synth.campus(C3["n_points"], C3["seed"], share=(r, P))).cuda()
              for r in range(P)]
    gens = [sharded.band_pipeline(shares[r], C3["d_s"], C3["r_g"], pct.TravParams(), r, P,
                                  gather_to=0) for r in range(P)]
    res = sharded.run_virtual(gens)
    del shares
    assert all(r.keep == keep for r in res)
    tom = res[0].tomogram
    assert [s.plane_height for s in tom.slices] == [float(t["heights"][k]) for k in keep]
    for m, k in enumerate(keep):
        sl = tom.slices[m]
        assert np.array_equal(sl.ground.values.view(np.uint32), t["ground"][k].view(np.uint32))
        assert np.array_equal(sl.ceiling.values.view(np.uint32), t["ceiling"][k].view(np.uint32))
        assert np.array_equal(sl.cost.values.view(np.uint32), cost[k].view(np.uint32))


def test_batched_native_call_matches_reference_cfg4():
    """pct_tomo_run_batch over 6 config-4 maps: map 0 (seed 1000) equals the
    reference's outputs for that map (golden synth_cfg4), all slices."""
    from paper_2403_07631_b200 import _lib
    from paper_2403_07631_b200.batch import BatchRunner
    from paper_2403_07631_b200.tomogram import DeviceStack, DeviceTomogram
    case = load_golden()["cases"]["synth_cfg4"]
    clouds = [synth.generate(4, None, 1000 + m) for m in range(6)]
    assert digest(clouds[0]) == case["input_sha256"]
    runner = BatchRunner(workers=2)
    ctx = runner.ctxs[0]
    bufs = [_lib.DeviceBuffer.from_host(ctx, c) for c in clouds]
    ctx.check(ctx.lib.pct_sync(ctx.h), "sync")
    try:
        res = runner.run([(b.ptr, len(c), _lib.PCT_F32, 0) for b, c in zip(bufs, clouds)],
                         0.5, 0.1, pct.TravParams())
    finally:
        runner.close()
    (hctx, handle), keep = res[0]
    dt = DeviceTomogram(hctx, handle)
    g, c = dt.stacks()
    fr = dt.frame
    cost = DeviceStack(hctx, hctx.lib.pct_tomo_layer(handle, _lib.LAYER_COST), fr.n_slices,
                       fr.rows, fr.cols, dt)
    assert [fr.n_slices, fr.rows, fr.cols] == case["shape"]
    assert [float(h) for h in dt.heights] == case["heights"]
    assert digest(g.host_all()) == case["ground_sha256"]
    assert digest(c.host_all()) == case["ceiling_sha256"]
    assert digest(cost.host_all()) == case["cost_sha256"]
    assert keep == case["keep"]
