"""Row-band sharded pipeline on one GPU with P virtual ranks: the assembled
bands must equal the single-GPU result bit for bit (ground, ceiling, cost,
surviving slices), for any split of the input points over the ranks."""

import numpy as np
import pytest

from golden_util import case_input

pytestmark = pytest.mark.gpu

pct = pytest.importorskip("paper_2403_07631_b200")


def _single(xyz, d_s, r_g):
    tom = pct.build_tomogram(pct.PointCloud(xyz), d_s, r_g)
    ev = pct.evaluate_tomogram(tom, pct.TravParams())
    simp = pct.simplify_tomogram(ev)
    heights = [s.plane_height for s in tom.slices]
    keep = [heights.index(s.plane_height) for s in simp.slices]
    return ev.ground_stack(), ev.ceiling_stack(), ev.cost_stack(), keep


def _sharded(xyz, d_s, r_g, P, split="interleave"):
    import torch
    from paper_2403_07631_b200 import sharded
    t = torch.from_numpy(np.ascontiguousarray(xyz)).cuda()
    if split == "interleave":
        shards = [t[r::P] for r in range(P)]
    else:  # contiguous chunks, the last rank may get nothing
        n = t.shape[0]
        shards = [t[n * r // (P + 1): n * (r + 1) // (P + 1)] for r in range(P - 1)]
        shards.append(t[n * (P - 1) // (P + 1):])
    gens = [sharded.band_pipeline(s.contiguous(), d_s, r_g, pct.TravParams(), r, P)
            for r, s in enumerate(shards)]
    res = sharded.run_virtual(gens)
    torch.cuda.synchronize()
    for r in res:
        assert r.keep == res[0].keep
    cat = lambda attr: torch.cat([getattr(r, attr) for r in res], dim=1).cpu().numpy()
    return cat("ground"), cat("ceiling"), cat("cost"), res[0].keep


@pytest.mark.parametrize("P", [1, 2, 3, 4])
def test_virtual_bands_equal_single_gpu(golden, P):
    case = golden["cases"]["synth_cfg0"]
    xyz = case_input("synth_cfg0", case)
    g1, c1, k1, keep1 = _single(xyz, 0.5, 0.1)
    g2, c2, k2, keep2 = _sharded(xyz, 0.5, 0.1, P, "interleave" if P % 2 else "chunks")
    assert np.array_equal(g1.view(np.uint32), g2.view(np.uint32))
    assert np.array_equal(c1.view(np.uint32), c2.view(np.uint32))
    assert np.array_equal(k1.view(np.uint32), k2.view(np.uint32))
    assert keep1 == keep2 == case["keep"]


def test_virtual_bands_fine_grid():
    """0.05 m: 17x17 inflation kernel and a 15-row halo."""
    from paper_2403_07631_b200 import synth
    xyz = synth.rough_terrain(400_000, seed=5, extent=20.0, n_boxes=20, n_stairs=4)
    g1, c1, k1, keep1 = _single(xyz, 0.3, 0.05)
    g2, c2, k2, keep2 = _sharded(xyz, 0.3, 0.05, 3)
    assert np.array_equal(g1.view(np.uint32), g2.view(np.uint32))
    assert np.array_equal(c1.view(np.uint32), c2.view(np.uint32))
    assert np.array_equal(k1.view(np.uint32), k2.view(np.uint32))
    assert keep1 == keep2


@pytest.mark.parametrize("mode", ["tiled", "hist"])
@pytest.mark.parametrize("P", [1, 3])
def test_virtual_bands_tiled_build(golden, monkeypatch, P, mode):
    """The tile-partitioned build (chosen automatically for maps whose key
    planes exceed ~1.5 GB, e.g. config 3) on row bands."""
    monkeypatch.setenv("PCT_BUILD", "tiled")
    case = golden["cases"]["synth_cfg0"]
    xyz = case_input("synth_cfg0", case)
    monkeypatch.setenv("PCT_BUILD", "atomic")
    g1, c1, k1, keep1 = _single(xyz, 0.5, 0.1)
    monkeypatch.setenv("PCT_BUILD", mode)
    g2, c2, k2, keep2 = _sharded(xyz, 0.5, 0.1, P)
    assert np.array_equal(g1.view(np.uint32), g2.view(np.uint32))
    assert np.array_equal(c1.view(np.uint32), c2.view(np.uint32))
    assert np.array_equal(k1.view(np.uint32), k2.view(np.uint32))
    assert keep1 == keep2 == case["keep"]


def _simplified_single(xyz, d_s, r_g):
    ev = pct.evaluate_tomogram(pct.build_tomogram(pct.PointCloud(xyz), d_s, r_g), pct.TravParams())
    return pct.simplify_tomogram(ev).materialize()


def _same_tomogram(a, b):
    assert len(a.slices) == len(b.slices)
    assert (a.rows, a.cols, a.resolution, a.origin, a.d_s, a.z_min) == \
        (b.rows, b.cols, b.resolution, b.origin, b.d_s, b.z_min)
    for sa, sb in zip(a.slices, b.slices):
        assert sa.plane_height == sb.plane_height and sa.index == sb.index
        for la, lb in ((sa.ground, sb.ground), (sa.ceiling, sb.ceiling), (sa.cost, sb.cost)):
            assert np.array_equal(la.values.view(np.uint32), lb.values.view(np.uint32))


@pytest.mark.parametrize("P", [1, 2, 4])
def test_virtual_bands_gather_tomogram(golden, P):
    """The surviving slices of every band gathered on one rank form the
    simplified Tomogram of the one-GPU chain (tomogram.py:65-96)."""
    import torch
    from paper_2403_07631_b200 import sharded
    case = golden["cases"]["synth_cfg0"]
    xyz = case_input("synth_cfg0", case)
    want = _simplified_single(xyz, 0.5, 0.1)
    t = torch.from_numpy(xyz).cuda()
    root = P - 1
    gens = [sharded.band_pipeline(t[r::P].contiguous(), 0.5, 0.1, pct.TravParams(), r, P,
                                  gather_to=root) for r in range(P)]
    res = sharded.run_virtual(gens)
    assert all(r.tomogram is None for i, r in enumerate(res) if i != root)
    got = res[root].tomogram
    assert [s.plane_height for s in got.slices] == [case["heights"][k] for k in case["keep"]]
    _same_tomogram(got.materialize(), want)


def test_tomogram_sharded_without_process_group():
    from paper_2403_07631_b200 import sharded, synth
    xyz = synth.spiral_ramp(300_000, seed=4)
    _same_tomogram(sharded.tomogram_sharded(pct.PointCloud(xyz), 0.4, 0.1).materialize(),
                   _simplified_single(xyz, 0.4, 0.1))


def test_virtual_bands_errors_on_every_rank():
    """A non-finite point on one rank, or a band thinner than the halo, fails
    every rank before the first point exchange (no rank left waiting)."""
    import torch
    from paper_2403_07631_b200 import sharded, synth
    xyz = torch.from_numpy(synth.two_storey(20_000, seed=1)).cuda()
    bad = xyz[1::2].clone()
    bad[5, 2] = float("nan")
    gens = [sharded.band_pipeline(s.contiguous(), 0.5, 0.1, pct.TravParams(), r, 2)
            for r, s in enumerate([xyz[0::2], bad])]
    reqs = [next(g) for g in gens]
    assert [r[0] for r in reqs] == ["bounds", "bounds"] and reqs[1][3] == 1.0
    for g in gens:  # the reduced flag reaches both ranks: both raise
        with pytest.raises(ValueError, match="non-finite"):
            g.send((np.zeros(3), np.ones(3), 1.0))
    # 203 rows over 40 ranks: 5-row bands against an 8-row halo
    gens = [sharded.band_pipeline(xyz[r::40].contiguous(), 0.5, 0.1, pct.TravParams(), r, 40)
            for r in range(40)]
    with pytest.raises(ValueError, match="thinner than"):
        sharded.run_virtual(gens)


def _gloo_worker(rank, size, port, q, n_points, gather="device"):
    import os
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        torch.cuda.set_device(0)
        import paper_2403_07631_b200 as p
        from paper_2403_07631_b200 import sharded, synth
        if gather == "host-p2p":  # no room in /dev/shm: bands sent to the root
            sharded._shm_free = lambda: 0
            gather = "host"
        xyz = synth.spiral_ramp(n_points, seed=4)
        mine = np.ascontiguousarray(xyz[rank::size])
        tom = sharded.tomogram_sharded(p.PointCloud(mine), 0.4, 0.1, root=0, gather=gather)
        if gather == "host" and rank == 0:  # a second call re-uses the segment
            again = sharded.tomogram_sharded(p.PointCloud(mine), 0.4, 0.1, root=0, gather=gather)
            assert all(np.array_equal(a.cost.values, b.cost.values)
                       for a, b in zip(tom.slices, again.slices))
            assert all(s.ground._values is not None for s in tom.slices)  # host-resident
        elif gather == "host":
            sharded.tomogram_sharded(p.PointCloud(mine), 0.4, 0.1, root=0, gather=gather)
        if rank == 0:
            tom.materialize()
            import hashlib
            dig = [hashlib.sha256(np.stack([l.values for l in layers]).tobytes()).hexdigest()
                   for layers in ([s.ground for s in tom.slices], [s.ceiling for s in tom.slices],
                                  [s.cost for s in tom.slices])]
            q.put((rank, [s.plane_height for s in tom.slices], dig))
        else:
            q.put((rank, tom is None, None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("gather", ["device", "host", "host-p2p"])
def test_two_processes_gloo_equal_single_gpu(gather):
    """The real band pipeline in two processes (gloo: collectives staged
    through host memory; both ranks share cuda:0) returns on rank 0 the
    Tomogram of the one-GPU chain, bit for bit -- gathered on the root's GPU,
    written by each rank into one shared host segment, or (no room in
    /dev/shm) sent to the root and read back there."""
    import hashlib
    import socket
    import torch.multiprocessing as mp
    from paper_2403_07631_b200 import synth
    n = 300_000
    want = _simplified_single(synth.spiral_ramp(n, seed=4), 0.4, 0.1)
    wdig = [hashlib.sha256(np.stack([l.values for l in layers]).tobytes()).hexdigest()
            for layers in ([s.ground for s in want.slices], [s.ceiling for s in want.slices],
                           [s.cost for s in want.slices])]
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q, n, gather)) for r in range(2)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(2):
        r = q.get(timeout=300)
        out[r[0]] = r
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert out[1][1] is True
    assert out[0][1] == [sl.plane_height for sl in want.slices]
    assert out[0][2] == wdig
