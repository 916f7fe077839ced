"""Host-side logic of the row-band sharded path on CPU: band geometry, the
sweep replay against the oracle, and the collective driver over a real
2-rank gloo group (127.0.0.1)."""

import os
import socket

import numpy as np
import pytest

import oracle
from golden_util import case_arrays
from paper_2403_07631_b200 import sharded


def test_band_geometry():
    for rows in (5, 203, 4002):
        for P in (1, 2, 3, 8):
            s = sharded.band_starts(rows, P)
            assert s[0] == 0 and s[-1] == rows and all(a <= b for a, b in zip(s, s[1:]))
    from types import SimpleNamespace
    p = SimpleNamespace(step_patch_radius=None)
    assert sharded.halo_rows(p, 0.1, 9) == 4 + 3 + 1
    assert sharded.halo_rows(p, 0.05, 17) == 8 + 6 + 1


def test_owner_band_rule_matches_rasterisation():
    rng = np.random.default_rng(0)
    y = rng.uniform(-3, 40, 10000)
    y0, r_g = float(y.min()), 0.1
    rows = int(np.floor((y.max() - y0) / r_g + 0.5)) + 2
    st = sharded.band_starts(rows, 4)
    b = sharded.owner_band_np(y, y0, r_g, st)
    i = np.floor((y - y0) / r_g + 0.5)
    for k in range(4):
        assert np.all((i[b == k] >= st[k]) & (i[b == k] < st[k + 1]))


def _any_table(G, Cst, rows_sl):
    """window table / triple any()s from the oracle on a row subset."""
    S = G.shape[0]
    g, c = G[:, rows_sl], Cst[:, rows_sl]
    tb = np.zeros((S, 17), np.uint8)  # columns 0..15: below = k-1-j; 16: no lower neighbour
    for k in range(S):
        above = k + 1 if k + 1 < S else None
        tb[k, 16] = oracle.unique_mask(g, c, k, None, above).any()
        for j in range(16):
            a = k - 1 - j
            if a >= 0:
                tb[k, j] = oracle.unique_mask(g, c, k, a, above).any()

    def triples(batch):
        return [bool(oracle.unique_mask(g, c, k, None if b < 0 else b, None if a < 0 else a).any())
                for b, k, a in batch]
    return tb, triples


@pytest.mark.parametrize("name", ["ref_spiral_s3", "synth_two_storey_small",
                                  "ref_random_multilayer_s9"])
def test_replay_sweep_matches_oracle(golden, name):
    case = golden["cases"][name]
    if "npz" not in case or "ground" not in case_arrays(case):
        from golden_util import case_input
        t = oracle.build(case_input(name, case), case["d_s"], case["r_g"])
        from golden_util import TABLE_PARAMS
        G = t["ground"]
        Cst = oracle.evaluate(G, t["ceiling"], case["r_g"], TABLE_PARAMS)
    else:
        arr = case_arrays(case)
        G, Cst = arr["ground"], arr["cost"]
    rows = G.shape[1]
    want = oracle.simplify(G, Cst)
    assert want == case["keep"]
    tb, tri = _any_table(G, Cst, slice(0, rows))
    assert sharded.replay_sweep(G.shape[0], tb, tri) == want
    # two bands: per-band any()s max-reduced give the same sweep
    h = rows // 2
    tb0, tri0 = _any_table(G, Cst, slice(0, h))
    tb1, tri1 = _any_table(G, Cst, slice(h, rows))
    merged = np.maximum(tb0, tb1)

    def tri(batch):
        return [a or b for a, b in zip(tri0(batch), tri1(batch))]
    assert sharded.replay_sweep(G.shape[0], merged, tri) == want


def test_expand_table_bits():
    t = np.array([1 << 32 | 1 << 3, 0, (1 << 16) - 1], np.uint64)
    e = sharded.expand_table(t)
    assert e.shape == (3, 17)
    assert e[0, 16] == 1 and e[0, 3] == 1 and e[0].sum() == 2
    assert e[1].sum() == 0 and e[2, :16].sum() == 16 and e[2, 16] == 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _fake_pipeline(rank, size):
    """Exercises every collective kind the band pipeline issues."""
    import torch
    lo, hi, bad = yield ("bounds", np.array([rank, -rank, 2.0 * rank]),
                         np.array([rank + 1.0, 5.0, -1.0]), float(rank == 1))
    assert bad == 1.0  # one rank's flag reaches every rank
    counts = [rank + d + 1 for d in range(size)]
    part = torch.cat([torch.full((counts[d], 3), float(10 * rank + d)) for d in range(size)])
    mine = yield ("alltoallv", part, counts)
    up = torch.full((2, 3, 1, 4), float(rank)) if rank > 0 else None
    down = torch.full((2, 3, 2, 4), float(rank) + 0.5) if rank + 1 < size else None
    top = 2 if rank > 0 else 0
    bot = 1 if rank + 1 < size else 0
    fu, fd = yield ("halo", up, down, (2, 3, top, 4), (2, 3, bot, 4))
    red = yield ("max_u8", np.array([rank, 7 - rank, 3], np.uint8))
    # gather to rank 1: rank 0 sends a (3, 2, 2, 4) band
    cpu = torch.device("cpu")
    if rank == 1:
        got = yield ("gather", None, 1, [(3, 2, 2, 4), (3, 2, 3, 4)], cpu)
        assert got[1] is None and got[0].shape == (3, 2, 2, 4)
        assert torch.all(got[0] == 42.0)
    else:
        got = yield ("gather", torch.full((3, 2, 2, 4), 42.0), 1, None, cpu)
        assert got is None
    return lo, hi, mine, fu, fd, red


def _worker(rank, size, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        lo, hi, mine, fu, fd, red = sharded.run_torch(_fake_pipeline(rank, size))
        q.put((rank, lo.tolist(), hi.tolist(), mine.numpy().tolist(),
               None if fu is None else fu.numpy().tolist(),
               None if fd is None else fd.numpy().tolist(), red.tolist()))
    finally:
        dist.destroy_process_group()


def test_run_torch_collectives_gloo_two_ranks():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(2):
        r = q.get(timeout=120)
        out[r[0]] = r
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    for r in (0, 1):
        _, lo, hi, mine, fu, fd, red = out[r]
        assert lo == [0.0, -1.0, 0.0] and hi == [2.0, 5.0, -1.0]
        # rank r receives counts[r] rows from each source s: value 10*s + r
        rows = np.array(mine)
        exp = np.concatenate([np.full((s + r + 1, 3), 10.0 * s + r) for s in range(2)])
        assert np.array_equal(rows, exp)
        assert red == [1, 7, 3]
    assert np.all(np.array(out[0][5]) == 1.0) and np.array(out[0][5]).shape == (2, 3, 1, 4)
    assert np.all(np.array(out[1][4]) == 0.5) and np.array(out[1][4]).shape == (2, 3, 2, 4)


def test_check_bands_decided_globally():
    """The thin-band error depends only on the shared frame: every rank raises
    (rows=10 over 4 ranks gives bands 2/3/2/3; a 3-row halo fails)."""
    st = sharded.band_starts(10, 4)
    assert [b - a for a, b in zip(st, st[1:])] == [2, 3, 2, 3]
    with pytest.raises(ValueError, match="thinner than"):
        sharded.check_bands(st, 3)
    sharded.check_bands(st, 2)
    sharded.check_bands(sharded.band_starts(4004, 8), 8)
    with pytest.raises(ValueError):
        sharded.check_bands(sharded.band_starts(203, 40), 8)
    # a halo is clipped at the grid edge: an edge band thinner than H is fine
    # when the neighbour's halo reaches the edge anyway; a middle one is not
    sharded.check_bands([0, 10, 12], 3)
    with pytest.raises(ValueError):
        sharded.check_bands([0, 10, 12, 20], 3)
