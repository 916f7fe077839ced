"""Compacted read-back of layer slices (csrc/k_xfer.cu, Tomogram.materialize):
lossless for every bit pattern, and the drop-in chain's host layers are the
same with and without it."""
import numpy as np
import pytest

import paper_2403_07631_b200 as pct
from golden_util import case_input, digest

pytestmark = pytest.mark.gpu


def _roundtrip(stack, ks, delta=False):
    tot = stack.count_nonempty(ks, delta=delta)
    p = stack.compact_start(list(ks), [int(t) for t in tot], delta)
    with stack.ctx.lock:
        stack.ctx.check(stack.ctx.lib.pct_sync(stack.ctx.h), "sync")
    stack.compact_finish(p, 8)
    return tot, [stack._host[k] for k in ks]


@pytest.mark.parametrize("rows,cols", [(1024, 1024), (1023, 1031), (7, 5)])
def test_compacted_slices_are_bit_exact(rows, cols):
    from paper_2403_07631_b200 import _lib
    from paper_2403_07631_b200.tomogram import DeviceStack
    rng = np.random.default_rng(rows * 7 + cols)
    n = 6
    a = rng.standard_normal((n, rows, cols)).astype(np.float32)
    u = a.view(np.uint32)
    empty = np.uint32(0x7FC00000)
    u[0] = empty                                   # all empty
    # slice 1 keeps every value; the others a random share of empty cells
    for k, share in ((2, 0.75), (3, 0.5), (4, 0.97), (5, 0.2)):
        u[k][rng.random((rows, cols)) < share] = empty
    # bit patterns that must travel as values: other NaN payloads, -0.0, inf
    u[3].flat[::97] = np.uint32(0x7FC00001)
    u[3].flat[5::89] = np.uint32(0xFFC00000)
    u[4].flat[::101] = np.uint32(0x80000000)
    u[5].flat[::103] = np.uint32(0x7F800000)
    ctx = _lib.context(0)
    buf = _lib.DeviceBuffer.from_host(ctx, a)
    stack = DeviceStack(ctx, buf.ptr, n, rows, cols, buf)
    ks = [0, 1, 2, 3, 4, 5]
    tot, got = _roundtrip(stack, ks)
    assert list(tot) == [int((u[k] != empty).sum()) for k in ks]
    for k, g in zip(ks, got):
        assert np.array_equal(g.view(np.uint32), u[k]), f"slice {k}"
    # a subset in another order, one slice repeated in a separate call
    stack2 = DeviceStack(ctx, buf.ptr, n, rows, cols, buf)
    _, got = _roundtrip(stack2, [4, 2])
    assert np.array_equal(got[0].view(np.uint32), u[4])
    assert np.array_equal(got[1].view(np.uint32), u[2])
    # delta chains: each slice against the previous listed one
    for ks in ([0, 1, 2, 3, 4, 5], [5, 3, 1], [2]):
        st = DeviceStack(ctx, buf.ptr, n, rows, cols, buf)
        tot, got = _roundtrip(st, ks, delta=True)
        prev = np.full(u[0].shape, 0x7FC00000, np.uint32)
        for k, t, g in zip(ks, tot, got):
            assert int(t) == int((u[k] != prev).sum())
            assert np.array_equal(g.view(np.uint32), u[k]), f"delta slice {k}"
            prev = u[k]
    # the pack from the count pass's kept chunk counts (pct_xfer_pack_counted)
    for delta in (False, True):
        ks = [0, 1, 2, 3, 4, 5]
        st = DeviceStack(ctx, buf.ptr, n, rows, cols, buf)
        tot = _lib.pinned_pool(ctx).array((len(ks),), np.int64)
        st.count_nonempty_async(ks, delta, tot, keep=True)
        with st.ctx.lock:
            st.ctx.check(st.ctx.lib.pct_sync(st.ctx.h), "sync")
        assert st._kept is not None
        p = st.compact_start(ks, [int(t) for t in tot], delta)
        assert st._kept is None
        with st.ctx.lock:
            st.ctx.check(st.ctx.lib.pct_sync(st.ctx.h), "sync")
        st.compact_finish(p, 8)
        for k in ks:
            assert np.array_equal(st._host[k].view(np.uint32), u[k]), f"kept {delta} slice {k}"
    # a delta chain copied and rebuilt in parts (pct_xfer_expand_from: the
    # second part continues from the rebuilt slice before it; ragged tails)
    for split in ((1,), (2,), (4,), (1, 3), (2, 3, 5)):
        ks = [0, 1, 2, 3, 4, 5]
        st = DeviceStack(ctx, buf.ptr, n, rows, cols, buf)
        tot = st.count_nonempty(ks, delta=True)
        fences = []
        p = st.compact_start(ks, [int(t) for t in tot], True, split=split,
                             fence=lambda: fences.append(1))
        assert len(fences) == len(split)
        with st.ctx.lock:
            st.ctx.check(st.ctx.lib.pct_sync(st.ctx.h), "sync")
        cuts = [0, *split, len(ks)]
        for a, b in zip(cuts[:-1], cuts[1:]):
            st.compact_finish(p, 8, part=(a, b))
        for k in ks:
            assert np.array_equal(st._host[k].view(np.uint32), u[k]), f"split {split} slice {k}"


@pytest.mark.parametrize("mode", ["1", "nan", "0"])
def test_materialize_modes_match_dense(golden, monkeypatch, mode):
    """The default read-back (delta chains where consecutive slices share
    most cells), NaN compaction only, and dense copies: the reference's
    layers, every slice."""
    name = "synth_cfg2_n2000000"
    case = golden["cases"][name]
    xyz = case_input(name, case)
    monkeypatch.setenv("PCT_XFER_COMPACT", mode)
    tom = pct.evaluate_tomogram(pct.build_tomogram(pct.PointCloud(xyz), case["d_s"], case["r_g"]),
                                pct.TravParams())
    tom.materialize()  # every slice (not only the kept ones): long chains
    for k, s in enumerate(tom.slices):
        assert digest(s.ground.values) == case["ground_slice_sha256"][k]
        assert digest(s.ceiling.values) == case["ceiling_slice_sha256"][k]
        assert digest(s.cost.values) == case["cost_slice_sha256"][k]


def test_materialize_compacted_matches_dense(golden, monkeypatch):
    """The drop-in chain (build -> evaluate -> simplify -> materialize) on a
    map of 4M cells: every surviving layer equal with the compacted read-back
    (the default) and with dense copies only, and equal to the reference's
    digests."""
    name = "synth_cfg2_n2000000"
    case = golden["cases"][name]
    xyz = case_input(name, case)

    def chain():
        tom = pct.simplify_tomogram(pct.evaluate_tomogram(
            pct.build_tomogram(pct.PointCloud(xyz), case["d_s"], case["r_g"]), pct.TravParams()))
        tom.materialize()
        return [(s.ground.values.copy(), s.ceiling.values.copy(), s.cost.values.copy())
                for s in tom.slices]

    got = chain()
    monkeypatch.setenv("PCT_XFER_COMPACT", "0")
    want = chain()
    assert len(got) == len(want) == len(case["keep"])
    for (g, c, k), (g2, c2, k2), kk in zip(got, want, case["keep"]):
        assert np.array_equal(g.view(np.uint32), g2.view(np.uint32))
        assert np.array_equal(c.view(np.uint32), c2.view(np.uint32))
        assert np.array_equal(k.view(np.uint32), k2.view(np.uint32))
        assert digest(g) == case["ground_slice_sha256"][kk]
        assert digest(c) == case["ceiling_slice_sha256"][kk]
        assert digest(k) == case["cost_slice_sha256"][kk]


def test_materialize_campus_frame_matches_reference():
    """The full 4004 x 4004 campus frame at 8M points (tests/golden/
    golden_r2.json "campus_sparse"): its kept slices mix dense layers and
    mostly-empty ones; materialize() (compacted where they are mostly empty)
    gives the reference's per-slice digests."""
    import json

    from golden_util import GOLDEN
    from paper_2403_07631_b200 import synth
    case = json.loads((GOLDEN / "golden_r2.json").read_text())["cases"]["campus_sparse"]
    box = tuple(case["box"]) if case["box"] else None
    xyz = synth.campus(case["n_full"], case["seed"], box=box)
    tom = pct.simplify_tomogram(pct.evaluate_tomogram(
        pct.build_tomogram(pct.PointCloud(xyz), case["d_s"], case["r_g"]), pct.TravParams()))
    tom.materialize()
    assert len(tom.slices) == len(case["keep"])
    for s, k in zip(tom.slices, case["keep"]):
        assert digest(s.ground.values) == case["ground_slice_sha256"][k]
        assert digest(s.ceiling.values) == case["ceiling_slice_sha256"][k]
