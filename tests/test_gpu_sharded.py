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


@pytest.mark.parametrize("P", [1, 3])
def test_virtual_bands_tiled_build(golden, monkeypatch, P):
    """The tile-partitioned build (chosen automatically for maps whose key
    planes exceed ~1.5 GB, e.g. config 3) on row bands."""
    monkeypatch.setenv("PCT_BUILD", "tiled")
    case = golden["cases"]["synth_cfg0"]
    xyz = case_input("synth_cfg0", case)
    monkeypatch.setenv("PCT_BUILD", "atomic")
    g1, c1, k1, keep1 = _single(xyz, 0.5, 0.1)
    monkeypatch.setenv("PCT_BUILD", "tiled")
    g2, c2, k2, keep2 = _sharded(xyz, 0.5, 0.1, P)
    assert np.array_equal(g1.view(np.uint32), g2.view(np.uint32))
    assert np.array_equal(c1.view(np.uint32), c2.view(np.uint32))
    assert np.array_equal(k1.view(np.uint32), k2.view(np.uint32))
    assert keep1 == keep2 == case["keep"]
