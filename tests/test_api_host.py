"""Host-side behaviour of the drop-in API that needs no GPU: parameter
objects, kernel weights, validation order and error types, the compat
installer."""

import numpy as np
import pytest

import oracle
import paper_2403_07631_b200 as pct


def test_travparams_defaults_and_invariants():
    p = pct.TravParams()
    assert (p.d_min, p.d_ref, p.theta_b, p.theta_s, p.theta_p, p.c_barrier) == \
        (0.5, 0.65, 1.7, 0.36, 0.2, 50.0)
    assert p.patch_radius(0.1) == 3 and p.patch_radius(0.05) == 6 and p.patch_radius(0.2) == 2
    for bad in (dict(d_min=0.7), dict(theta_s=2.0), dict(theta_p=1.5), dict(c_barrier=0),
                dict(d_inf=0.5), dict(r_c=0.3)):
        with pytest.raises(ValueError):
            pct.TravParams(**bad)


@pytest.mark.parametrize("r_g", [0.1, 0.05, 0.2, 0.15])
def test_build_kernel_matches_oracle(r_g):
    k = pct.build_kernel(0.2, 0.4, r_g)
    assert np.array_equal(k.weights, oracle.kernel_weights(0.2, 0.4, r_g))
    assert k.radius_cells == int(np.ceil(0.4 / r_g))
    ws = [w for w, _ in k.weight_classes()]
    assert ws == sorted(ws, reverse=True) and all(w > 0 for w in ws)
    with pytest.raises(ValueError):
        pct.build_kernel(0.4, 0.4, 0.1)
    with pytest.raises(ValueError):
        pct.build_kernel(0.05, 0.4, 0.1)


def test_rasterize_index_kats():
    # test_tomogram.py:10-33
    assert pct.rasterize_index((0.0, 0.0), (0.0, 0.0), 0.1) == (0, 0)
    assert pct.rasterize_index((0.26, 0.14), (0.0, 0.0), 0.1) == (1, 3)
    assert pct.rasterize_index((-0.06, 0.0), (0.0, 0.0), 0.1) == (0, -1)
    with pytest.raises(IndexError):
        pct.rasterize_index((-0.06, 0.0), (0.0, 0.0), 0.1, shape=(10, 10))
    rng = np.random.default_rng(5)
    for _ in range(200):
        x, y = rng.uniform(-3, 3, 2)
        r = rng.uniform(0.05, 0.5)
        assert pct.rasterize_index((x, y), (0.0, 0.0), r) == \
            (int(np.floor(y / r + 0.5)), int(np.floor(x / r + 0.5)))


def test_pointcloud_validation():
    with pytest.raises(pct.CloudFormatError):
        pct.PointCloud(np.zeros((0, 3)))
    with pytest.raises(ValueError):
        pct.PointCloud(np.zeros((3, 2)))
    with pytest.raises(ValueError):
        pct.PointCloud(np.array([[0.0, np.nan, 0.0]]))
    # xyz is float64 like the reference's (cloud_io.py:35); the device path
    # uploads the caller's float32 array (``points``) without that copy
    f32 = np.arange(6, dtype=np.float32).reshape(2, 3) + 0.1
    c = pct.PointCloud(f32)
    assert c.points.dtype == np.float32 and c.points is not None
    assert c.xyz.dtype == np.float64 and c.xyz.flags.c_contiguous
    assert np.array_equal(c.xyz, f32.astype(np.float64))
    assert pct.PointCloud(np.zeros((2, 3), np.int32)).xyz.dtype == np.float64
    assert len(c) == 2 and c.dropped == 0 and pct.PointCloud(f32, 3).dropped == 3


def test_argument_errors_before_any_device_call():
    cloud = pct.PointCloud(np.ones((3, 3)))
    for d_s, r_g in ((0.0, 0.1), (0.5, -1.0)):
        with pytest.raises(ValueError, match="d_s and r_g must be positive"):
            pct.build_tomogram(cloud, d_s, r_g)
    g = pct.Layer(np.zeros((2, 2)), 0.1, (0, 0))
    c = pct.Layer(np.zeros((3, 2)), 0.1, (0, 0))
    with pytest.raises(ValueError, match="misaligned"):
        pct.interval_cost(g, c, pct.TravParams())
    with pytest.raises(ValueError):
        pct.Layer(np.zeros((0, 3)), 0.1, (0, 0))
    with pytest.raises(ValueError):
        pct.Layer(np.zeros((2, 3)), 0.0, (0, 0))


def test_unique_cells_errors_before_device():
    from paper_2403_07631_b200.tomogram import Tomogram, TomogramSlice, Layer
    z = np.zeros((3, 3), np.float32)
    t = Tomogram([TomogramSlice(Layer(z, 0.1, (0, 0)), Layer(z, 0.1, (0, 0)), 0.5, 0),
                  TomogramSlice(Layer(z, 0.1, (0, 0)), Layer(z, 0.1, (0, 0)), 1.0, 1)], 0.5, 0.0)
    with pytest.raises(IndexError):
        pct.unique_cells(t, 5)
    with pytest.raises(ValueError, match="cost layer"):
        pct.unique_cells(t, 0)
    with pytest.raises(ValueError, match="cost layer"):
        pct.simplify_tomogram(t)
    one = Tomogram([TomogramSlice(Layer(z, 0.1, (0, 0)), Layer(z, 0.1, (0, 0)), 0.5, 0)], 0.5, 0.0)
    out = pct.simplify_tomogram(one)            # single slice: returned unchanged, no error
    assert len(out.slices) == 1 and out.slices[0].index == 0


def test_compat_install_patches_reference_names():
    tomoplan = pytest.importorskip("tomoplan")  # only where the reference is importable
    from paper_2403_07631_b200 import compat
    patched = compat.install(tomoplan)
    try:
        assert tomoplan.build_tomogram is pct.build_tomogram
        assert tomoplan.tomogram.build_tomogram is pct.build_tomogram
        assert tomoplan.traversability.evaluate_tomogram is pct.evaluate_tomogram
        assert tomoplan.simplify.simplify_tomogram is pct.simplify_tomogram
        assert tomoplan.cli.build_tomogram is pct.build_tomogram
        assert len(patched) >= 12
    finally:
        compat.uninstall()
    assert tomoplan.build_tomogram is not pct.build_tomogram
