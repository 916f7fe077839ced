"""Binary PCD ingest (SURVEY.md §8 f rank 3): the oracle and the host-side
header validation against the reference's recorded outcomes (CPU), and the
device ingest (pct_pcd_load / pct_pcd_extract) against both (GPU).

Reference tests this mirrors: test_cloud_io.py round trips and malformed-file
cases for pcd_binary; outcomes pinned in tests/golden/golden_pcd.json."""

from __future__ import annotations

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

import pcd_cases

GOLD = json.loads((Path(__file__).parent / "golden" / "golden_pcd.json").read_text())["cases"]
OK_CASES = [k for k, v in GOLD.items() if "error" not in v]
ERR_CASES = [k for k, v in GOLD.items() if "error" in v]
# errors raised by the header / size checks before any device work
HOST_ERR_CASES = [k for k in ERR_CASES if GOLD[k]["message"] != "<path>: zero valid points"]


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _oracle_load(path):
    from oracle import cloud_io as ocio
    from paper_2403_07631_b200.cloud_io import _binary_layout, pcd_record_dtype, read_pcd_header
    with open(path, "rb") as fh:
        names, sizes, kinds, counts, n, data = pcd_record_dtype(read_pcd_header(fh))
        dt = _binary_layout(names, sizes, kinds, counts)
        payload = fh.read(dt.itemsize * n)
    return ocio.extract(payload, n, dt.itemsize, [dt.fields[a][1] for a in "xyz"])


@pytest.mark.parametrize("name", list(GOLD))
def test_case_files_are_the_golden_ones(name, tmp_path):
    path = pcd_cases.write_case(name, tmp_path)
    assert hashlib.sha256(path.read_bytes()).hexdigest() == GOLD[name]["file_sha256"]


@pytest.mark.parametrize("name", OK_CASES)
def test_oracle_matches_reference(name, tmp_path):
    xyz, dropped = _oracle_load(pcd_cases.write_case(name, tmp_path))
    g = GOLD[name]
    assert (xyz.shape[0], dropped) == (g["n"], g["dropped"])
    assert _sha(xyz) == g["xyz_sha256"]


@pytest.mark.parametrize("name", HOST_ERR_CASES)
def test_header_errors_match_reference(name, tmp_path):
    from paper_2403_07631_b200 import cloud_io
    path = pcd_cases.write_case(name, tmp_path)
    with pytest.raises(Exception) as ei:
        cloud_io.load_cloud(path, "pcd_binary")
    g = GOLD[name]
    assert type(ei.value).__name__ == g["error"]
    assert str(ei.value).replace(str(path), "<path>") == g["message"]


def test_load_cloud_arguments(tmp_path):
    from paper_2403_07631_b200 import CloudFormatError, cloud_io
    with pytest.raises(ValueError, match="unknown format"):
        cloud_io.load_cloud(tmp_path / "a.pcd", "las")
    with pytest.raises(CloudFormatError, match="no such file"):
        cloud_io.load_cloud(tmp_path / "missing.pcd", "pcd_binary")
    p = pcd_cases.write_case("plain_xyz", tmp_path)
    assert cloud_io.sniff_format(p) == "pcd_binary"
    assert cloud_io.sniff_format(pcd_cases.write_case("ascii_data", tmp_path)) == "pcd_ascii"
    assert cloud_io.sniff_format(tmp_path / "x.ply") == "ply_ascii"
    assert cloud_io.sniff_format(tmp_path / "x.txt") == "xyz_text"


# ----------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("chunk", [0, 4096 * 16 + 12])
@pytest.mark.parametrize("name", OK_CASES)
def test_device_ingest_matches_reference(name, chunk, tmp_path):
    from paper_2403_07631_b200 import cloud_io
    path = pcd_cases.write_case(name, tmp_path)
    cloud = cloud_io.load_pcd_binary(path, chunk_bytes=chunk)
    g = GOLD[name]
    assert (len(cloud), cloud.dropped) == (g["n"], g["dropped"])
    assert cloud.points.dtype == np.float32         # what the device path keeps
    xyz = cloud.xyz                                  # the reference's float64 view
    assert xyz.dtype == np.float64
    assert _sha(xyz) == g["xyz_sha256"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", [k for k in ERR_CASES if k not in HOST_ERR_CASES])
def test_device_ingest_errors(name, tmp_path):
    from paper_2403_07631_b200 import cloud_io
    path = pcd_cases.write_case(name, tmp_path)
    with pytest.raises(Exception) as ei:
        cloud_io.load_cloud(path, "pcd_binary")
    g = GOLD[name]
    assert type(ei.value).__name__ == g["error"]
    assert str(ei.value).replace(str(path), "<path>") == g["message"]


@pytest.mark.gpu
def test_records_in_memory_and_bounds(tmp_path):
    from paper_2403_07631_b200 import cloud_io
    path = pcd_cases.write_case("nonfinite_rows", tmp_path)
    with open(path, "rb") as fh:
        names, sizes, kinds, counts, n, _ = cloud_io.pcd_record_dtype(cloud_io.read_pcd_header(fh))
        dt = cloud_io._binary_layout(names, sizes, kinds, counts)
        rec = np.frombuffer(fh.read(dt.itemsize * n), dt, count=n)
    cloud = cloud_io.pcd_records_to_device(rec)
    ref, dropped = _oracle_load(path)
    assert cloud.dropped == dropped
    np.testing.assert_array_equal(cloud.xyz.astype(np.float64), ref)
    lo, hi = cloud.bounds
    np.testing.assert_array_equal(lo, ref.min(axis=0))
    np.testing.assert_array_equal(hi, ref.max(axis=0))


@pytest.mark.gpu
def test_build_from_device_cloud_equals_host_build(tmp_path):
    """A PCD-ingested cloud builds in place (no host copy) and gives the same
    bytes as building from the host points."""
    from paper_2403_07631_b200 import PointCloud, build_tomogram, cloud_io, synth
    xyz = synth.two_storey(200_000, seed=3).astype(np.float32)
    xyz[::997, 2] = np.nan  # dropped at ingest
    head = ("VERSION 0.7\nFIELDS x y z\nSIZE 4 4 4\nTYPE F F F\nCOUNT 1 1 1\n"
            f"WIDTH {len(xyz)}\nHEIGHT 1\nPOINTS {len(xyz)}\nDATA binary\n").encode()
    path = tmp_path / "scene.pcd"
    path.write_bytes(head + xyz.tobytes())
    dev = cloud_io.load_cloud(path, "pcd_binary")
    good = xyz[np.isfinite(xyz).all(axis=1)]
    assert dev.dropped == len(xyz) - len(good)
    a = build_tomogram(dev, 0.5, 0.1)
    b = build_tomogram(PointCloud(good), 0.5, 0.1)
    assert len(a.slices) == len(b.slices)
    for sa, sb in zip(a.slices, b.slices):
        assert sa.ground.values.tobytes() == sb.ground.values.tobytes()
        assert sa.ceiling.values.tobytes() == sb.ceiling.values.tobytes()


def _reference_tomoplan():
    """The reference package, where it is importable (the build container)."""
    import sys
    from pathlib import Path
    src = Path("/root/reference/pkg/src")
    if src.is_dir() and str(src) not in sys.path:
        sys.path.append(str(src))
    return pytest.importorskip("tomoplan")


def test_product_load_cloud_has_no_text_parsers(tmp_path):
    """The product reads pcd_binary only; text formats raise (no CPU
    fallback through the reference inside the package)."""
    from paper_2403_07631_b200 import CloudFormatError, cloud_io
    p = tmp_path / "pts.xyz"
    p.write_text("0 0 0\n1 2 3\n")
    for fmt in ("xyz_text", "pcd_ascii", "ply_ascii"):
        with pytest.raises(CloudFormatError, match="no device ingest"):
            cloud_io.load_cloud(p, fmt)
    import paper_2403_07631_b200 as pkg
    for mod in ("cloud_io", "cloud", "tomogram", "traversability", "simplify", "sharded",
                "batch", "archive", "planner_ctx", "trajectory"):
        src = (Path(pkg.__file__).parent / f"{mod}.py").read_text()
        code = "\n".join(ln for ln in src.splitlines() if not ln.strip().startswith("#"))
        assert "import tomoplan" not in code and "from tomoplan" not in code, mod


def test_compat_dispatches_text_formats_to_the_reference(tmp_path):
    """After compat.install, tomoplan.load_cloud keeps the reference's
    parser for text formats (cloud_io.py:281-288) and uses the device ingest
    for pcd_binary."""
    tp = _reference_tomoplan()
    from paper_2403_07631_b200 import compat
    p = tmp_path / "pts.xyz"
    p.write_text("# comment\n0 0 0\n1.5 2 3\nnan 1 1\n")
    want = tp.load_cloud(p, "xyz_text")
    compat.install(tp)
    try:
        got = tp.load_cloud(p, "xyz_text")
        assert type(got) is type(want)
        assert np.array_equal(got.xyz, want.xyz) and got.dropped == want.dropped == 1
        assert tp.cloud_io.load_cloud is tp.load_cloud
    finally:
        compat.uninstall()
    assert tp.load_cloud(p, "xyz_text").dropped == 1
