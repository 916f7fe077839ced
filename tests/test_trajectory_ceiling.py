"""Trajectory ceiling inflation (SURVEY.md §8 f rank 4,
trajectory.py:277-317): oracle pinned to the reference's outputs (CPU), the
device kernels pinned to both (GPU)."""

from __future__ import annotations

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

import traj_cases

GOLD = json.loads((Path(__file__).parent / "golden" / "golden_traj.json").read_text())["cases"]
LAYERS = {name: (v, res) for name, v, res in traj_cases.layers()}


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _ids(c):
    return f"{c['layer']}-e{c['erosion']}-s{c['slope']}"


@pytest.mark.parametrize("case", GOLD, ids=_ids)
def test_oracle_matches_reference(case):
    from oracle import trajectory as otraj
    v, res = LAYERS[case["layer"]]
    assert _sha(v) == case["values_sha256"]
    flat, skirt = otraj.inflate_ceiling(v, np.isfinite(v), res, case["erosion"], case["slope"])
    assert flat.dtype == np.float64 and skirt.dtype == np.float64
    assert _sha(flat) == case["flat_sha256"]
    assert _sha(skirt) == case["skirted_sha256"]


def test_compat_replaces_inflate_ceiling():
    from paper_2403_07631_b200 import compat, trajectory
    assert compat.REPLACEMENTS["_inflate_ceiling"] is trajectory.inflate_ceiling
    assert ".trajectory" in compat.MODULES


@pytest.mark.gpu
@pytest.mark.parametrize("case", GOLD, ids=_ids)
def test_device_matches_reference(case):
    from paper_2403_07631_b200.trajectory import inflate_ceiling
    v, res = LAYERS[case["layer"]]
    flat, skirt = inflate_ceiling(v, np.isfinite(v), res, case["erosion"], case["slope"])
    assert _sha(flat) == case["flat_sha256"]
    assert _sha(skirt) == case["skirted_sha256"]


@pytest.mark.gpu
def test_all_slices_of_a_device_tomogram():
    """One call for every slice of a built tomogram (ceiling stack read in
    place) equals the per-slice oracle; cfg0-sized grid, many 64x64 tiles."""
    from oracle import trajectory as otraj
    from paper_2403_07631_b200 import PointCloud, build_tomogram, synth
    from paper_2403_07631_b200.trajectory import inflate_ceilings
    tom = build_tomogram(PointCloud(synth.two_storey(250_000, seed=0)), 0.5, 0.1)
    flat, skirt = inflate_ceilings(tom)
    assert flat.shape == (len(tom.slices), tom.rows, tom.cols)
    for k, sl in enumerate(tom.slices):
        c = sl.ceiling.values
        f, s = otraj.inflate_ceiling(c, np.isfinite(c), 0.1, 0.20, 0.30)
        assert flat[k].tobytes() == f.tobytes(), k
        assert skirt[k].tobytes() == s.tobytes(), k
