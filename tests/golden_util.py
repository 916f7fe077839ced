"""Helpers to read tests/golden (fixtures written by tests/golden/make_golden.py)."""

import hashlib
import json
from pathlib import Path
from types import SimpleNamespace

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"

# TravParams defaults (traversability.py:25-37; Table I)
TABLE_PARAMS = SimpleNamespace(d_min=0.50, d_ref=0.65, theta_b=1.70, theta_s=0.36,
                               theta_p=0.20, c_barrier=50.0, alpha_d=20.0, alpha_b=20.0,
                               alpha_s=15.0, d_inf=0.20, d_sm=0.40, r_c=0.20,
                               step_patch_radius=None)


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def load_golden():
    return json.loads((GOLDEN / "golden.json").read_text())


def case_input(name, case):
    """The case's input cloud: from its npz, or regenerated from synth."""
    if case["source"] == "tomoplan.generate_scene":
        return np.load(GOLDEN / case["npz"])["xyz"]
    from paper_2403_07631_b200 import synth
    if case["source"] == "paper_2403_07631_b200.synth":
        xyz = synth.generate(case["config"], case["n_override"])
    else:
        xyz = synth.two_storey(case["n"], seed=case["seed"])
    assert digest(xyz) == case["input_sha256"], f"{name}: generator drift"
    return xyz


def case_arrays(case):
    return np.load(GOLDEN / case["npz"]) if "npz" in case else None
