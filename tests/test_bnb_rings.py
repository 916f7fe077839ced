"""The compiled weight-class tables of the branch-and-bound inflation kernel
(csrc/bnb_rings.h) are what scripts/gen_bnb_rings.py derives from the
reference's build_kernel formula (traversability.py:194-202).  The library
re-checks any caller's kernel against them at run time; this pins the header."""

import subprocess
import sys
from pathlib import Path

import numpy as np

import oracle

ROOT = Path(__file__).resolve().parents[1]


def test_header_is_current():
    r = subprocess.run([sys.executable, str(ROOT / "scripts" / "gen_bnb_rings.py"), "--check"])
    assert r.returncode == 0, "bnb_rings.h is stale: run scripts/gen_bnb_rings.py"


def test_generator_weights_equal_oracle():
    sys.path.insert(0, str(ROOT / "scripts"))
    import gen_bnb_rings as g
    for r_g, d_inf, d_sm in g.CASES:
        assert np.array_equal(g.weights(d_inf, d_sm, r_g), oracle.kernel_weights(d_inf, d_sm, r_g))


def test_classes_partition_the_positive_taps():
    sys.path.insert(0, str(ROOT / "scripts"))
    import gen_bnb_rings as g
    text = g.render()
    for r_g, d_inf, d_sm in g.CASES:
        w = g.weights(d_inf, d_sm, r_g)
        R = w.shape[0] // 2
        vals = sorted({float(v) for v in w.ravel() if v > 0}, reverse=True)
        # class 0 is the compiled disk a^2 + b^2 <= (d_inf / r_g)^2 (DiskShape)
        a, b = np.meshgrid(np.arange(-R, R + 1), np.arange(-R, R + 1), indexing="ij")
        disk = a * a + b * b <= round(d_inf / r_g) ** 2
        assert np.array_equal(w == vals[0], disk)
        assert f"struct BnbRings<{R}>" in text and f"NCLS = {len(vals)};" in text
