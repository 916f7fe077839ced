"""CPU checks of the C ABI boundary: libpct.so loads without a GPU, exports
every function include/pct.h declares, and the ctypes binding covers them."""

import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "pct.h"
LIB = ROOT / "paper_2403_07631_b200" / "lib" / "libpct.so"


def header_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(pct_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__
    __graft_entry__.build()  # incremental
    from paper_2403_07631_b200 import _lib
    return _lib.load()


def test_header_declares_the_binding():
    from paper_2403_07631_b200 import _lib
    assert header_functions() == _lib.declared_symbols()


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", str(LIB)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (pct_[a-z0-9_]+)", out))
    missing = set(header_functions()) - exported
    assert not missing, f"declared but not exported: {sorted(missing)}"
    for name in header_functions():
        assert hasattr(lib, name)


def test_abi_version_and_no_device(lib):
    import ctypes as C
    assert lib.pct_abi_version() == 1
    h = C.c_void_p()
    import torch
    if not torch.cuda.is_available():
        assert lib.pct_ctx_create(0, C.byref(h)) != 0   # fails loudly, no CPU fallback


def test_frame_compute_matches_reference_formula(lib):
    """pct_frame_compute is host code: check it against tomogram.py:138-145
    (restated in the oracle) on random bounds, bit for bit."""
    import ctypes as C

    import numpy as np

    import oracle
    from paper_2403_07631_b200 import _lib
    rng = np.random.default_rng(0)
    for _ in range(2000):
        lo = rng.uniform(-500, 500, 3)
        hi = lo + rng.uniform(0, 60, 3)
        d_s, r_g = float(rng.uniform(0.05, 1.0)), float(rng.uniform(0.02, 0.5))
        fr = _lib.FrameC()
        hts = np.empty(4096)
        rc = lib.pct_frame_compute(lo.ctypes.data, hi.ctypes.data, d_s, r_g, 16384, C.byref(fr),
                                   hts.ctypes.data, 4096)
        want = oracle.frame(lo, hi, d_s, r_g)
        assert rc == 0
        assert (fr.rows, fr.cols) == (want["rows"], want["cols"])
        assert fr.n_slices == len(want["heights"])
        assert np.array_equal(hts[:fr.n_slices], want["heights"])
    # grid limit -> PCT_E_GRID
    lo, hi = np.zeros(3), np.array([100.0, 100.0, 1.0])
    fr = _lib.FrameC()
    assert lib.pct_frame_compute(lo.ctypes.data, hi.ctypes.data, 0.5, 0.005, 1000, C.byref(fr),
                                 None, 0) == _lib.PCT_E_GRID
