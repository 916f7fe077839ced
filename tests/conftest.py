import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))
# the reference package, importable only in the build container (CPU tests
# that compare against it skip elsewhere; nothing on the GPU box reads it)
_REF = Path("/root/reference/pkg/src")
if _REF.is_dir() and str(_REF) not in sys.path:
    sys.path.append(str(_REF))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: takes more than a few seconds on CPU")


@pytest.fixture(scope="session")
def golden():
    from golden_util import load_golden
    return load_golden()
