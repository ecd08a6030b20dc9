import os
import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "tests"))  # test helpers (large_golden)
TESTS_DIR = REPO / "tests"
# the reference frontend, when installed beside the repo (baseline/_ref) or
# present in this container; never required by the -m gpu parity tests
for cand in (REPO / "baseline" / "_ref", Path("/root/reference/pkg/src")):
    if (cand / "lagen").is_dir() and str(cand) not in sys.path:
        sys.path.append(str(cand))
        break

os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def has_lagen():
    try:
        import lagen  # noqa: F401
        return True
    except Exception:
        return False


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle
    oracle.build()
    return oracle
