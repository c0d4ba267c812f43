import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
# the reference package (dllmsim) from its offline install, if not importable already
import paper_2605_24832_b200  # noqa: E402,F401


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU and the built C-ABI library")


@pytest.fixture(scope="session")
def golden_dir():
    return ROOT / "tests" / "golden"
