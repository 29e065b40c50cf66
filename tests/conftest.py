import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libfovnet.so")


@pytest.fixture(scope="session")
def golden():
    return GOLDEN


@pytest.fixture(scope="session")
def stack_values():
    from oracle import fovray_oracle as O

    return O.load_rnkstack(ROOT / "paper_2209_09965_b200" / "data" / "stbn_64x64x8_s1.noise")
