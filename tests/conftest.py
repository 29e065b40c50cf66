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


def metrics_inputs():
    """The seeded inputs of tests/golden/metrics_small.npz (same PCG64 streams as make_golden.py)."""
    import numpy as np

    rng = np.random.default_rng(21)
    a = rng.random((64, 80, 3))
    b = np.clip(a + 0.05 * rng.standard_normal(a.shape), 0, 1)
    yy, xx = np.mgrid[0:192, 0:256]
    big_a = np.stack([np.exp(-((xx - 90 - 20 * c) ** 2 + (yy - 100) ** 2) / 3000.0) for c in range(3)], -1)
    big_b = np.clip(big_a + 0.02 * rng.standard_normal(big_a.shape), 0, 1)
    s = a[:32, :40]
    seq_p = [np.clip(s + 0.03 * k + 0.02 * rng.standard_normal(s.shape), 0, 1) for k in range(4)]
    seq_g = [np.clip(s + 0.03 * k, 0, 1) for k in range(4)]
    return a, b, big_a, big_b, seq_p, seq_g
