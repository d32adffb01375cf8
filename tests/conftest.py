import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (large band-limits)")


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def load(name):
        if name not in cache:
            cache[name] = dict(np.load(GOLDEN / f"{name}.npz"))
        return cache[name]

    return load


def rel_err(x, ref):
    """Normwise relative error max|x - ref| / max|ref|."""
    x, ref = np.asarray(x), np.asarray(ref)
    scale = np.abs(ref).max()
    if scale == 0:
        return float(np.abs(x).max())
    return float(np.abs(x - ref).max() / scale)
