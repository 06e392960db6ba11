"""Test configuration: `gpu` marks tests that need a B200 and libqmb200.so (run with -m gpu)."""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libqmb200.so")
    config.addinivalue_line("markers", "slow: large configurations (tens of GB on the device)")


@pytest.fixture(autouse=True)
def _fixed_numpy_printoptions():
    with np.printoptions(precision=17):
        yield
