import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libntdgpu.so")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture
def rng():
    # same seed as the reference suite (tests/conftest.py:13-15)
    return np.random.default_rng(20240811)


@pytest.fixture(scope="session")
def golden():
    return np.load(os.path.join(GOLDEN, "small_cases.npz"))


def grid_of(name):
    return tuple(int(t) for t in name.split("_")[0][1:].split("x"))
