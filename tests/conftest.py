"""Shared test configuration.

Markers: `gpu` — needs a CUDA device (run on the B200 box with `-m gpu`);
everything else runs on the CPU build container (`-m "not gpu"`).
"""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: multi-second CPU work")


@pytest.fixture
def rng():
    import numpy as np
    return np.random.default_rng(1234)
