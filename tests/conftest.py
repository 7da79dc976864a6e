"""Shared test setup: the `gpu` marker and import paths.

`-m "not gpu"` tests run on the CPU build container (oracle vs golden
vectors, host logic, ABI surface, gloo multi-process); `-m gpu` tests are the
CUDA parity tests and call the native library through the C ABI.
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)

GOLDEN = os.path.join(TESTS, "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built native library")


@pytest.fixture
def rng():
    return np.random.default_rng(12345)


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)
