"""Shared test configuration.

``-m "not gpu"`` runs on CPU (oracle vs golden fixtures, host logic, C-ABI
exports, multi-process gloo paths); ``-m gpu`` runs the CUDA parity tests on a
B200 through the C ABI.  GPU tests never skip silently: without a device they
fail (there is no CPU fallback to hide behind).
"""

import os
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
for p in (os.path.dirname(HERE), HERE):
    if p not in sys.path:
        sys.path.insert(0, p)

from ssb_testutil import golden_cases  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs through libssb.so")


@pytest.fixture(scope="session")
def cases():
    return golden_cases()
