"""Shared fixtures; mirrors the reference's pkg/tests/conftest.py (rel_err at :29-32, rng at :40-42)."""
from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libjigsaw_sm100.so")


def rel_err(actual, expected) -> float:
    """max|a - e| / max|e| — the reference's tolerance metric (conftest.py:29-32)."""
    a = np.asarray(actual, dtype=np.float64)
    e = np.asarray(expected, dtype=np.float64)
    denom = np.max(np.abs(e))
    if denom == 0:
        return float(np.max(np.abs(a)))
    return float(np.max(np.abs(a - e)) / denom)


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2507_05753_b200 import _lib
    _lib.load()
    return torch.device("cuda:0")
