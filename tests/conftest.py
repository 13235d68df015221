import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

GOLD = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs through libvxg.so)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def load(name):
        if name not in cache:
            cache[name] = np.load(GOLD / f"{name}.npz")
        return cache[name]

    return load


@pytest.fixture(scope="session")
def oracle():
    from oracle.refbind import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1606_05688_b200 import Context
    return Context(0)


def rel_error(a, b) -> float:
    """oracle::rel_error (proj/tests/oracles.hpp:41-50): max|a-b| / max|b|."""
    cplx = np.iscomplexobj(a) or np.iscomplexobj(b)
    dt = np.complex128 if cplx else np.float64  # rel_error_complex, oracles.hpp:52-61
    a = np.asarray(a, dt)
    b = np.asarray(b, dt)
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b))) / max(float(np.max(np.abs(b))), 1e-300)
