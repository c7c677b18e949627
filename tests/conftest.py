"""Shared fixtures.  `gpu`-marked tests need a B200 (run through gpurun);
everything else runs on the CPU container."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def O():
    """The plain-C oracle (oracle/liboracle.so)."""
    import oracle
    return oracle.load("oracle")


@pytest.fixture(scope="session")
def R():
    """The compiled reference core (oracle/_ref/libref.so), when present."""
    import oracle
    if not oracle.have_ref():
        pytest.skip("oracle/_ref/libref.so not built (needs /root/reference)")
    return oracle.load("ref")


@pytest.fixture(scope="session")
def cuda_ok():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True


def rand_x(rng: np.random.Generator, B: int, n: int, problem: int) -> np.ndarray:
    lo = 0.0 if problem == 0 else -1.0
    return rng.uniform(lo, 1.0, size=(B, n))
