"""Shared fixtures.  `-m gpu` tests need a CUDA device and the built libaqp.so;
`-m "not gpu"` tests run anywhere (oracle, host logic, ABI surface)."""

import json
import os
import sys

# Row-shard tests run several virtual ranks (one CUDA stream each) on the one
# GPU of the test box; their spinning exchanges need every rank's stream on
# its own hardware queue (no head-of-line blocking behind another rank), so
# ask for the maximum number of queues before CUDA is initialised.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libaqp.so")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture
def rng():
    # same seed as the reference's suite (tests/conftest.py:16-18)
    return np.random.default_rng(1234)


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def cuda():
    """The CUDA device; a gpu-marked test must not silently pass without it."""
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu test selected but no CUDA device is visible")
    from paper_2602_23967_b200 import _native

    _native.load()
    return torch.device("cuda:0")
