"""Shared test setup.

Markers: ``gpu`` — needs a CUDA device (run on the B200 box with -m gpu).
Everything unmarked runs on CPU: the oracle against the reference's golden
vectors, host-side logic, and the C-ABI library's exports.
"""

import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def golden_small():
    return dict(np.load(GOLDEN / "ref_small.npz"))


@pytest.fixture(scope="session")
def golden_large():
    path = GOLDEN / "ref_large.npz"
    if not path.exists():
        pytest.fail("tests/golden/ref_large.npz missing (run tests/golden/make_golden.py)")
    return dict(np.load(path))


@pytest.fixture(scope="session")
def small_cases():
    from tests.golden import cases

    return cases.small_cases()


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu test collected on a host without CUDA (run with -m 'not gpu')")
    import paper_1707_06468_b200._lib as L

    L.load()
    return torch.device("cuda", 0)
