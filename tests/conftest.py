import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLD = os.path.join(ROOT, "tests", "golden")
DATA = os.path.join(ROOT, "data")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def golden(name):
    return np.load(os.path.join(GOLD, name), allow_pickle=False)


def rel_errs(a, b, nd):
    """Max-norm error per density normalised by max |ref| (test_fmm.py:41-48)."""
    errs = []
    for l in range(nd):
        scale = np.abs(b[l]).max() if np.size(b[l]) else 0.0
        diff = np.abs(a[l] - b[l]).max() if np.size(b[l]) else 0.0
        errs.append(diff / scale if scale > 0 else diff)
    return max(errs)


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2111_10743_b200 import _lib, _build
    _build.build(verbose=False)
    _lib.load()
    return torch
