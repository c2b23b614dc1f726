"""Shared test setup. `-m gpu` tests need a CUDA device; everything else runs on CPU."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")


@pytest.fixture(scope="session")
def ref():
    from oracle import ref as r
    if not r.available():
        pytest.skip("oracle/_ref not built (make -C oracle)")
    return r


@pytest.fixture(scope="session")
def mg():
    import paper_2408_03204_b200 as m
    return m


def cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
