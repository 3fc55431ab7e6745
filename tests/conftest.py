import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a); parity tests proper")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def gio():
    from oracle import gio as g
    g.build()
    return g


def cuda_ok() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def gi():
    """The product binding (CUDA path).  Fails loudly if the extension is missing."""
    if not cuda_ok():
        pytest.fail("gpu test selected but no CUDA device is visible")
    from paper_2403_08551_b200 import gi as g
    g.load()
    return g
