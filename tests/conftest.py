"""Test configuration: `-m gpu` tests need a B200 (run through gpurun); the
rest run on the CPU and cover the oracle (against the reference's own known
answers), the host logic and the C-ABI surface."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run via gpurun")


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build()
    return oracle


@pytest.fixture(scope="session")
def fb():
    """The product package; its CUDA library must be built (no fallback)."""
    import paper_1810_06825_b200 as P
    from paper_1810_06825_b200 import _lib
    _lib.load()
    return P


@pytest.fixture(scope="session")
def ctx(fb):
    return fb.default_context()
