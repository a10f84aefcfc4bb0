import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU and libgpmatern.so")
    config.addinivalue_line("markers", "slow: full-size config parity (minutes)")


@pytest.fixture(scope="session")
def gpm():
    """The product binding; GPU tests fail loudly if the CUDA library is missing."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test collected on a machine without CUDA")
    import paper_2508_01864_b200 as g
    g.load_library()          # raises if libgpmatern.so is absent -- no fallback
    return g
