import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the CUDA extension")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def cuda_lib():
    """The built C-ABI library on a GPU box; fails loudly when it is missing."""
    import torch

    if not torch.cuda.is_available():
        pytest.fail("-m gpu test run without a visible CUDA device")
    from paper_2306_09784_b200 import sar

    sar.load()
    return sar
