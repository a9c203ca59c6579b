import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU and the built CUDA library")


@pytest.fixture(scope="session")
def cuda():
    """The CUDA path must be present on a GPU test run: fail (never skip) otherwise."""
    import torch

    from paper_2601_21444_b200 import spava

    assert torch.cuda.is_available(), "gpu test without a visible CUDA device"
    assert spava.device_ok(), "libspava_b200.so sees no sm_100 device"
    return torch.device("cuda:0")
