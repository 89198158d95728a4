import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) GPU; runs through the C-ABI")
    config.addinivalue_line("markers", "slow: longer parity runs")


@pytest.fixture(scope="session")
def ctx():
    import torch
    from paper_2210_08803_b200 import Context
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    return Context(0)
