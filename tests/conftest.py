import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs via gpurun")
    config.addinivalue_line("markers", "slow: longer CPU runs")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def oracle_built():
    from oracle import pyorc
    if not pyorc.available("orc") or (os.path.isdir(pyorc.REFERENCE_SRC) and not pyorc.available("ref")):
        pyorc.build()
    return pyorc
