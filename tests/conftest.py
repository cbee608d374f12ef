import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def gpu_available():
    try:
        import ctypes
        ctypes.CDLL("libcuda.so.1")
    except OSError:
        return False
    return True


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as o
    o.build()
    return o
