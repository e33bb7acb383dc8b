import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200) and the built libnid.so")
    config.addinivalue_line("markers", "slow: long-running parity case")


def golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def _has_cuda_device():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture(scope="session")
def nid():
    """The loaded CUDA library.  On a machine with a GPU a missing or
    broken library is a failure, never a silent fallback."""
    from paper_1804_03807_b200 import _lib

    if not _has_cuda_device():
        pytest.skip("no CUDA device")
    return _lib.lib()
