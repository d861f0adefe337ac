import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 GPU (runs on the B200 box via gpurun)")
    config.addinivalue_line("markers", "slow: longer CPU test")


@pytest.fixture(scope="session")
def deformer():
    """Session-wide CUDA context. Builds the in-tree library if missing (nvcc is in the image)."""
    import torch

    from paper_2211_15601_b200 import build as B
    B.build()
    from paper_2211_15601_b200.deformer import Deformer
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return Deformer(0)
