import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA) device; run on the GPU box")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session", autouse=True)
def _build_cpu_libs():
    import gen
    import oracle
    gen.build()
    oracle.build()
    yield


def cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
