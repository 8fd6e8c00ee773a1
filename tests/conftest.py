"""Test configuration.

Markers:
  gpu  -- needs a CUDA device (B200); run with ``pytest -m gpu``.
Everything unmarked runs on a CPU-only box (``pytest -m "not gpu"``).
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: multi-second CPU test")


@pytest.fixture(scope="session")
def has_gpu():
    import torch
    return torch.cuda.is_available()
