"""Shared pytest setup.

Markers: `gpu` -- needs a CUDA device (run on the B200 box with `-m gpu`).
Everything unmarked runs on the CPU-only build container.
"""

import os
import sys

import pytest

# before any CUDA context: multi-engine peer tests use two streams per engine
# (see paper_1405_6162_b200/__init__.py)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: test needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def golden():
    import json

    import numpy as np

    here = os.path.join(ROOT, "tests", "golden")
    with open(os.path.join(here, "reference_golden.json")) as fh:
        meta = json.load(fh)
    small = dict(np.load(os.path.join(here, "reference_small.npz")))
    return meta, small


def gpu_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
