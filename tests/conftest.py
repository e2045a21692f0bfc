"""Shared pytest configuration.

`-m gpu` tests need a B200 (run through gpurun); everything else runs on CPU.
The oracle (oracle/) is test infrastructure and is importable from tests only.
"""

from __future__ import annotations

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device; run under gpurun")
    config.addinivalue_line("markers", "slow: long-running")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    gdir = os.path.join(ROOT, "tests", "golden")
    return {name: np.load(os.path.join(gdir, f"{name}.npz")) for name in ("codec", "quantize", "linear")}
