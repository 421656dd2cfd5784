"""pytest configuration: the `gpu` marker and shared fixtures.

`-m "not gpu"` runs here (no GPU): oracle vs golden vectors, host logic, C-ABI load/exports.
`-m gpu` runs on a B200 via gpurun: parity of the CUDA path against the oracle.
"""
from __future__ import annotations

import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through gpurun)")


@pytest.fixture(scope="session")
def oracle():
    import vxoracle as o  # oracle/vxoracle.py (test infrastructure)
    o.build()
    return o


@pytest.fixture(scope="session")
def vxlib():
    from paper_2511_02062_b200 import build
    build.build()
    from paper_2511_02062_b200 import _lib
    return _lib.load()


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    def load(name):
        return dict(np.load(ROOT / "tests" / "golden" / f"{name}.npz"))
    return load
