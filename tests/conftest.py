"""Shared test configuration.

`-m gpu` tests need a B200 and the in-tree CUDA library; everything else runs
on the CPU build container (oracle vs golden vectors, host logic, C-ABI
exports, gloo world-size-2 sharding logic).
"""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built sm_100a library")


def load_golden(name: str):
    return np.load(GOLDEN / f"{name}.npz", allow_pickle=False)


def unpack_occ(bits, dims):
    n = int(np.prod(dims))
    return np.unpackbits(bits)[:n].astype(bool).reshape(tuple(int(d) for d in dims))


def i32_to_sq(a):
    a = np.asarray(a)
    return np.where(a < 0, np.inf, a.astype(np.float64))


@pytest.fixture(scope="session")
def golden():
    return load_golden
