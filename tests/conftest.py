import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI library)")
    config.addinivalue_line("markers", "slow: long validation runs")


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)


def load_golden(name):
    return dict(np.load(GOLDEN / f"{name}.npz"))


def unpack_cp(store, prefix):
    d = int(store[f"{prefix}_d"])
    return [store[f"{prefix}_{k}"] for k in range(d)]


def unpack_ht(store, prefix, nodes):
    frames = [store.get(f"{prefix}_F{i}") for i in range(len(nodes))]
    transfers = [store.get(f"{prefix}_B{i}") for i in range(len(nodes))]
    return frames, transfers
