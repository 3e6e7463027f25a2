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


def tree_nodes(store, name):
    """(dims, parent, left, right) node tuples of a golden tree (dims rebuilt from the leaves)."""
    arr = store[f"{name}_tree"]
    leafdim = store[f"{name}_dims"]
    n = len(arr)
    dims = [None] * n

    def walk(i):
        p, lf, rt = (int(x) for x in arr[i])
        if lf < 0:
            dims[i] = (int(leafdim[i]),)
        else:
            dims[i] = walk(lf) + walk(rt)
        return dims[i]

    walk(0)
    return [(dims[i], int(arr[i][0]), int(arr[i][1]), int(arr[i][2])) for i in range(n)]
