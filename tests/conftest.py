import gzip
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def load_json(name):
    path = os.path.join(GOLDEN, name)
    opener = gzip.open if name.endswith(".gz") else open
    with opener(path, "rt") as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def small_plans():
    return load_json("plans_small.json.gz")


@pytest.fixture(scope="session")
def large_plans():
    return dict(np.load(os.path.join(GOLDEN, "plans_large.npz")))


@pytest.fixture(scope="session")
def verify_golden():
    return load_json("verify.json.gz")


@pytest.fixture(scope="session")
def arena_golden():
    return load_json("arena.json.gz")


@pytest.fixture(scope="session")
def trace_golden():
    return load_json("traces.json")


@pytest.fixture(scope="session")
def profile_golden():
    return load_json("profiles.json")


def blocks_arrays(blocks):
    if len(blocks) == 0:
        z = np.zeros(0, np.int64)
        return z, z, z
    b = np.asarray(blocks, dtype=np.int64)
    return b[:, 1].copy(), b[:, 2].copy(), b[:, 0].copy()  # alloc, free, size
