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


@pytest.fixture(scope="session")
def huge_golden():
    """Reference digests at 10^5 / 10^6 and for the 4096 LSTM profiles
    (tests/golden/make_huge_golden.py, generated from the reference)."""
    out = {}
    for name in ("huge.json", "huge_lstm.json"):
        with open(os.path.join(GOLDEN, name)) as fh:
            out.update({c["name"]: c for c in json.load(fh)["cases"]})
    return out


def sha64(a) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


def family_instance(name: str):
    """(alloc, free, size) of a huge.json case ("uniform_1e5_s0", ...) built
    with the product's own generators and ingest (alignment 512)."""
    import paper_1804_10001_b200 as mp
    from paper_1804_10001_b200.profiler import ingest_arrays
    from paper_1804_10001_b200.workloads import uniform_blocks, walk_trace
    fam, n, seed = name.split("_")
    n, seed = int(float(n)), int(seed[1:])
    if fam == "uniform":
        b = np.asarray(uniform_blocks(n, seed), np.int64)
        s = ((b[:, 0] + 511) // 512) * 512
        return b[:, 1].copy(), b[:, 2].copy(), s
    if fam == "cnn":
        txt = mp.cnn_like_trace(mp.GenSpec(model="cnn", layers=n // 2, seed=seed))
    else:
        txt = walk_trace(n, seed)
    return ingest_arrays(txt, alignment=512)[:3]


def lstm_instances(layers: int, alignment: int = 512):
    """The 4096 LSTM profiles of BASELINE.json configs[3] as CSR columns."""
    from paper_1804_10001_b200.profiler import ingest_arrays
    from paper_1804_10001_b200.workloads import lstm_profiles
    cols = [ingest_arrays(t, alignment=alignment)[:3]
            for t in lstm_profiles(4096, layers=layers)]
    tp = np.zeros(len(cols) + 1, np.int64)
    np.cumsum([len(c[0]) for c in cols], out=tp[1:])
    return tp, *(np.concatenate([c[i] for c in cols]) for i in range(3))
