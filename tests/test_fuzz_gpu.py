"""Randomised parity sweep across every planner path: mixed batches whose
traces land on the fused small-trace kernel (TIER_TINY, with its TIER_SCAN
restart), single traces on k_tiny / TIER_ALL / TIER_SKEL, batches on the
general and register-capped kernels, 64-bit heights, tie-heavy and
staircase shapes — all against the C oracle (itself pinned to the
reference's golden vectors and digests)."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _trace(rng, n, kind):
    if kind == "uniform":
        a = rng.integers(0, 2 * n, n)
        f = a + 1 + rng.integers(0, 2 * n, n) % (2 * n - a)
        s = rng.integers(1, 1 << 20, n)
    elif kind == "narrow":  # many equal lifetimes / sizes (tie-breaks)
        a = rng.integers(0, max(2, n // 8), n)
        f = a + rng.integers(1, 4, n)
        s = rng.choice([512, 1024, 2048], n)
    elif kind == "stair":  # long skylines
        a = np.arange(n) * 2
        f = a + 1 + rng.integers(0, 3, n)
        s = rng.integers(1, 64, n)
    elif kind == "big":  # 64-bit heights
        a = rng.integers(0, 4 * n, n)
        f = a + 1 + rng.integers(0, 4 * n, n)
        s = rng.integers(1, 1 << 40, n)
    else:  # nested, cnn-like
        a = np.sort(rng.integers(0, n, n))
        f = (2 * n - a) + rng.integers(0, 3, n)
        s = rng.integers(1, 1 << 16, n) * 512
    return a.astype(np.int64), f.astype(np.int64), s.astype(np.int64)


KINDS = ["uniform", "narrow", "stair", "big", "nested"]


def test_fuzz_single_traces():
    from paper_1804_10001_b200.bestfit import solve_bestfit_arrays
    rng = np.random.default_rng(2026)
    for trial in range(250):
        kind = KINDS[trial % len(KINDS)]
        n = int(rng.choice([1, 2, 7, 31, 64, 129, 500, 2048, 2049, 4096, 4097, 9000]))
        a, f, s = _trace(rng, n, kind)
        off, pk = solve_bestfit_arrays(a, f, s)
        ooff, opk = oracle.solve_bestfit(a, f, s)
        assert pk == opk and np.array_equal(off, ooff), (trial, kind, n)


@pytest.mark.parametrize("mix", ["small", "mixed", "many"])
def test_fuzz_batches(mix):
    from paper_1804_10001_b200.bestfit import solve_bestfit_batched_arrays
    rng = np.random.default_rng({"small": 1, "mixed": 2, "many": 3}[mix])
    if mix == "small":
        sizes = rng.integers(0, 130, 400)
    elif mix == "mixed":
        sizes = rng.choice([0, 5, 100, 700, 2048, 3000, 6000], 60)
    else:
        sizes = rng.integers(1, 1500, 320)
    cols = [_trace(rng, int(n), KINDS[i % len(KINDS)]) if n else (np.zeros(0, np.int64),) * 3
            for i, n in enumerate(sizes)]
    tp = np.zeros(len(cols) + 1, np.int64)
    np.cumsum([len(c[0]) for c in cols], out=tp[1:])
    A, F, S = (np.concatenate([c[i] for c in cols]) for i in range(3))
    off, pks = solve_bestfit_batched_arrays(tp, A, F, S)
    for t, (a, f, s) in enumerate(cols):
        ooff, opk = oracle.solve_bestfit(a, f, s)
        assert pks[t] == opk and np.array_equal(off[tp[t]:tp[t + 1]], ooff), (mix, t, len(a))


def test_fuzz_tiny_tall_heights():
    """Single traces on k_tiny whose heights pass 2^27 units (unpacked
    choose keys: heights relative to the last chosen one, with the
    saturated fallback when the lowest line jumps by >= 2^27) and windows
    long enough for the block-summary query."""
    from paper_1804_10001_b200.bestfit import plan_info, solve_bestfit_arrays
    rng = np.random.default_rng(77)
    tiny = 0
    for trial in range(40):
        n = int(rng.choice([40, 300, 1500, 4000]))
        a, f, _ = _trace(rng, n, KINDS[trial % len(KINDS)] if trial % 5 != 3 else "uniform")
        s = rng.integers(1, 100, n)
        tall = rng.choice(n, size=min(n, 12), replace=False)
        s[tall] = (1 << 28) + rng.integers(0, 1 << 20, len(tall))
        s = s.astype(np.int64)
        off, pk = solve_bestfit_arrays(a, f, s)
        tiny += bool(plan_info()["engine"] & 512)  # TIER_TINY ran
        ooff, opk = oracle.solve_bestfit(a, f, s)
        assert pk == opk and np.array_equal(off, ooff), (trial, n)
    assert tiny >= 20, tiny
