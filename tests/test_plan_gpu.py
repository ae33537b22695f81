"""GPU planner parity against the reference golden vectors and the oracle."""
import numpy as np
import pytest

import oracle
from conftest import blocks_arrays

pytestmark = pytest.mark.gpu


def test_small_golden(small_plans):
    from paper_1804_10001_b200.bestfit import solve_bestfit_arrays
    for case in small_plans:
        a, f, s = blocks_arrays(case["blocks"])
        off, peak = solve_bestfit_arrays(a, f, s)
        assert peak == case["peak"], case["name"]
        assert off.tolist() == case["offsets"], case["name"]


@pytest.mark.parametrize("name", ["cnn_1e4", "uniform_1e4", "walk_1e4"])
def test_large_golden(large_plans, name):
    from paper_1804_10001_b200.bestfit import solve_bestfit_arrays, plan_info
    b = large_plans[name + "_blocks"]
    for flags in (0, 4):
        off, peak = solve_bestfit_arrays(b[:, 1], b[:, 2], b[:, 0], flags=flags)
        assert peak == int(large_plans[name + "_peak"][0])
        assert np.array_equal(off, large_plans[name + "_offsets"])
        print(name, flags, plan_info())


def test_batched_golden(small_plans):
    from paper_1804_10001_b200.bestfit import solve_bestfit_batched_arrays
    cases = small_plans
    sizes = [len(c["blocks"]) for c in cases]
    tp = np.zeros(len(cases) + 1, np.int64)
    np.cumsum(sizes, out=tp[1:])
    cols = [blocks_arrays(c["blocks"]) for c in cases]
    a = np.concatenate([c[0] for c in cols]); f = np.concatenate([c[1] for c in cols])
    s = np.concatenate([c[2] for c in cols])
    off, peaks = solve_bestfit_batched_arrays(tp, a, f, s)
    for t, c in enumerate(cases):
        assert peaks[t] == c["peak"], c["name"]
        assert off[tp[t]:tp[t + 1]].tolist() == c["offsets"], c["name"]


def test_random_vs_oracle():
    from paper_1804_10001_b200.bestfit import solve_bestfit_arrays
    rng = np.random.default_rng(0)
    for trial in range(60):
        n = int(rng.integers(1, 3000))
        T = int(rng.integers(2, 4 * n + 3))
        a = rng.integers(0, T - 1, n)
        f = a + 1 + (rng.integers(0, T, n) % (T - a))
        s = rng.integers(1, 1 << int(rng.integers(1, 40)), n)
        off, peak = solve_bestfit_arrays(a, f, s)
        ooff, opeak = oracle.solve_bestfit(a, f, s)
        assert peak == opeak and np.array_equal(off, ooff), trial


def test_line_overflow_restart():
    """A staircase of 3000 disjoint blocks needs 5999 skyline lines, more than
    the shared-memory line capacity: the planner must restart it with global
    line storage and still match the oracle."""
    from paper_1804_10001_b200.bestfit import solve_bestfit_arrays, plan_info
    k = np.arange(3000, dtype=np.int64)
    a, f, s = 2 * k, 2 * k + 1, k + 1
    off, peak = solve_bestfit_arrays(a, f, s)
    ooff, opeak = oracle.solve_bestfit(a, f, s)
    assert peak == opeak == 3000 and np.array_equal(off, ooff)
    assert plan_info()["engine"] & 32  # restarted with global lines


def test_wide_heights_64bit():
    """Total bytes above 2^32 units select the 64-bit height engine."""
    from paper_1804_10001_b200.bestfit import solve_bestfit_arrays, plan_info
    rng = np.random.default_rng(5)
    n = 500
    a = rng.integers(0, 900, n)
    f = a + 1 + rng.integers(0, 100, n)
    s = rng.integers(1, 1 << 40, n) * 3 + 1
    off, peak = solve_bestfit_arrays(a, f, s)
    ooff, opeak = oracle.solve_bestfit(a, f, s)
    assert peak == opeak and np.array_equal(off, ooff)
    assert not (plan_info()["engine"] & 16)


def test_huge_time_span_disables_lifetime_pruning():
    """Raw times spread over 2^40 ticks: the planner's lifetime bounds (31-bit
    relative times) switch off and the result must still be bit-exact."""
    from paper_1804_10001_b200.bestfit import solve_bestfit_arrays
    rng = np.random.default_rng(9)
    n = 4000
    a = rng.integers(0, 1 << 40, n)
    f = a + 1 + rng.integers(0, 1 << 38, n)
    s = rng.integers(1, 1 << 20, n)
    off, peak = solve_bestfit_arrays(a, f, s)
    ooff, opeak = oracle.solve_bestfit(a, f, s)
    assert peak == opeak and np.array_equal(off, ooff)


@pytest.mark.parametrize("flags", [0, 4])
def test_edge_shapes(flags):
    """Degenerate shapes: one block, identical blocks, nested, all disjoint,
    a single long-lived block over many short ones."""
    from paper_1804_10001_b200.bestfit import solve_bestfit_arrays
    cases = [
        ([0], [1], [7]),
        ([0] * 50, [10] * 50, [3] * 50),
        (list(range(40)), [80 - i for i in range(40)], [i + 1 for i in range(40)]),
        ([2 * i for i in range(300)], [2 * i + 1 for i in range(300)], [5] * 300),
        ([0] + list(range(1, 600)), [1000] + list(range(2, 601)), [1 << 30] + [1] * 599),
    ]
    for a, f, s in cases:
        a, f, s = (np.asarray(x, np.int64) for x in (a, f, s))
        off, peak = solve_bestfit_arrays(a, f, s, flags=flags)
        ooff, opeak = oracle.solve_bestfit(a, f, s)
        assert peak == opeak and np.array_equal(off, ooff)


def test_large_batch_mixed_sizes():
    """A batch mixing tiny, medium and 3*10^4-block traces (several layout
    tiers in one launch) against the oracle."""
    from paper_1804_10001_b200.bestfit import solve_bestfit_batched_arrays
    from paper_1804_10001_b200.workloads import uniform_arrays
    sizes = [0, 1, 13, 129, 2000, 30000, 7, 5000]
    cols = []
    for i, n in enumerate(sizes):
        a, f, s = uniform_arrays(n, 100 + i) if n else (np.zeros(0, np.int64),) * 3
        cols.append((a, f, ((s + 511) // 512) * 512))
    tp = np.zeros(len(cols) + 1, np.int64)
    np.cumsum([len(c[0]) for c in cols], out=tp[1:])
    A = np.concatenate([c[0] for c in cols]); F = np.concatenate([c[1] for c in cols])
    S = np.concatenate([c[2] for c in cols])
    off, peaks = solve_bestfit_batched_arrays(tp, A, F, S)
    for t, (a, f, s) in enumerate(cols):
        ooff, opeak = oracle.solve_bestfit(a, f, s)
        assert peaks[t] == opeak and np.array_equal(off[tp[t]:tp[t + 1]], ooff), t


@pytest.mark.parametrize("nwarps", ["1", "8"])
@pytest.mark.parametrize("tier", ["0", "1", "2", "3", "4"])
def test_every_layout_tier_and_warp_count(monkeypatch, nwarps, tier):
    """The planner's shared-memory tiers (0 global, 1 group skeleton, 2 +chunk
    skeleton, 3 +table) and the 8-warp variant give identical plans."""
    from paper_1804_10001_b200.bestfit import solve_bestfit_arrays, solve_bestfit_batched_arrays
    from paper_1804_10001_b200.workloads import uniform_arrays
    import paper_1804_10001_b200 as mp
    monkeypatch.setenv("MEMPLAN_NWARPS", nwarps)
    monkeypatch.setenv("MEMPLAN_TIER", tier)
    a, f, s = uniform_arrays(6000, 4)
    s = ((s + 511) // 512) * 512
    c = mp.profile_to_instance(mp.record(mp.parse_trace(mp.cnn_like_trace(
        mp.GenSpec(model="cnn", layers=1500, seed=2)))), alignment=512).arrays()
    for arr in ((a, f, s), c):
        off, peak = solve_bestfit_arrays(*arr)
        ooff, opeak = oracle.solve_bestfit(*arr)
        assert peak == opeak and np.array_equal(off, ooff)
    tp = np.array([0, 2000, 2001, 6000], np.int64)
    off, peaks = solve_bestfit_batched_arrays(tp, a, f, s)
    for t in range(3):
        sl = slice(tp[t], tp[t + 1])
        ooff, opeak = oracle.solve_bestfit(a[sl], f[sl], s[sl])
        assert peaks[t] == opeak and np.array_equal(off[sl], ooff)


@pytest.mark.parametrize("mode", ["raw", "dense", "wide"])
def test_large_batch_composite_key_prep(monkeypatch, mode):
    """Batches of >= 2^16 blocks take K0's composite-key sorts (one sort per
    ordering, key widths cut to the batch's ranges); with a time span below
    2^25 the raw relative times serve as ranks (no rank compression),
    otherwise (MEMPLAN_DENSE_RANKS, or a wide span) ranks are compressed.
    Every trace must match the oracle in every mode."""
    from paper_1804_10001_b200.bestfit import solve_bestfit_batched_arrays
    from paper_1804_10001_b200.workloads import uniform_arrays
    import paper_1804_10001_b200 as mp
    if mode == "dense":
        monkeypatch.setenv("MEMPLAN_DENSE_RANKS", "1")
    cols = []
    if mode == "wide":  # a far-away trace: batch span >= 2^25
        a, f, s = uniform_arrays(3000, 77)
        cols.append((a + (1 << 40), f + (1 << 40), ((s + 511) // 512) * 512))
    for i in range(6):
        a, f, s = uniform_arrays(10000 + 37 * i, 300 + i)
        cols.append((a + 1000 * i, f + 1000 * i, ((s + 511) // 512) * 512))
    cols.append(mp.profile_to_instance(mp.record(mp.parse_trace(mp.cnn_like_trace(
        mp.GenSpec(model="cnn", layers=6000, seed=5)))), alignment=512).arrays())
    cols.append(tuple(np.zeros(0, np.int64) for _ in range(3)))
    # equal raw times across traces and duplicate times inside one trace
    cols.append((np.array([5, 5, 5, 7]), np.array([9, 6, 9, 9]), np.array([512, 1024, 512, 512])))
    tp = np.zeros(len(cols) + 1, np.int64)
    np.cumsum([len(c[0]) for c in cols], out=tp[1:])
    assert tp[-1] >= 1 << 16
    A = np.concatenate([c[0] for c in cols]); F = np.concatenate([c[1] for c in cols])
    S = np.concatenate([c[2] for c in cols])
    off, peaks = solve_bestfit_batched_arrays(tp, A, F, S)
    for t, (a, f, s) in enumerate(cols):
        ooff, opeak = oracle.solve_bestfit(a, f, s)
        assert peaks[t] == opeak and np.array_equal(off[tp[t]:tp[t + 1]], ooff), t


def _batch(cols):
    tp = np.zeros(len(cols) + 1, np.int64)
    np.cumsum([len(c[0]) for c in cols], out=tp[1:])
    cat = [np.concatenate([c[k] for c in cols]) if tp[-1] else np.zeros(0, np.int64)
           for k in range(3)]
    return tp, cat


def _check_batch(cols):
    from paper_1804_10001_b200.bestfit import solve_bestfit_batched_arrays, plan_info
    tp, (A, F, S) = _batch(cols)
    off, peaks = solve_bestfit_batched_arrays(tp, A, F, S)
    info = plan_info()
    for t, (a, f, s) in enumerate(cols):
        ooff, opeak = oracle.solve_bestfit(a, f, s)
        assert peaks[t] == opeak and np.array_equal(off[tp[t]:tp[t + 1]], ooff), t
    return info


@pytest.mark.parametrize("lo,hi", [(0, 128), (100, 512), (400, 2048), (2049, 4096)])
def test_fused_small_trace_path(lo, hi):
    """Traces of <= 4096 blocks run K0 + planner in one CTA per trace (one-warp
    CTAs up to 256 blocks, 4 / 8 warps beyond; 2049-4096 blocks only while
    the batch has no more traces than SMs)."""
    from paper_1804_10001_b200.workloads import uniform_arrays
    rng = np.random.default_rng(lo)
    cols = []
    for i in range(200 if hi <= 512 else 40):
        n = int(rng.integers(lo, hi + 1))
        a, f, s = uniform_arrays(n, 1000 + i) if n else (np.zeros(0, np.int64),) * 3
        d = int(rng.integers(0, 5))
        cols.append((a + d, f + d, ((s + 511) // 512) * 512))
    info = _check_batch(cols)
    assert info["engine"] & 256, info  # the fused path ran


@pytest.mark.parametrize("tier", ["0", "1", "2", "3", "4"])
def test_register_capped_batched_kernel(monkeypatch, tier):
    """More traces than SMs (and traces too large for the fused path) select
    the 128-register batched kernel and up to 16 traces per SM; every shared
    memory tier of it must reproduce the oracle."""
    from paper_1804_10001_b200.workloads import uniform_arrays
    monkeypatch.setenv("MEMPLAN_TIER", tier)
    rng = np.random.default_rng(7)
    cols = []
    for i in range(160):
        n = int(rng.integers(2049, 2600))
        a, f, s = uniform_arrays(n, 500 + i)
        cols.append((a, f, ((s + 511) // 512) * 512))
    info = _check_batch(cols)
    assert not info["engine"] & 256


def test_concurrent_host_threads():
    """Plans issued from several host threads at once (ctypes drops the GIL)
    equal the same plans issued one after another: per-thread state and
    the serialised attribute-set + launch keep them independent."""
    import threading
    from paper_1804_10001_b200.bestfit import solve_bestfit_batched_arrays, solve_bestfit_arrays
    from paper_1804_10001_b200.workloads import uniform_arrays
    jobs = []
    for i in range(6):
        cols = []
        for k in range(3 + 60 * (i % 2)):
            n = [40, 700, 3000, 9000][(i + k) % 4]
            a, f, s = uniform_arrays(n, 50 * i + k)
            cols.append((a, f, ((s + 511) // 512) * 512))
        jobs.append(_batch(cols))
    single = [uniform_arrays(20000, 999)]
    ref = [solve_bestfit_batched_arrays(tp, *cat) for tp, cat in jobs]
    ref_single = solve_bestfit_arrays(*single[0])
    out = [None] * len(jobs)
    out_single = [None]

    def run(i):
        tp, cat = jobs[i]
        out[i] = solve_bestfit_batched_arrays(tp, *cat)

    def run_single():
        out_single[0] = solve_bestfit_arrays(*single[0])

    threads = [threading.Thread(target=run, args=(i,)) for i in range(len(jobs))]
    threads.append(threading.Thread(target=run_single))
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    for (o, p), (ro, rp) in zip(out, ref):
        assert np.array_equal(o, ro) and np.array_equal(p, rp)
    assert np.array_equal(out_single[0][0], ref_single[0]) and out_single[0][1] == ref_single[1]



def test_batches_beyond_one_pass_are_chunked(small_plans, monkeypatch):
    """A batch above the per-pass block limit (32-bit K0 ranks, device
    memory) is planned as consecutive trace ranges inside the library; the
    results equal one pass (limit lowered with MEMPLAN_MAX_BATCH_BLOCKS)."""
    from paper_1804_10001_b200.bestfit import plan_info, solve_bestfit_batched_arrays
    cases = small_plans
    tp = np.zeros(len(cases) + 1, np.int64)
    np.cumsum([len(c["blocks"]) for c in cases], out=tp[1:])
    cols = [blocks_arrays(c["blocks"]) for c in cases]
    a, f, s = (np.concatenate([c[i] for c in cols]) for i in range(3))
    one_off, one_pk = solve_bestfit_batched_arrays(tp, a, f, s)
    launches_one = plan_info()["launches"]
    monkeypatch.setenv("MEMPLAN_MAX_BATCH_BLOCKS", "3000")
    off, pk = solve_bestfit_batched_arrays(tp, a, f, s)
    assert plan_info()["launches"] > launches_one
    assert np.array_equal(off, one_off) and np.array_equal(pk, one_pk)
    for t, c in enumerate(cases):
        assert pk[t] == c["peak"] and off[tp[t]:tp[t + 1]].tolist() == c["offsets"], c["name"]
