"""C++ host ingest (mp_ingest_trace) == parse_trace -> record ->
profile_to_instance (profiler.py:97-231, core.py:184-224).  CPU only: the
ingest is host code in libmemplan_b200.so."""
import random
import time

import numpy as np
import pytest

import paper_1804_10001_b200 as mp


def _python_path(text, alignment):
    prof = mp.record(mp.parse_trace(text))
    inst = mp.profile_to_instance(prof, alignment=alignment)
    a, f, s = inst.arrays()
    return a, f, s, prof.unmanaged_count, prof.horizon


def _same(text, alignment=1):
    got = mp.ingest_arrays(text, alignment)
    ref = _python_path(text, alignment)
    for g, r in zip(got[:3], ref[:3]):
        assert np.array_equal(g, r)
    assert got[3:] == ref[3:]


def test_golden_profiles(profile_golden):
    for case in profile_golden:
        a, f, s, unmanaged, horizon = mp.ingest_arrays(case["text"])
        got = [[i + 1, int(s[i]), int(a[i]), int(f[i])] for i in range(len(a))]
        assert got == [m[:4] for m in case["managed"]]
        assert unmanaged == case["unmanaged_count"] and horizon == case["horizon"]


@pytest.mark.parametrize("alignment", [1, 8, 512])
def test_generators(alignment):
    texts = [mp.cnn_like_trace(mp.GenSpec(model="cnn", layers=L, seed=s))
             for L, s in ((1, 0), (20, 42), (300, 7))]
    spec = mp.GenSpec(model="rnn", layers=6, batch=16, seed=2024, variable_length=(10, 50))
    texts += [mp.rnn_like_trace(spec, ell) for ell in mp.rnn_epoch_lengths(spec, 5)]
    texts += [mp.net_trace("googlenet", 64)]
    from paper_1804_10001_b200.workloads import walk_trace
    texts += [walk_trace(2000, seed=3)]
    for t in texts:
        _same(t, alignment)


def test_random_traces_with_interrupts_zero_sizes_and_noise():
    rng = random.Random(11)
    for trial in range(200):
        lines, n_alloc, live, depth = [], 0, [], 0
        for _ in range(rng.randint(0, 60)):
            r = rng.random()
            if r < 0.45:
                size = rng.choice([0, rng.randint(1, 5000)])
                lab = rng.choice(["", " conv1", "\tx y  z"])
                lines.append(f"{rng.choice(['', '  '])}A {size}{lab}")
                n_alloc += 1
                live.append(n_alloc)
            elif r < 0.75 and live:
                lines.append(f"F {live.pop(rng.randrange(len(live)))}")
            elif r < 0.82:
                lines.append("I")
                depth += 1
            elif r < 0.88 and depth:
                lines.append("R")
                depth -= 1
            elif r < 0.94:
                lines.append(rng.choice(["# comment", "", "   ", "#"]))
            else:
                lines.append(f"A {rng.randint(1, 9)}_{rng.randint(0, 9)}")
                n_alloc += 1
                live.append(n_alloc)
        sep = rng.choice(["\n", "\r\n", "\r"])
        text = sep.join(lines) + rng.choice(["", sep])
        _same(text, rng.choice([1, 4, 512]))


ERRORS = [
    "A 4\nX 1\n", "A\n", "A 1\nA 2\nF x\n", "F 0\n", "I now\n", "R x\n", "F 1 2\n", "A -3\n",
    "A 1x\n", "A 1__0\n", "A _1\n", "A 1_\n", "AA 3\n", "a 3\n", "F\n",
    "F 1\n", "A 3\nF 1\nF 1\n", "R\n", "A 3\nF 2\n",
    # syntax errors take precedence over earlier recording errors
    "F 5\nA 1\nQ\n", "R\nA 2 x\nA\n",
    # recording errors: the first in event order wins
    "A 1\nF 1\nF 1\nF 9\n", "A 1\nF 3\nF 1\nF 1\n",
]


@pytest.mark.parametrize("text", ERRORS)
def test_errors_match_python_path(text):
    with pytest.raises(mp.MemplanError) as ref:
        _python_path(text, 1)
    with pytest.raises(mp.MemplanError) as got:
        mp.ingest_arrays(text, 1)
    assert type(got.value) is type(ref.value)
    assert str(got.value) == str(ref.value)
    assert getattr(got.value, "line_no", None) == getattr(ref.value, "line_no", None)


def test_fallbacks_stay_exact():
    _same("A 3 café\nA 4\nF 1\n", 1)  # non-ASCII label
    _same("A 0007\nA +5\nF 2\n", 1)
    with pytest.raises(ValueError):
        mp.ingest_arrays("A 99999999999999999999999\n", 1)


def test_faster_than_python_at_scale():
    text = mp.cnn_like_trace(mp.GenSpec(model="cnn", layers=25000, seed=0))  # 10^5 events
    t0 = time.perf_counter()
    got = mp.ingest_arrays(text, 512)
    t1 = time.perf_counter()
    ref = _python_path(text, 512)
    t2 = time.perf_counter()
    assert all(np.array_equal(g, r) for g, r in zip(got[:3], ref[:3]))
    assert (t1 - t0) * 5 < (t2 - t1), (t1 - t0, t2 - t1)
