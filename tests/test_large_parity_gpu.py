"""GPU parity at the largest configurations (VERDICT r1 "what's weak" 1):
single traces of every synthetic family at 10^5 and uniform / cnn at 10^6,
the same traces through the batched kernels, and all 4096 LSTM profiles
with full offsets at L=6 and L=64 — every one bit-exact against the
REFERENCE's own plans (sha256 digests in tests/golden/huge*.json, generated
from memplan.solve_bestfit by tests/golden/make_huge_golden.py)."""
import os

import numpy as np
import pytest

import oracle
from conftest import family_instance, lstm_instances, sha64

pytestmark = pytest.mark.gpu

SINGLE = ["uniform_1e5_s0", "cnn_1e5_s0", "walk_1e5_s0", "uniform_1e5_s1", "walk_1e5_s1",
          "uniform_1e6_s0", "cnn_1e6_s0", "walk_1e6_s0"]


@pytest.mark.parametrize("name", SINGLE)
def test_single_trace_matches_reference(huge_golden, name):
    from paper_1804_10001_b200.bestfit import solve_bestfit_arrays
    if name not in huge_golden:
        pytest.skip(f"{name}: reference digest not generated")
    a, f, s = family_instance(name)
    g = huge_golden[name]
    assert sha64(np.stack([s, a, f], 1)) == g["blocks_sha256"]
    off, peak = solve_bestfit_arrays(a, f, s)
    assert peak == g["peak"], (peak, g["peak"])
    assert sha64(off) == g["offsets_sha256"]


def test_1e5_families_batched_match_reference(huge_golden, monkeypatch):
    """The five 10^5 traces as one batch, through the general batched path
    and the register-capped batched kernel (MEMPLAN_OCC=1)."""
    from paper_1804_10001_b200.bestfit import solve_bestfit_batched_arrays
    names = [n for n in SINGLE if "1e5" in n]
    cols = [family_instance(n) for n in names]
    tp = np.zeros(len(cols) + 1, np.int64)
    np.cumsum([len(c[0]) for c in cols], out=tp[1:])
    A, F, S = (np.concatenate([c[i] for c in cols]) for i in range(3))
    for occ in ("0", "1"):
        monkeypatch.setenv("MEMPLAN_OCC", occ)
        off, pks = solve_bestfit_batched_arrays(tp, A, F, S)
        for t, n in enumerate(names):
            g = huge_golden[n]
            assert pks[t] == g["peak"], (occ, n)
            assert sha64(off[tp[t]:tp[t + 1]]) == g["offsets_sha256"], (occ, n)


@pytest.mark.parametrize("layers", [6, 64])
def test_lstm_all_profiles_full_offsets(huge_golden, layers):
    """configs[3]: all 4096 profiles batched, every offset against the C
    oracle and the whole batch against the reference digest."""
    from paper_1804_10001_b200.bestfit import solve_bestfit_batched_arrays
    tp, a, f, s = lstm_instances(layers)
    off, pks = solve_bestfit_batched_arrays(tp, a, f, s)
    g = huge_golden[f"lstm_L{layers}_a512"]
    assert sha64(off) == g["offsets_sha256"]
    assert sha64(pks) == g["peaks_sha256"]
    for t in range(len(tp) - 1):
        o, p = oracle.solve_bestfit(a[tp[t]:tp[t + 1]], f[tp[t]:tp[t + 1]], s[tp[t]:tp[t + 1]])
        assert p == pks[t] and np.array_equal(o, off[tp[t]:tp[t + 1]]), t


@pytest.mark.parametrize("name", ["uniform_1e5_s0", "cnn_1e5_s0", "walk_1e5_s1"])
def test_cluster_tier_engaged_and_exact(huge_golden, name, monkeypatch):
    """A 10^5-block single trace runs on the cluster tier (the planner CTA
    plus worker CTAs serving the table over DSMEM, staged by bulk copies);
    the same trace with the tier disabled (L2 table) gives the same plan."""
    from paper_1804_10001_b200.bestfit import plan_info, solve_bestfit_arrays
    a, f, s = family_instance(name)
    g = huge_golden[name]
    monkeypatch.setenv("MEMPLAN_CLUSTER", "1")
    off, peak = solve_bestfit_arrays(a, f, s)
    info = plan_info()
    assert info["engine"] & 1024 and info["cluster"] > 1, info
    assert peak == g["peak"] and sha64(off) == g["offsets_sha256"]
    monkeypatch.delenv("MEMPLAN_CLUSTER")
    off2, peak2 = solve_bestfit_arrays(a, f, s)
    assert not plan_info()["engine"] & 1024
    assert peak2 == peak and np.array_equal(off2, off)


def test_cluster_tier_random_vs_oracle(monkeypatch):
    """Mid-size single traces (skeletons fit one SM, the table does not) on
    the cluster tier against the C oracle, several seeds and shapes."""
    from paper_1804_10001_b200.bestfit import plan_info, solve_bestfit_arrays
    monkeypatch.setenv("MEMPLAN_CLUSTER", "1")
    rng = np.random.default_rng(5)
    for trial in range(4):
        n = int(rng.integers(30000, 60000))
        T = int(rng.integers(n // 4, 3 * n))
        a = rng.integers(0, T - 1, n)
        f = a + 1 + (rng.integers(0, T, n) % (T - a))
        s = rng.integers(1, 1 << 16, n) * 512
        off, peak = solve_bestfit_arrays(a, f, s)
        info = plan_info()
        ooff, opeak = oracle.solve_bestfit(a, f, s)
        assert peak == opeak and np.array_equal(off, ooff), (trial, info)
