"""Pin the CPU oracle against golden vectors produced by the reference
(tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest

import oracle
from conftest import blocks_arrays


def test_oracle_matches_reference_small(small_plans):
    for case in small_plans:
        a, f, s = blocks_arrays(case["blocks"])
        off, peak = oracle.solve_bestfit(a, f, s)
        assert peak == case["peak"], case["name"]
        assert off.tolist() == case["offsets"], case["name"]
        assert oracle.clique_lb(a, f, s) == case["clique_lb"], case["name"]


def test_oracle_pinned_constants(small_plans):
    by = {c["name"]: c for c in small_plans}
    assert by["worked"]["offsets"] == [2, 0, 2] and by["worked"]["peak"] == 6
    assert by["G1_size_tiebreak"]["offsets"] == [2, 0]
    assert by["G2_size_tiebreak"]["peak"] == 7
    assert by["cnn20_seed42"]["peak"] == 500448
    assert by["cnn20_seed42"]["pool_peak"] == 704864
    assert by["rnn6_maxlen"]["peak"] == 107744
    assert by["G3_staircase"]["peak"] == 2000


@pytest.mark.parametrize("name", ["cnn_1e4", "uniform_1e4", "walk_1e4"])
def test_oracle_matches_reference_large(large_plans, name):
    b = large_plans[name + "_blocks"]
    off, peak, st = oracle.solve_bestfit(b[:, 1], b[:, 2], b[:, 0], with_stats=True)
    assert peak == int(large_plans[name + "_peak"][0])
    assert np.array_equal(off, large_plans[name + "_offsets"])
    assert st["steps"] <= 3 * len(b) + 4


def test_oracle_verify_matches_reference(verify_golden):
    for case in verify_golden:
        a, f, s = blocks_arrays(case["blocks"])
        r = oracle.verify(a, f, s, case["offsets"])
        assert r["peak_recomputed"] == case["peak_recomputed"]
        assert [list(v) for v in r["violations"]] == case["violations"]
        valid = r["n_violations"] == 0 and r["offsets_ok"] and r["peak_recomputed"] == case["peak"]
        assert valid == case["valid"]
        t_lo, t_hi = (int(a.min()), int(f.max())) if len(a) else (0, 0)
        span, pk = t_hi - t_lo, r["peak_recomputed"]
        util = r["used"] / (pk * span) if pk > 0 and span > 0 else 0.0
        assert repr(util) == case["utilization"]


def test_numpy_port_matches_reference(small_plans, large_plans):
    from oracle.bestfit_np import solve_bestfit_np
    for case in small_plans[:400]:
        a, f, s = blocks_arrays(case["blocks"])
        off, peak = solve_bestfit_np(a, f, s)
        assert peak == case["peak"] and off.tolist() == case["offsets"], case["name"]
    b = large_plans["walk_1e4_blocks"]
    off, peak = solve_bestfit_np(b[:, 1], b[:, 2], b[:, 0])
    assert np.array_equal(off, large_plans["walk_1e4_offsets"])
