"""GPU validator (K3) and lower bound (K4) against reference golden vectors
and the independent CPU sweep oracle."""
import numpy as np
import pytest

import oracle
import paper_1804_10001_b200 as mp
from conftest import blocks_arrays

pytestmark = pytest.mark.gpu


def test_verify_matches_reference(verify_golden):
    for case in verify_golden:
        inst = mp.build_instance([tuple(b) for b in case["blocks"]], capacity=case["capacity"])
        plan = mp.Plan(dict(enumerate(case["offsets"], start=1)), case["peak"],
                       mp.Provenance.BESTFIT)
        rep = mp.verify_plan(inst, plan)
        assert rep.valid == case["valid"]
        assert rep.peak_recomputed == case["peak_recomputed"]
        assert rep.capacity_ok == case["capacity_ok"]
        assert repr(rep.utilization) == case["utilization"]
        assert [[v.pair[0], v.pair[1], v.overlap_bytes, v.overlap_ticks]
                for v in rep.violations] == case["violations"]
        assert mp.report_to_json(rep) == case["report_json"]


def test_clique_lb_matches_reference(small_plans):
    for case in small_plans:
        a, f, s = blocks_arrays(case["blocks"])
        from paper_1804_10001_b200.verifier import clique_lower_bound_arrays
        assert clique_lower_bound_arrays(a, f, s) == case["clique_lb"], case["name"]
    inst = mp.build_instance([(4, 1, 3), (2, 2, 5), (3, 4, 6)])
    assert mp.clique_lower_bound(inst) == 6


def test_worked_verify_cases():
    inst = mp.build_instance([(4, 1, 3), (2, 2, 5), (3, 4, 6)])
    ok = mp.verify_plan(inst, mp.Plan({1: 2, 2: 0, 3: 2}, 6, mp.Provenance.BESTFIT))
    assert ok.valid and ok.utilization == pytest.approx(20 / 30)
    bad = mp.verify_plan(inst, mp.Plan({1: 0, 2: 0, 3: 2}, 6, mp.Provenance.BESTFIT))
    assert not bad.valid and bad.violations[0].pair == (1, 2)
    assert bad.violations[0].overlap_bytes == 2 and bad.violations[0].overlap_ticks == 1
    neg = mp.verify_plan(inst, mp.Plan({1: -1, 2: 4, 3: 4}, 8, mp.Provenance.BESTFIT))
    assert not neg.valid
    with pytest.raises(mp.MissingOffset):
        mp.verify_plan(inst, mp.Plan({1: 2, 2: 0}, 6, mp.Provenance.BESTFIT))
    empty = mp.verify_plan(mp.build_instance([]), mp.Plan({}, 0, mp.Provenance.BESTFIT))
    assert empty.valid and empty.utilization == 0.0


@pytest.mark.parametrize("name", ["cnn_1e4", "uniform_1e4", "walk_1e4"])
def test_verify_large_vs_oracle(large_plans, name):
    b = large_plans[name + "_blocks"]
    a, f, s = b[:, 1], b[:, 2], b[:, 0]
    off = large_plans[name + "_offsets"].copy()
    r = mp.verify_arrays(a, f, s, off)
    assert r["n_violations"] == 0 and r["peak_recomputed"] == int(large_plans[name + "_peak"][0])
    o = oracle.verify(a, f, s, off)
    assert r["used"] == o["used"]
    # crafted mutations: drop random blocks; every violation must match the oracle
    rng = np.random.default_rng(1)
    moved = 0
    while moved < 25:
        i, j = rng.integers(0, len(off), 2)
        if i != j and max(a[i], a[j]) < min(f[i], f[j]):  # colliding pair
            off[i] = off[j] + 512 * int(rng.integers(0, 2))
            moved += 1
    r = mp.verify_arrays(a, f, s, off)
    o = oracle.verify(a, f, s, off, viol_cap=1 << 20)
    assert r["n_violations"] == o["n_violations"] > 0
    assert r["violations"] == o["violations"]
    assert r["offsets_ok"] == o["offsets_ok"]
