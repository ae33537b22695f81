"""The reference acceptance criteria (tests/test_acceptance.py) that touch
the hot path, run through this package on the GPU."""
import random

import numpy as np
import pytest

import oracle
import paper_1804_10001_b200 as mp

pytestmark = pytest.mark.gpu


def test_5_pool_vs_plan_reduction():
    events = mp.parse_trace(mp.cnn_like_trace(mp.GenSpec(model="cnn", layers=20, seed=42)))
    inst = mp.profile_to_instance(mp.record(events))
    plan = mp.solve_bestfit(inst)
    pool = mp.simulate_pool(events)
    assert plan.peak == 500448 and pool.peak == 704864
    assert mp.reduction_vs(plan.peak, pool.peak) >= 0.15


def test_8_worked_instance():
    inst = mp.build_instance([(4, 1, 3), (2, 2, 5), (3, 4, 6)])
    plan = mp.solve_bestfit(inst)
    assert plan.offsets == {1: 2, 2: 0, 3: 2} and plan.peak == 6
    assert plan.provenance is mp.Provenance.BESTFIT
    assert mp.clique_lower_bound(inst) == 6


def test_3_verification_soundness():
    rng = random.Random(31415)
    mutations = detected = 0
    for _ in range(200):
        n = rng.randint(1, 200)
        blocks = []
        for _ in range(n):
            a = rng.randint(0, 399)
            blocks.append((rng.randint(1, 64), a, rng.randint(a + 1, 400)))
        inst = mp.build_instance(blocks)
        plan = mp.solve_bestfit(inst)
        assert mp.verify_plan(inst, plan).valid
        by = {b.id: b for b in inst.blocks}
        target = None
        for i, j in mp.colliding_pairs(inst):
            if plan.offsets[i] == plan.offsets[j] + by[j].size:
                target = i
                break
            if plan.offsets[j] == plan.offsets[i] + by[i].size:
                target = j
                break
        if target is None:
            continue
        mutated = dict(plan.offsets)
        mutated[target] -= 1
        mutations += 1
        detected += not mp.verify_plan(inst, mp.Plan(mutated, plan.peak, plan.provenance)).valid
    assert mutations > 100 and detected == mutations


def test_determinism_and_uniform_scaling():
    rng = random.Random(5)
    for _ in range(40):
        blocks = []
        for _ in range(rng.randint(1, 20)):
            a = rng.randint(0, 79)
            blocks.append((rng.randint(1, 32), a, rng.randint(a + 1, 80)))
        inst = mp.build_instance(blocks)
        base = mp.solve_bestfit(inst)
        assert base == mp.solve_bestfit(inst)
        c = rng.randint(2, 9)
        big = mp.solve_bestfit(mp.build_instance([(b.size * c, b.alloc_time, b.free_time)
                                                  for b in inst.blocks]))
        assert big.peak == base.peak * c
        assert big.offsets == {i: o * c for i, o in base.offsets.items()}


@pytest.mark.parametrize("net,batch", [("alexnet", 32), ("googlenet", 64), ("resnet50", 64),
                                       ("inception_resnet_v2", 128)])
def test_net_configs_bit_exact(net, batch):
    inst = mp.profile_to_instance(mp.record(mp.parse_trace(mp.net_trace(net, batch))),
                                  alignment=512)
    plan = mp.solve_bestfit(inst)
    a, f, s = inst.arrays()
    off, peak = oracle.solve_bestfit(a, f, s)
    assert plan.peak == peak and [plan.offsets[i + 1] for i in range(len(a))] == off.tolist()
    assert mp.verify_plan(inst, plan).valid
    assert plan.peak >= mp.clique_lower_bound(inst)


def test_lstm_batched_bit_exact():
    from paper_1804_10001_b200.workloads import lstm_profiles
    insts = [mp.profile_to_instance(mp.record(mp.parse_trace(t)), alignment=512)
             for t in lstm_profiles(512)]
    plans = mp.solve_bestfit_batched(insts)
    for inst, plan in zip(insts, plans):
        a, f, s = inst.arrays()
        off, peak = oracle.solve_bestfit(a, f, s)
        assert plan.peak == peak and list(plan.offsets.values()) == off.tolist()


def test_full_size_properties():
    """BASELINE's largest synthetic size (10^6 blocks), checked through
    size-independent properties instead of the oracle: the GPU validator
    finds no overlap and recomputes the same peak, and the clique lower
    bound does not exceed it.  At 10^5 blocks: scaling all sizes by c scales
    offsets and peak by c; a strictly increasing relabelling of the times
    (shift, stretch — the stretched one leaves the raw-rank range of K0)
    leaves every offset unchanged; the batched path equals the single one."""
    from paper_1804_10001_b200.bestfit import solve_bestfit_arrays, solve_bestfit_batched_arrays
    from paper_1804_10001_b200.verifier import verify_arrays, clique_lower_bound_arrays
    from paper_1804_10001_b200.workloads import uniform_arrays
    a, f, s = uniform_arrays(1_000_000, 11)
    s = ((s + 511) // 512) * 512
    off, peak = solve_bestfit_arrays(a, f, s)
    rep = verify_arrays(a, f, s, off, viol_cap=16)
    assert rep["n_violations"] == 0 and rep["offsets_ok"] and rep["peak_recomputed"] == peak
    assert clique_lower_bound_arrays(a, f, s) <= peak
    assert np.all(off % 512 == 0)

    a, f, s = uniform_arrays(100_000, 12)
    s = ((s + 511) // 512) * 512
    off, peak = solve_bestfit_arrays(a, f, s)
    off3, peak3 = solve_bestfit_arrays(a, f, 3 * s)
    assert peak3 == 3 * peak and np.array_equal(off3, 3 * off)
    for aa, ff in ((a + 12345, f + 12345), (7 * a + 3, 7 * f + 3), (1000 * a, 1000 * f)):
        o2, p2 = solve_bestfit_arrays(aa, ff, s)
        assert p2 == peak and np.array_equal(o2, off)
    # three copies in one batch, one of them stretched (batch span > 2^25:
    # dense ranks), all equal to the single plan
    tp = np.arange(4, dtype=np.int64) * len(a)
    A = np.concatenate([a, 1000 * a, a]); F = np.concatenate([f, 1000 * f, f])
    offb, peaks = solve_bestfit_batched_arrays(tp, A, F, np.concatenate([s, s, s]))
    assert list(peaks) == [peak] * 3
    for t in range(3):
        assert np.array_equal(offb[tp[t]:tp[t + 1]], off)
