"""CPU-only tests of the host-side façade: boundary types, ingest, JSON,
generators (pinned to reference output), and the C-ABI library surface."""
import ctypes
import hashlib
import json
import os
import random
import re

import numpy as np
import pytest

import paper_1804_10001_b200 as mp
from paper_1804_10001_b200 import _native as N
from paper_1804_10001_b200 import workloads as W
from conftest import GOLDEN, ROOT


# ---- boundary types (reference core.py) ----------------------------------
def test_block_request_validation():
    with pytest.raises(ValueError):
        mp.BlockRequest(0, 4, 0, 1)
    with pytest.raises(mp.ZeroSize):
        mp.BlockRequest(1, 0, 0, 1)
    with pytest.raises(ValueError):
        mp.BlockRequest(1, 4, -1, 1)
    with pytest.raises(mp.EmptyLifetime):
        mp.BlockRequest(1, 4, 3, 3)
    assert mp.BlockRequest(1, 4, 2, 7).lifetime == 5


def test_instance_validation_and_build():
    inst = mp.build_instance([(5, 0, 2), (3, 1, 4, "x")], alignment=4)
    assert [b.size for b in inst.blocks] == [8, 4]
    assert inst.capacity == 12 and inst.blocks[1].label == "x"
    assert inst.span() == (0, 4) and inst.total_bytes == 12
    with pytest.raises(mp.ZeroSize):
        mp.build_instance([(0, 0, 1)])
    with pytest.raises(mp.CapacityTooSmall):
        mp.build_instance([(5, 0, 1)], capacity=4)
    with pytest.raises(ValueError):
        mp.build_instance([(5, 0, 1)], alignment=0)
    with pytest.raises(ValueError):
        mp.DsaInstance((mp.BlockRequest(2, 4, 0, 1),), capacity=4)
    with pytest.raises(ValueError):
        mp.DsaInstance((mp.BlockRequest(1, 5, 0, 1),), capacity=8, alignment=4)
    assert mp.build_instance([]).span() == (0, 0)
    a, f, s = inst.arrays()
    assert a.tolist() == [0, 1] and f.tolist() == [2, 4] and s.tolist() == [8, 4]


def test_int64_guard():
    inst = mp.build_instance([(1, 0, 1 << 64)])
    with pytest.raises(ValueError):
        inst.arrays()


def test_plan_from_offsets():
    inst = mp.build_instance([(4, 1, 3), (2, 2, 5), (3, 4, 6)])
    p = mp.Plan.from_offsets(inst, {1: 2, 2: 0, 3: 2}, mp.Provenance.BESTFIT)
    assert p.peak == 6
    with pytest.raises(mp.MissingOffset):
        mp.Plan.from_offsets(inst, {1: 2}, mp.Provenance.BESTFIT)


def test_plan_json_byte_identical_to_reference():
    text = open(os.path.join(GOLDEN, "plan_worked.json")).read()
    inst, plan = mp.plan_from_json(text)
    assert mp.plan_to_json(inst, plan) == text
    assert plan.offsets == {1: 2, 2: 0, 3: 2} and inst.blocks[1].label == "w2"
    with pytest.raises(mp.MemplanError):
        mp.plan_from_json(json.dumps({"blocks": []}))


def test_colliding_pairs_brute_force():
    rng = random.Random(3)
    for _ in range(50):
        blocks = []
        for _ in range(rng.randint(0, 25)):
            a = rng.randint(0, 20)
            blocks.append((rng.randint(1, 9), a, a + rng.randint(1, 8)))
        inst = mp.build_instance(blocks)
        want = {(x.id, y.id) for x in inst.blocks for y in inst.blocks
                if x.id < y.id and max(x.alloc_time, y.alloc_time) < min(x.free_time, y.free_time)}
        got = mp.colliding_pairs(inst)
        assert set(got.pairs) == want and len(got) == len(want)
        assert list(got) == sorted(want)


def test_reduction_and_report_json():
    assert mp.reduction_vs(4, 6) == pytest.approx(1 / 3)
    assert mp.reduction_vs(9, 6) == pytest.approx(-0.5)
    with pytest.raises(mp.ZeroBaseline):
        mp.reduction_vs(1, 0)
    rep = mp.VerifyReport(False, (mp.Violation((1, 2), 2, 1),), 5, True, 0.5)
    doc = json.loads(mp.report_to_json(rep))
    assert doc["violations"] == [{"pair": [1, 2], "overlap_bytes": 2, "overlap_ticks": 1}]


# ---- ingest (reference profiler.py), pinned to reference output -----------
def test_profiles_match_reference(profile_golden):
    for case in profile_golden:
        ev = mp.parse_trace(case["text"])
        assert [[e.kind, e.size, e.ref, e.label] for e in ev] == case["events"]
        prof = mp.record(ev)
        got = [[b.id, b.size, b.alloc_time, b.free_time, b.label] for b in prof.managed]
        assert got == case["managed"]
        assert prof.unmanaged_count == case["unmanaged_count"]
        assert prof.horizon == case["horizon"]


def test_parse_errors():
    with pytest.raises(mp.TraceSyntaxError, match="line 2"):
        mp.parse_trace("A 4\nX 1\n")
    with pytest.raises(mp.TraceSyntaxError, match="line 1"):
        mp.parse_trace("A\n")
    with pytest.raises(mp.TraceSyntaxError, match="line 3"):
        mp.parse_trace("A 1\nA 2\nF x\n")
    for bad in ("F 0\n", "I now\n", "R x\n", "F 1 2\n"):
        with pytest.raises(mp.TraceSyntaxError):
            mp.parse_trace(bad)
    with pytest.raises(mp.NegativeSize):
        mp.parse_trace("A -3\n")
    assert mp.parse_trace("A 0\n") == [mp.alloc(0)]


def test_record_errors():
    with pytest.raises(mp.UnknownBlockRef):
        mp.record([mp.free(1)])
    with pytest.raises(mp.DoubleFree):
        mp.record([mp.alloc(3), mp.free(1), mp.free(1)])
    with pytest.raises(mp.UnbalancedResume):
        mp.record([mp.resume()])
    with pytest.raises(mp.NegativeSize):
        mp.record([mp.alloc(-1)])


# ---- generators, pinned by hash to the reference's text -------------------
def test_generators_match_reference(trace_golden):
    for c in trace_golden["cnn"]:
        txt = mp.cnn_like_trace(mp.GenSpec(model="cnn", layers=c["layers"], batch=c["batch"],
                                           seed=c["seed"], workspace=c["workspace"]))
        assert hashlib.sha256(txt.encode()).hexdigest() == c["sha256"], c
    for c in trace_golden["rnn"]:
        vl = tuple(c["variable_length"]) if c["variable_length"] else None
        spec = mp.GenSpec(model="rnn", layers=c["layers"], batch=c["batch"], seed=c["seed"],
                          variable_length=vl, untimed=c["untimed"])
        txt = mp.rnn_like_trace(spec, c["length"])
        assert hashlib.sha256(txt.encode()).hexdigest() == c["sha256"], c
    for c in trace_golden["rnn_lengths"]:
        vl = tuple(c["variable_length"]) if c["variable_length"] else None
        spec = mp.GenSpec(model="rnn", seed=c["seed"], variable_length=vl)
        assert mp.rnn_epoch_lengths(spec, 64) == c["lengths"]
    for c in trace_golden["walk"]:
        txt = W.walk_trace(c["n"], c["seed"])
        assert hashlib.sha256(txt.encode()).hexdigest() == c["sha256"]
    u = [list(t) for t in W.uniform_blocks(1000, 0)]
    assert hashlib.sha256(json.dumps(u).encode()).hexdigest() == trace_golden["uniform_1000_0_sha256"]


def test_genspec_validation():
    for kw in ({"model": "x"}, {"model": "cnn", "layers": 0}, {"model": "cnn", "batch": 0},
               {"model": "rnn", "variable_length": (5, 2)}):
        with pytest.raises(ValueError):
            mp.GenSpec(**kw)
    with pytest.raises(ValueError):
        mp.rnn_like_trace(mp.GenSpec(model="rnn"), 0)


@pytest.mark.parametrize("net,batch,lo,hi", [("alexnet", 32, 50, 300),
                                             ("googlenet", 64, 300, 3000),
                                             ("resnet50", 64, 300, 3000),
                                             ("inception_resnet_v2", 128, 1000, 20000)])
def test_net_traces(net, batch, lo, hi):
    txt = W.net_trace(net, batch)
    prof = mp.record(mp.parse_trace(txt))
    n = len(prof.managed)
    assert lo <= n <= hi, n
    # every allocation is released within the iteration
    assert all(b.free_time < prof.horizon for b in prof.managed)
    inst = mp.profile_to_instance(prof, alignment=512)
    assert all(b.size % 512 == 0 for b in inst.blocks)


def test_lstm_profiles():
    traces = W.lstm_profiles(8)
    assert len(traces) == 8
    spec = mp.GenSpec(model="rnn", layers=6, batch=64, seed=2024, variable_length=(10, 50))
    assert traces[3] == mp.rnn_like_trace(spec, mp.rnn_epoch_lengths(spec, 8)[3])
    assert len(mp.record(mp.parse_trace(traces[0])).managed) == 13


# ---- C ABI surface ---------------------------------------------------------
def test_library_exports_every_header_symbol():
    header = open(os.path.join(ROOT, "include", "memplan_b200.h")).read()
    header = re.sub(r"/\*.*?\*/", "", header, flags=re.S)
    declared = set(re.findall(r"\b(mp_[a-z0-9_]+)\s*\(", header))
    lib = ctypes.CDLL(N.LIB_PATH)
    missing = [s for s in sorted(declared) if not hasattr(lib, s)]
    assert declared and not missing, missing
    assert {s for s, _, _ in N.SIGNATURES} == declared


def test_no_cpu_fallback_without_device():
    if N.lib().mp_device_count() > 0:
        pytest.skip("a CUDA device is present")
    inst = mp.build_instance([(4, 1, 3), (2, 2, 5), (3, 4, 6)])
    with pytest.raises(mp.NoDevice):
        mp.solve_bestfit(inst)
    with pytest.raises(mp.NoDevice):
        mp.verify_plan(inst, mp.Plan({1: 2, 2: 0, 3: 2}, 6, mp.Provenance.BESTFIT))


def test_pool_and_simulate_pool_host_only():
    """The pool is host C++ (no device needed): reference arena.py:59-129."""
    ev = mp.parse_trace("A 4\nF 1\nA 2\nA 2\nF 2\nF 3\n")
    assert mp.simulate_pool(ev).peak == 6
    pool = mp.PoolAllocator()
    assert pool.alloc(8) == 0 and pool.alloc(4) == 8
    pool.free(1)
    assert pool.alloc(3) == 0 and pool.peak == 12 and pool.live_bytes() == 12
    with pytest.raises(mp.DoubleFree):
        pool.free(1) or pool.free(1)
    with pytest.raises(mp.UnknownId):
        pool.free(99)
    small = mp.PoolAllocator(capacity=10)
    small.alloc(6)
    small.free(1)
    assert small.alloc(8) == 6  # flush then bump
    with pytest.raises(mp.OutOfMemory):
        small.alloc(5)


def test_pool_peak_matches_reference(small_plans):
    by = {c["name"]: c for c in small_plans}
    spec = mp.GenSpec(model="cnn", layers=20, seed=42, workspace=True)
    events = mp.parse_trace(mp.cnn_like_trace(spec))
    assert mp.simulate_pool(events).peak == by["cnn20_seed42"]["pool_peak"] == 704864
    from paper_1804_10001_b200.arena import simulate_pool_peak
    assert simulate_pool_peak(events) == 704864


def test_host_skyline_types_drive_equals_oracle():
    """The host skyline types (skyline.py: OffsetLineSet, find_block,
    _RemainingBlocks — the reference's step-by-step surface) driven one
    operation at a time reproduce the oracle's plans (the reference's
    test_skyline_tracks_placed_blocks_and_solver_agrees, on CPU)."""
    import random

    import oracle
    import paper_1804_10001_b200 as mp
    from paper_1804_10001_b200.skyline import _RemainingBlocks
    rng = random.Random(17)
    for _ in range(60):
        n = rng.randint(1, 40)
        blocks = []
        for _ in range(n):
            a = rng.randint(0, 49)
            blocks.append((rng.randint(1, 16), a, rng.randint(a + 1, 50)))
        inst = mp.build_instance(blocks)
        t_lo = min(b.alloc_time for b in inst.blocks)
        t_hi = max(b.free_time for b in inst.blocks)
        ls = mp.OffsetLineSet(t_lo, t_hi)
        remaining = _RemainingBlocks(inst.blocks)
        offsets = {}
        while len(remaining):
            line = ls.choose_offset()
            block = remaining.take_best(line.time_lo, line.time_hi)
            if block is None:
                ls.lift_up(line)
            else:
                offsets[block.id] = ls.place(line, block)
            tiles = ls.as_tuples()
            assert tiles[0][0] == t_lo and tiles[-1][1] == t_hi
            assert all(x[1] == y[0] and x[2] != y[2] for x, y in zip(tiles, tiles[1:]))
        a, f, s = inst.arrays()
        ref, _ = oracle.solve_bestfit(a, f, s)
        assert [offsets[i + 1] for i in range(len(a))] == ref.tolist()
