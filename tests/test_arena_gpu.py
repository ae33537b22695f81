"""Replay arena (H1) against scripted reference sessions and the reference
acceptance criteria 6/7 (test_acceptance.py:192-253)."""
import pytest

import paper_1804_10001_b200 as mp

pytestmark = pytest.mark.gpu


def _run_script(arena, script):
    log = []
    for op in script:
        kind = op[0]
        try:
            if kind == "A":
                r = arena.alloc(op[1])
            elif kind == "F":
                r = arena.free(op[1])
            elif kind == "I":
                r = arena.interrupt()
            elif kind == "R":
                r = arena.resume()
            elif kind == "X":
                r = arena.reset()
            elif kind == "C":
                r = arena.close()
            elif kind == "O":
                r = arena.reoptimize().peak
            log.append(["ok", r])
        except mp.MemplanError as exc:
            log.append(["err", type(exc).__name__])
        log[-1].append({
            "lam": arena.lam, "reopt": arena.reopt_count, "forced": arena.forced_closes,
            "peak": arena.plan.peak, "usage": arena.peak_usage(),
            "pool_peak": arena.fallback.peak,
            "live": sorted([k, v[0], v[1]] for k, v in arena.live_blocks().items()),
        })
    return log


def test_scripts_match_reference(arena_golden):
    for case in arena_golden:
        if "script" not in case:
            continue
        inst = mp.build_instance([tuple(b) for b in case["blocks"]])
        arena = mp.Arena(mp.solve_bestfit(inst), inst, base=case["base"], mode=case["mode"])
        log = _run_script(arena, case["script"])
        assert log == case["log"], case["name"]
        assert [arena.plan.offsets[k] for k in sorted(arena.plan.offsets)] == case["final_offsets"]


def test_rnn_growth_matches_reference(arena_golden):
    case = next(c for c in arena_golden if c["name"] == "rnn_growth")
    spec = mp.GenSpec(model="rnn", layers=6, batch=16, seed=2024, variable_length=(10, 50))
    lengths = mp.rnn_epoch_lengths(spec, 60)
    inst = mp.profile_to_instance(mp.record(mp.parse_trace(mp.rnn_like_trace(spec, lengths[0]))))
    arena = mp.Arena(mp.solve_bestfit(inst), inst)
    for (length, reopt, peak, addrs), ell in zip(case["per_epoch"], lengths):
        assert length == ell
        got = mp.replay_events(arena, mp.parse_trace(mp.rnn_like_trace(spec, ell)))
        arena.reset()
        assert (got, arena.reopt_count, arena.plan.peak) == (addrs, reopt, peak)


def test_invalid_plan_rejected():
    inst = mp.build_instance([(4, 1, 3), (2, 2, 5), (3, 4, 6)])
    with pytest.raises(mp.InvalidPlan):
        mp.Arena(mp.Plan({1: 0, 2: 0, 3: 2}, 6, mp.Provenance.BESTFIT), inst)
    with pytest.raises(ValueError):
        mp.Arena(mp.solve_bestfit(inst), inst, mode="loose")


def test_acceptance_6_hot_replay_determinism():
    spec = mp.GenSpec(model="cnn", layers=12, seed=7)
    events = mp.parse_trace(mp.cnn_like_trace(spec))
    inst = mp.profile_to_instance(mp.record(events))
    arena = mp.Arena(mp.solve_bestfit(inst), inst)
    first = None
    for _ in range(100):
        addrs = mp.replay_events(arena, events)
        first = first or addrs
        assert addrs == first
        arena.reset()
    assert arena.reopt_count == 0 and arena.forced_closes == 0


def test_acceptance_7_reoptimisation_on_growth():
    spec = mp.GenSpec(model="rnn", layers=6, batch=16, seed=2024, variable_length=(10, 50))
    lengths = mp.rnn_epoch_lengths(spec, 200)
    expected, running = 0, lengths[0]
    for ell in lengths[1:]:
        if ell > running:
            expected, running = expected + 1, ell
    inst = mp.profile_to_instance(mp.record(mp.parse_trace(mp.rnn_like_trace(spec, lengths[0]))))
    arena = mp.Arena(mp.solve_bestfit(inst), inst)
    for ell in lengths:
        mp.replay_events(arena, mp.parse_trace(mp.rnn_like_trace(spec, ell)))
        arena.reset()
    assert arena.reopt_count == expected
    mx = mp.profile_to_instance(mp.record(mp.parse_trace(mp.rnn_like_trace(spec, max(lengths)))))
    assert arena.peak_usage() == mp.solve_bestfit(mx).peak == 107744
    mp.replay_events(arena, mp.parse_trace(mp.rnn_like_trace(spec, min(lengths))))
    arena.reset()
    assert arena.reopt_count == expected and arena.fallback.peak == 0


def test_live_blocks_never_overlap_during_replay():
    import random
    rng = random.Random(12)
    for _ in range(20):
        lines, live, count = [], [], 0
        for _ in range(rng.randint(1, 30)):
            if live and rng.random() < 0.45:
                lines.append(f"F {live.pop(rng.randrange(len(live)))}")
            else:
                count += 1
                live.append(count)
                lines.append(f"A {rng.randint(1, 16)}")
        events = mp.parse_trace("\n".join(lines) + "\n")
        inst = mp.profile_to_instance(mp.record(events))
        arena = mp.Arena(mp.solve_bestfit(inst), inst)
        for ev in events:
            if ev.kind == "alloc":
                arena.alloc(ev.size)
                spans = sorted(arena.live_blocks().values())
                for (a1, s1), (a2, s2) in zip(spans, spans[1:]):
                    assert a1 + s1 <= a2
            else:
                arena.free(ev.ref)


def test_arena_ns_per_alloc():
    """C-ABI replay cost on the hot cnn-like L=5000 trace."""
    from paper_1804_10001_b200.arena import encode_events
    import ctypes
    from paper_1804_10001_b200 import _native as N
    events = mp.parse_trace(mp.cnn_like_trace(mp.GenSpec(model="cnn", layers=5000, seed=0)))
    inst = mp.profile_to_instance(mp.record(events))
    arena = mp.Arena(mp.solve_bestfit(inst), inst)
    kinds, values = encode_events(events)
    ns = ctypes.c_double()
    assert N.lib().mp_arena_bench(arena._h, N.ptr(kinds), N.ptr(values), len(kinds), 20,
                                  ctypes.byref(ns)) == 0
    print("arena ns/alloc", ns.value)
    assert ns.value < 200


def test_fallback_is_a_full_pool_allocator():
    """Arena.fallback is the arena's own PoolAllocator (arena.py:172): the
    interrupted requests it served are visible through its full interface
    (test_arena.py:66-71 reads .peak; cursor / live_bytes / alloc / free
    complete the reference PoolAllocator surface)."""
    inst = mp.build_instance([(4, 1, 3), (2, 2, 5), (3, 4, 6)])
    arena = mp.Arena(mp.solve_bestfit(inst), inst)
    arena.interrupt()
    arena.alloc(9)
    arena.resume()
    fb = arena.fallback
    assert isinstance(fb, mp.PoolAllocator)
    assert fb.peak == 9 and fb.cursor == 9 and fb.live_bytes() == 9 and fb.last_ref == 1
    addr = fb.alloc(5)
    assert addr == 9 and fb.cursor == 14 and fb.live_bytes() == 14
    fb.free(fb.last_ref)
    assert fb.live_bytes() == 9
    assert arena.peak_usage() == arena.plan.peak + fb.peak


def test_replay_events_applies_prefix_before_unknown_kind():
    """replay_events applies the events before an unknown kind, then raises
    (the reference's event-by-event loop, arena.py:325-340)."""
    inst = mp.build_instance([(4, 1, 3), (2, 2, 5), (3, 4, 6)])
    arena = mp.Arena(mp.solve_bestfit(inst), inst)
    bad = mp.TraceEvent("bogus")
    events = [mp.alloc(4), mp.alloc(2), bad, mp.alloc(3)]
    with pytest.raises(mp.MemplanError):
        mp.replay_events(arena, events)
    assert arena.lam == 3
