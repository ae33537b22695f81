"""Generate the golden fixtures under tests/golden/ FROM THE REFERENCE ITSELF.

Runs only in the build container, where the read-only reference package is
importable (PYTHONPATH=/root/reference/pkg/src).  The outputs are committed;
nothing on the GPU box reads /root/reference.

    python tests/golden/make_golden.py

Every fixture records what the reference's public API returns
(solve_bestfit, verify_plan, clique_lower_bound, record, the generators,
Arena/replay_events, simulate_pool, plan_to_json) on seeded inputs, including
the size tie-break vectors G1/G2 and the staircase G3 from SURVEY.md §8(c).
"""

from __future__ import annotations

import gzip
import hashlib
import json
import os
import random
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
import memplan as M  # noqa: E402  (the reference)

OUT = os.path.dirname(os.path.abspath(__file__))


def inst_blocks(inst):
    return [[b.size, b.alloc_time, b.free_time] for b in inst.blocks]


def plan_case(name, inst, extra=None):
    plan = M.solve_bestfit(inst)
    case = {
        "name": name,
        "alignment": inst.alignment,
        "capacity": inst.capacity,
        "blocks": inst_blocks(inst),
        "offsets": [plan.offsets[b.id] for b in inst.blocks],
        "peak": plan.peak,
        "clique_lb": M.clique_lower_bound(inst),
    }
    if extra:
        case.update(extra)
    return case


# ---- instance families (restated identically in the product's workloads) ----
def random_instance(rng, max_n=60, max_tick=80, max_size=32):
    """tests/test_bestfit.py:19-26 style."""
    n = rng.randint(1, max_n)
    blocks = []
    for _ in range(n):
        a = rng.randint(0, max_tick - 1)
        f = rng.randint(a + 1, max_tick)
        blocks.append((rng.randint(1, max_size), a, f))
    return M.build_instance(blocks)


def uniform_blocks(n, seed):
    """SURVEY.md Appendix A step 2 'uniform'."""
    r = random.Random(seed)
    out = []
    for _ in range(n):
        a = r.randint(0, 2 * n - 1)
        f = r.randint(a + 1, 2 * n)
        out.append((r.randint(1, 1 << 20), a, f))
    return out


def walk_trace(n, seed, p_free=0.45, max_size=1 << 20):
    """SURVEY.md Appendix A step 2 'walk' as trace text."""
    r = random.Random(seed)
    lines, live, count = [], [], 0
    while count < n:
        if live and r.random() < p_free:
            lines.append(f"F {live.pop(r.randrange(len(live)))}")
        else:
            count += 1
            live.append(count)
            lines.append(f"A {r.randint(1, max_size)}")
    return "\n".join(lines) + "\n"


def small_cases():
    cases = []
    cases.append(plan_case("worked", M.build_instance([(4, 1, 3), (2, 2, 5), (3, 4, 6)])))
    cases.append(plan_case("single", M.build_instance([(7, 0, 9)])))
    cases.append(plan_case("disjoint", M.build_instance([(3, 0, 2), (5, 3, 6)])))
    cases.append(plan_case("empty", M.build_instance([])))
    cases.append(plan_case("G1_size_tiebreak", M.build_instance([(1, 5, 6), (2, 5, 6)])))
    cases.append(plan_case("G2_size_tiebreak",
                           M.build_instance([(5, 4, 8), (1, 0, 3), (5, 1, 4), (2, 3, 6)])))
    cases.append(plan_case("G3_staircase",
                           M.build_instance([(k + 1, 2 * k, 2 * k + 1) for k in range(2000)])))
    # ties everywhere: equal lifetimes and sizes, equal alloc times
    rng = random.Random(99)
    for t in range(20):
        blocks = []
        for _ in range(rng.randint(1, 80)):
            a = rng.randint(0, 6)
            blocks.append((rng.choice([1, 2, 4]), a, a + rng.choice([1, 2, 3])))
        cases.append(plan_case(f"ties_{t}", M.build_instance(blocks)))
    # int64-scale sizes and times
    rng = random.Random(1234)
    for t in range(10):
        blocks = []
        for _ in range(rng.randint(1, 60)):
            a = rng.randint(0, 1 << 40)
            f = a + rng.randint(1, 1 << 40)
            blocks.append((rng.randint(1, 1 << 44), a, f))
        cases.append(plan_case(f"bigint_{t}", M.build_instance(blocks, alignment=512)))
    # test_bestfit random_instance style, several seeds
    for seed in range(300):
        rng = random.Random(seed)
        cases.append(plan_case(f"rand_{seed}", random_instance(rng)))
    # acceptance small corpus (tests/test_acceptance.py:42-60)
    rng = random.Random(20260808)
    got = 0
    while got < 200:
        n = rng.randint(1, 10)
        blocks = []
        for _ in range(n):
            a = rng.randint(0, 29)
            f = rng.randint(a + 1, 30)
            blocks.append((rng.randint(1, 16), a, f))
        inst = M.build_instance(blocks)
        if len(M.colliding_pairs(inst)) > 20:
            continue
        cases.append(plan_case(f"acc_{got}", inst))
        got += 1
    # acceptance criterion 5 (cnn L=20 seed 42, alignment 1)
    spec = M.GenSpec(model="cnn", layers=20, seed=42, workspace=True)
    events = M.parse_trace(M.cnn_like_trace(spec))
    inst = M.profile_to_instance(M.record(events))
    cases.append(plan_case("cnn20_seed42", inst, {"pool_peak": M.simulate_pool(events).peak}))
    # acceptance criterion 7 max-length rnn instance
    spec = M.GenSpec(model="rnn", layers=6, batch=16, seed=2024, variable_length=(10, 50))
    lengths = M.rnn_epoch_lengths(spec, 200)
    inst = M.profile_to_instance(M.record(M.parse_trace(M.rnn_like_trace(spec, max(lengths)))))
    cases.append(plan_case("rnn6_maxlen", inst))
    # small uniform / walk / cnn at alignment 512
    for seed in range(3):
        cases.append(plan_case(f"uniform300_{seed}",
                               M.build_instance(uniform_blocks(300, seed), alignment=512)))
        cases.append(plan_case(f"walk300_{seed}", M.profile_to_instance(
            M.record(M.parse_trace(walk_trace(300, seed))), alignment=512)))
        cases.append(plan_case(f"cnn300_{seed}", M.profile_to_instance(M.record(M.parse_trace(
            M.cnn_like_trace(M.GenSpec(model="cnn", layers=150, seed=seed)))), alignment=512)))
    return cases


def large_cases():
    """n = 10^4 instances: store only offsets/peak (inputs are regenerated by
    the product's own generators, whose traces are pinned in traces.json)."""
    out = {}
    n = 10000
    insts = {
        "cnn_1e4": M.profile_to_instance(M.record(M.parse_trace(M.cnn_like_trace(
            M.GenSpec(model="cnn", layers=n // 2, seed=0)))), alignment=512),
        "uniform_1e4": M.build_instance(uniform_blocks(n, 0), alignment=512),
        "walk_1e4": M.profile_to_instance(M.record(M.parse_trace(walk_trace(n, 0))),
                                          alignment=512),
    }
    for name, inst in insts.items():
        plan = M.solve_bestfit(inst)
        out[name + "_offsets"] = np.array([plan.offsets[b.id] for b in inst.blocks], np.int64)
        out[name + "_peak"] = np.array([plan.peak], np.int64)
        out[name + "_blocks"] = np.array(inst_blocks(inst), np.int64)
        print(name, plan.peak, flush=True)
    return out


def trace_cases():
    t = {"cnn": [], "rnn": [], "rnn_lengths": [], "walk": []}
    for layers, batch, seed, ws in [(20, 32, 42, True), (12, 32, 7, True), (5, 8, 0, False),
                                    (100, 64, 3, True), (5000, 32, 0, True), (64, 1, 1, True)]:
        txt = M.cnn_like_trace(M.GenSpec(model="cnn", layers=layers, batch=batch, seed=seed,
                                         workspace=ws))
        t["cnn"].append({"layers": layers, "batch": batch, "seed": seed, "workspace": ws,
                         "sha256": hashlib.sha256(txt.encode()).hexdigest(),
                         "head": txt[:200]})
    for layers, batch, seed, vl, untimed, length in [
            (6, 16, 2024, (10, 50), False, 17), (6, 64, 2024, (10, 50), False, 50),
            (64, 64, 2024, (10, 50), False, 33), (3, 4, 5, None, True, 16)]:
        spec = M.GenSpec(model="rnn", layers=layers, batch=batch, seed=seed,
                         variable_length=vl, untimed=untimed)
        txt = M.rnn_like_trace(spec, length)
        t["rnn"].append({"layers": layers, "batch": batch, "seed": seed,
                         "variable_length": vl, "untimed": untimed, "length": length,
                         "sha256": hashlib.sha256(txt.encode()).hexdigest(), "text": txt
                         if len(txt) < 800 else None})
        t["rnn_lengths"].append({"seed": seed, "variable_length": vl,
                                 "lengths": M.rnn_epoch_lengths(spec, 64)})
    for n, seed in [(300, 0), (10000, 0)]:
        txt = walk_trace(n, seed)
        t["walk"].append({"n": n, "seed": seed,
                          "sha256": hashlib.sha256(txt.encode()).hexdigest()})
    u = uniform_blocks(1000, 0)
    t["uniform_1000_0_sha256"] = hashlib.sha256(json.dumps(u).encode()).hexdigest()
    return t


def profile_cases():
    traces = [
        "A 4\nA 2\nF 1\nA 3\nF 2\nF 3\n",
        "# hdr\nA 4 conv1\nI\nA 9\nR\nF 1\n",
        "A 4\nA 0\nA 3\nF 2\nF 1\nI\nA 5\nI\nA 6\nR\nF 5\nR\nF 3\nA 7 tail\n",
        M.cnn_like_trace(M.GenSpec(model="cnn", layers=6, seed=1)),
        M.rnn_like_trace(M.GenSpec(model="rnn", layers=3, batch=4, seed=5, untimed=True), 12),
        walk_trace(200, 3),
    ]
    out = []
    for txt in traces:
        ev = M.parse_trace(txt)
        prof = M.record(ev)
        out.append({
            "text": txt,
            "events": [[e.kind, e.size, e.ref, e.label] for e in ev],
            "managed": [[b.id, b.size, b.alloc_time, b.free_time, b.label] for b in prof.managed],
            "unmanaged_count": prof.unmanaged_count,
            "horizon": prof.horizon,
        })
    return out


def verify_cases():
    out = []
    rng = random.Random(31415)
    for t in range(150):
        n = rng.randint(1, 120)
        blocks = []
        for _ in range(n):
            a = rng.randint(0, 199)
            f = rng.randint(a + 1, 200)
            blocks.append((rng.randint(1, 64), a, f))
        inst = M.build_instance(blocks, capacity=None if t % 3 else 10 ** 6)
        plan = M.solve_bestfit(inst)
        offsets = dict(plan.offsets)
        peak = plan.peak
        # mutate some plans: drop a random block by a random amount
        if t % 2 == 1:
            k = rng.randint(1, n)
            offsets[k] = max(-3, offsets[k] - rng.randint(1, 40))
        if t % 7 == 3:
            peak += 1
        rep = M.verify_plan(inst, M.Plan(offsets, peak, M.Provenance.BESTFIT))
        out.append({
            "blocks": inst_blocks(inst), "capacity": inst.capacity,
            "offsets": [offsets[b.id] for b in inst.blocks], "peak": peak,
            "valid": rep.valid, "peak_recomputed": rep.peak_recomputed,
            "capacity_ok": rep.capacity_ok, "utilization": repr(rep.utilization),
            "violations": [[v.pair[0], v.pair[1], v.overlap_bytes, v.overlap_ticks]
                           for v in rep.violations],
            "report_json": M.report_to_json(rep),
        })
    return out


def arena_cases():
    """Scripted Arena sessions; each op's observable result is recorded."""
    out = []

    def run(inst, script, mode="lenient", base=0):
        arena = M.Arena(M.solve_bestfit(inst), inst, base=base, mode=mode)
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
            except M.MemplanError as exc:
                log.append(["err", type(exc).__name__])
            log[-1].append({
                "lam": arena.lam, "reopt": arena.reopt_count, "forced": arena.forced_closes,
                "peak": arena.plan.peak, "usage": arena.peak_usage(),
                "pool_peak": arena.fallback.peak,
                "live": sorted([k, v[0], v[1]] for k, v in arena.live_blocks().items()),
            })
        final_offsets = [arena.plan.offsets[k] for k in sorted(arena.plan.offsets)]
        return {"log": log, "final_offsets": final_offsets}

    worked = M.build_instance([(4, 1, 3), (2, 2, 5), (3, 4, 6)])
    scripts = [
        ("order", [("A", 4), ("A", 2), ("F", 1), ("A", 3)]),
        ("smaller", [("A", 3)]),
        ("growth", [("A", 5)]),
        ("growth_live", [("A", 4), ("A", 2), ("F", 1), ("A", 7)]),
        ("fallback", [("I",), ("A", 9), ("R",), ("F", 1), ("I",), ("A", 5)]),
        ("zero", [("A", 0), ("A", 4)]),
        ("close", [("C",), ("A", 4)]),
        ("double_free", [("A", 4), ("F", 1), ("F", 1), ("F", 3), ("F", 0)]),
        ("reset", [("A", 4), ("F", 1), ("X",), ("A", 4), ("X",)]),
        ("extra", [("A", 4), ("A", 2), ("F", 1), ("A", 3), ("A", 5), ("F", 2), ("F", 3),
                   ("F", 4), ("X",), ("A", 4), ("A", 2), ("F", 1), ("A", 3), ("A", 5),
                   ("A", 9), ("X",)]),
        ("resume_unbalanced", [("R",), ("I",), ("I",), ("A", 3), ("R",), ("A", 4), ("R",)]),
        ("explicit_reopt", [("A", 4), ("O",), ("A", 2)]),
    ]
    for name, script in scripts:
        for mode in ("lenient", "strict"):
            out.append({"name": f"{name}_{mode}", "blocks": inst_blocks(worked),
                        "mode": mode, "base": 1000 if name == "order" else 0,
                        "script": [list(s) for s in script],
                        **run(worked, script, mode=mode, base=1000 if name == "order" else 0)})
    # acceptance 7: growth-driven reoptimisation on the rnn workload
    spec = M.GenSpec(model="rnn", layers=6, batch=16, seed=2024, variable_length=(10, 50))
    lengths = M.rnn_epoch_lengths(spec, 60)
    inst = M.profile_to_instance(M.record(M.parse_trace(M.rnn_like_trace(spec, lengths[0]))))
    arena = M.Arena(M.solve_bestfit(inst), inst)
    per_epoch = []
    for length in lengths:
        addrs = M.replay_events(arena, M.parse_trace(M.rnn_like_trace(spec, length)))
        arena.reset()
        per_epoch.append([length, arena.reopt_count, arena.plan.peak, addrs])
    out.append({"name": "rnn_growth", "per_epoch": per_epoch})
    return out


def main():
    small = small_cases()
    with gzip.open(os.path.join(OUT, "plans_small.json.gz"), "wt") as fh:
        json.dump(small, fh)
    print("small cases:", len(small))
    with open(os.path.join(OUT, "traces.json"), "w") as fh:
        json.dump(trace_cases(), fh, indent=1)
    with open(os.path.join(OUT, "profiles.json"), "w") as fh:
        json.dump(profile_cases(), fh, indent=1)
    with gzip.open(os.path.join(OUT, "verify.json.gz"), "wt") as fh:
        json.dump(verify_cases(), fh)
    with gzip.open(os.path.join(OUT, "arena.json.gz"), "wt") as fh:
        json.dump(arena_cases(), fh)
    worked = M.build_instance([(4, 1, 3), (2, 2, 5, "w2"), (3, 4, 6)], capacity=50, alignment=1)
    with open(os.path.join(OUT, "plan_worked.json"), "w") as fh:
        fh.write(M.plan_to_json(worked, M.solve_bestfit(worked)))
    np.savez_compressed(os.path.join(OUT, "plans_large.npz"), **large_cases())


if __name__ == "__main__":
    main()
