"""Generate the LARGE-trace golden fixtures FROM THE REFERENCE ITSELF.

Runs only in the build container (the read-only reference package is
importable from /root/reference/pkg/src); the output `huge.json` is
committed and nothing on the GPU box reads /root/reference.

    python tests/golden/make_huge_golden.py [--jobs 7] [--only name,...]

For each configuration of SURVEY.md §8(d) item 5 (uniform / cnn / walk at
10^5, uniform / cnn / walk at 10^6) and BASELINE.json config 4 (all 4096 LSTM
profiles at L=6 and L=64) it records what the reference's
`solve_bestfit` (bestfit.py:276-309) returns, as

* `blocks_sha256`: sha256 of the int64 (size, alloc, free) rows of the
  instance in id order (the product's own generators must reproduce it),
* `offsets_sha256`: sha256 of the int64 offsets in id order,
* `peak`, `n`, and the reference's wall time on one core (`ref_s`).

10^6-block solves take ~30-60 min each on one core; the configurations run
in parallel worker processes and the file is rewritten after every result,
so a partial run keeps what it finished.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import multiprocessing as mp_
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "huge.json")


def _sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


def instance(name: str):
    import memplan as M  # the reference
    from make_golden import uniform_blocks, walk_trace
    fam, n, seed = name.split("_")
    n, seed = int(float(n)), int(seed[1:])
    if fam == "uniform":
        return M.build_instance(uniform_blocks(n, seed), alignment=512)
    if fam == "cnn":
        return M.profile_to_instance(M.record(M.parse_trace(M.cnn_like_trace(
            M.GenSpec(model="cnn", layers=n // 2, seed=seed)))), alignment=512)
    if fam == "walk":
        return M.profile_to_instance(M.record(M.parse_trace(walk_trace(n, seed))),
                                     alignment=512)
    raise ValueError(name)


def solve_one(name: str) -> dict:
    import memplan as M
    inst = instance(name)
    blocks = np.array([[b.size, b.alloc_time, b.free_time] for b in inst.blocks], np.int64)
    t0 = time.perf_counter()
    plan = M.solve_bestfit(inst)
    dt = time.perf_counter() - t0
    off = np.array([plan.offsets[b.id] for b in inst.blocks], np.int64)
    return {"name": name, "n": len(inst.blocks), "alignment": inst.alignment,
            "blocks_sha256": _sha(blocks), "offsets_sha256": _sha(off),
            "peak": int(plan.peak), "clique_lb": int(M.clique_lower_bound(inst)),
            "ref_s": round(dt, 2)}


def lstm_one(layers: int, alignment: int = 1) -> dict:
    """All 4096 profiles of BASELINE.json config 4 (workloads.py:74-126)."""
    import memplan as M
    spec = M.GenSpec(model="rnn", layers=layers, batch=64, seed=2024, variable_length=(10, 50))
    peaks, offs, rows, ns = [], [], [], []
    t0 = time.perf_counter()
    for ell in M.rnn_epoch_lengths(spec, 4096):
        inst = M.profile_to_instance(M.record(M.parse_trace(M.rnn_like_trace(spec, ell))),
                                     alignment=alignment)
        plan = M.solve_bestfit(inst)
        peaks.append(plan.peak)
        ns.append(len(inst.blocks))
        offs.extend(plan.offsets[b.id] for b in inst.blocks)
        rows.extend([b.size, b.alloc_time, b.free_time] for b in inst.blocks)
    dt = time.perf_counter() - t0
    return {"name": f"lstm_L{layers}" + (f"_a{alignment}" if alignment != 1 else ""),
            "alignment": alignment, "profiles": 4096, "blocks_total": int(sum(ns)),
            "n_per_profile": sorted(set(ns)),
            "blocks_sha256": _sha(np.array(rows, np.int64)),
            "offsets_sha256": _sha(np.array(offs, np.int64)),
            "peaks_sha256": _sha(np.array(peaks, np.int64)),
            "peaks_head": [int(p) for p in peaks[:16]], "peak_max": int(max(peaks)),
            "ref_s": round(dt, 2)}


def run(job: str) -> dict:
    if job.startswith("lstm_L"):
        parts = job[6:].split("_a")
        return lstm_one(int(parts[0]), int(parts[1]) if len(parts) > 1 else 1)
    return solve_one(job)


JOBS = ["lstm_L6", "lstm_L64", "lstm_L6_a512", "lstm_L64_a512",
        "uniform_1e5_s0", "cnn_1e5_s0", "walk_1e5_s0", "uniform_1e5_s1", "walk_1e5_s1",
        "cnn_1e6_s0", "uniform_1e6_s0", "walk_1e6_s0"]


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--jobs", type=int, default=7)
    ap.add_argument("--only", default="")
    ap.add_argument("--out", default=OUT)
    args = ap.parse_args()
    jobs = [j for j in JOBS if not args.only or j in args.only.split(",")]
    done = {}
    if os.path.exists(args.out):
        with open(args.out) as fh:
            done = {c["name"]: c for c in json.load(fh)["cases"]}
    jobs = [j for j in jobs if j not in done]
    # the 10^6 solves first: they bound the wall time
    jobs.sort(key=lambda j: "1e6" not in j)
    with mp_.Pool(min(args.jobs, max(1, len(jobs)))) as pool:
        for res in pool.imap_unordered(run, jobs):
            done[res["name"]] = res
            print(json.dumps(res), flush=True)
            with open(args.out, "w") as fh:
                json.dump({"generator": "tests/golden/make_huge_golden.py (reference memplan)",
                           "cases": [done[k] for k in sorted(done)]}, fh, indent=1)


if __name__ == "__main__":
    main()
