"""Replay allocation cost (SURVEY §8(d) "Replay"): ns per allocation for the
same size sequence served by

  memplan   memplan's CUDAPluggableAllocator hooks in replay mode: every
            planned request gets base + offset[lambda] inside ONE
            cudaMalloc'd region of plan.peak bytes (north_star)
  caching   PyTorch's native CUDA caching allocator
  async     PyTorch's cudaMallocAsync backend
  carena    memplan's C-ABI arena alone (mp_arena_bench, no torch)

The sequence is the hot cnn-like trace (GenSpec(model="cnn", layers=L,
seed=0), reference cli.py:213 style), 2L allocations per epoch, all epochs
identical; the best epoch of --reps is reported.  Each torch allocator needs
its own process (the allocator is fixed at CUDA initialisation), so

    python tools/replay_bench.py --alloc all

spawns one child per allocator and prints one JSON line with all of them.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _events(layers: int):
    import paper_1804_10001_b200 as mp
    from paper_1804_10001_b200.arena import encode_events
    events = mp.parse_trace(mp.cnn_like_trace(mp.GenSpec(model="cnn", layers=layers, seed=0)))
    kinds, values = encode_events(events)
    return mp, events, kinds, values


def run_child(alloc: str, layers: int, reps: int) -> dict:
    import numpy as np
    if alloc == "async":
        os.environ["PYTORCH_CUDA_ALLOC_CONF"] = "backend:cudaMallocAsync"
    import torch
    from paper_1804_10001_b200 import _native as N
    if alloc == "memplan":
        pa = torch.cuda.memory.CUDAPluggableAllocator(N.LIB_PATH, "mp_torch_alloc",
                                                      "mp_torch_free")
        torch.cuda.memory.change_current_allocator(pa)
    torch.cuda.init()
    torch.empty(1, device="cuda")  # materialise the allocator for device 0
    sys.path.insert(0, os.path.join(ROOT, "tools", "replay"))
    from build_ext import import_built
    ext = import_built()
    mp, events, kinds, values = _events(layers)
    n_alloc = int((kinds == 0).sum())
    tk, tv = torch.from_numpy(kinds), torch.from_numpy(values)
    out = {"allocator": alloc, "n_allocs_per_epoch": n_alloc, "layers": layers}
    lo = span = 0
    lib = N.lib()
    keep = []
    if alloc in ("memplan", "carena"):
        inst = mp.profile_to_instance(mp.record(events), alignment=512)
        plan = mp.solve_bestfit(inst)
        out["plan_peak_bytes"] = plan.peak
        out["pool_peak_bytes"] = mp.simulate_pool(events).peak
        if alloc == "memplan":
            # the one cudaMalloc'd region of plan.peak bytes; the arena is
            # rebased onto it and the hooks switch to replay mode
            arena = mp.Arena(plan, inst, base=0)
            keep.append(arena)
            base = ctypes.c_uint64()
            assert lib.mp_torch_replay_begin(arena._h, 0, ctypes.byref(base)) == 0
            lo, span = int(base.value), plan.peak
        else:
            arena = mp.Arena(plan, inst, base=0)
            ns = ctypes.c_double()
            assert lib.mp_arena_bench(arena._h, N.ptr(kinds), N.ptr(values), len(kinds), reps,
                                      ctypes.byref(ns)) == 0
            out["ns_per_alloc"] = ns.value
            return out
    if alloc == "memplan":
        # the hooks alone (C loop over mp_torch_alloc / mp_torch_free)
        hns = ctypes.c_double()
        assert lib.mp_torch_bench(N.ptr(kinds), N.ptr(values), len(kinds), reps,
                                  ctypes.byref(hns)) == 0
        out["hook_ns_per_alloc"] = hns.value
    best, outside = float("inf"), 0.0
    for r in range(reps + 2):  # two warm-up epochs
        if alloc == "memplan":
            assert lib.mp_torch_epoch_reset() == 0
        ns, outs = ext.replay_epoch(tk, tv, lo, span)
        if r >= 2:
            best = min(best, ns)
            outside = max(outside, outs)
    torch.cuda.synchronize()
    out["ns_per_alloc"] = best / n_alloc
    if alloc == "memplan":
        # placement check: the replayed addresses are exactly base + offset
        assert lib.mp_torch_epoch_reset() == 0
        addrs = np.asarray(ext.epoch_addresses(tk, tv), dtype=np.int64)
        st = arena.plan
        inst_offsets = np.array([st.offsets[b] for b in range(1, len(st.offsets) + 1)])
        out["addresses_match_plan"] = bool(np.array_equal(addrs - lo, inst_offsets))
        out["outside_region"] = int(outside)
        assert lib.mp_torch_replay_end() == 0
    return out


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--alloc", default="all", choices=["all", "memplan", "caching", "async",
                                                      "carena"])
    p.add_argument("--layers", type=int, default=5000)
    p.add_argument("--reps", type=int, default=20)
    args = p.parse_args()
    if args.alloc != "all":
        print(json.dumps(run_child(args.alloc, args.layers, args.reps)), flush=True)
        return
    res = {}
    for a in ("carena", "memplan", "caching", "async"):
        r = subprocess.run([sys.executable, os.path.abspath(__file__), "--alloc", a, "--layers",
                            str(args.layers), "--reps", str(args.reps)],
                           capture_output=True, text=True, timeout=600)
        line = [x for x in r.stdout.splitlines() if x.startswith("{")]
        if not line:
            err = r.stderr or ""
            at = err.find("Error")
            res[a] = {"error": err[max(0, at - 300):at + 500]}
        else:
            res[a] = json.loads(line[-1])
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
