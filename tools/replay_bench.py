"""Replay allocation cost (SURVEY §8(d) "Replay"): ns per allocation for the
same size sequence served by

  memplan   memplan's CUDAPluggableAllocator hooks in replay mode: every
            planned request gets base + offset[lambda] inside ONE
            cudaMalloc'd region of plan.peak bytes (north_star)
  caching   PyTorch's native CUDA caching allocator
  async     PyTorch's cudaMallocAsync backend
  carena    memplan's C-ABI arena alone (mp_arena_bench, no torch)
  floor     a pluggable allocator whose hooks only hand out distinct
            addresses (tools/replay/replay_ext.cpp floor_alloc/floor_free):
            the cost of torch's CUDAPluggableAllocator front end itself,
            i.e. the floor under any pluggable allocator

Every torch allocator is timed twice: raw_alloc/raw_delete from C++
(`ns_per_alloc`, the allocator path alone) and `torch.empty` from Python
(`torch_empty_ns_per_alloc`, what a user's tensor creation costs end to
end, Python dispatch included).

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


def _torch_empty_ns(torch, lib, kinds, values, reps: int) -> float:
    """Best epoch of the same sequence as torch.empty(size, uint8) calls from
    Python (tensor deleted at its free event): a user's end-to-end cost."""
    import time
    ev = list(zip(kinds.tolist(), values.tolist()))
    n_alloc = sum(1 for k, _ in ev if k == 0)
    best = float("inf")
    empty, u8, dev = torch.empty, torch.uint8, torch.device("cuda")
    for r in range(min(reps, 5) + 1):
        if lib is not None:
            assert lib.mp_torch_epoch_reset() == 0
        live = []
        t0 = time.perf_counter_ns()
        for k, v in ev:
            if k == 0:
                live.append(empty(v, dtype=u8, device=dev))
            elif k == 1:
                live[v - 1] = None
        t1 = time.perf_counter_ns()
        live.clear()
        if r:
            best = min(best, t1 - t0)
    return best / n_alloc


def run_child(alloc: str, layers: int, reps: int) -> dict:
    import numpy as np
    if alloc == "async":
        os.environ["PYTORCH_CUDA_ALLOC_CONF"] = "backend:cudaMallocAsync"
    import torch
    from paper_1804_10001_b200 import _native as N
    sys.path.insert(0, os.path.join(ROOT, "tools", "replay"))
    from build_ext import BUILD, import_built
    if alloc == "memplan":
        pa = torch.cuda.memory.CUDAPluggableAllocator(N.LIB_PATH, "mp_torch_alloc",
                                                      "mp_torch_free")
        torch.cuda.memory.change_current_allocator(pa)
    elif alloc == "floor":
        pa = torch.cuda.memory.CUDAPluggableAllocator(
            os.path.join(BUILD, "memplan_replay_ext.so"), "floor_alloc", "floor_free")
        torch.cuda.memory.change_current_allocator(pa)
    torch.cuda.init()
    torch.empty(1, device="cuda")  # materialise the allocator for device 0
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
    out["torch_empty_ns_per_alloc"] = _torch_empty_ns(torch, lib if alloc == "memplan" else None,
                                                      kinds, values, reps)
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
                                                      "carena", "floor"])
    p.add_argument("--layers", type=int, default=5000)
    p.add_argument("--reps", type=int, default=20)
    args = p.parse_args()
    if args.alloc != "all":
        print(json.dumps(run_child(args.alloc, args.layers, args.reps)), flush=True)
        return
    res = {}
    for a in ("carena", "memplan", "floor", "caching", "async"):
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
