"""Profile-guided allocation for a real PyTorch training iteration (paper §4):
record one iteration's allocation trace through memplan's
CUDAPluggableAllocator hooks, plan it on the GPU (best-fit, bit-exact with
the reference), then replay later iterations out of ONE cudaMalloc'd region
of plan.peak bytes.

    python tools/torch_model_replay.py --alloc memplan   # record -> plan -> replay
    python tools/torch_model_replay.py --alloc caching   # PyTorch caching allocator
    python tools/torch_model_replay.py --alloc all       # both, one JSON line

The memplan run checks that replayed iterations compute bit-identical loss
and gradients to a passthrough (cudaMalloc-per-tensor) iteration on the same
weights and batch, and counts requests the plan did not cover.  The caching
run reports the allocator's own peak (max_memory_allocated / reserved) for
the same iteration, so the two peaks can be compared.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def make_model(torch, width: int):
    nn = torch.nn
    layers = []
    c = 3
    for i, w in enumerate([width, width, 2 * width, 2 * width, 4 * width, 4 * width]):
        layers += [nn.Conv2d(c, w, 3, padding=1, bias=False), nn.BatchNorm2d(w), nn.ReLU()]
        if i % 2 == 1:
            layers.append(nn.MaxPool2d(2))
        c = w
    layers += [nn.AdaptiveAvgPool2d(1), nn.Flatten(), nn.Linear(c, 100)]
    return nn.Sequential(*layers)


def iteration(torch, model, x, y):
    """Forward + backward; everything allocated inside is freed inside."""
    for p in model.parameters():
        p.grad.zero_()
    out = model(x)
    loss = torch.nn.functional.cross_entropy(out, y)
    loss.backward()
    lv = loss.detach().clone()
    g = torch.cat([p.grad.reshape(-1) for p in model.parameters()]).clone()
    del out, loss
    return lv, g


def run(alloc: str, batch: int, width: int, iters: int) -> dict:
    import torch
    replay = None
    if alloc == "memplan":
        from paper_1804_10001_b200.torch_replay import TorchReplay
        replay = TorchReplay.install(alignment=512)
    torch.backends.cudnn.benchmark = False
    torch.backends.cudnn.deterministic = True
    torch.use_deterministic_algorithms(True, warn_only=True)
    torch.manual_seed(0)
    dev = torch.device("cuda")
    model = make_model(torch, width).to(dev)
    x = torch.randn(batch, 3, 64, 64, device=dev)
    y = torch.randint(0, 100, (batch,), device=dev)
    for p in model.parameters():
        p.grad = torch.zeros_like(p)
    # warm-up iterations: cuDNN/cuBLAS handles, workspaces, lazy modules
    for _ in range(2):
        iteration(torch, model, x, y)
    torch.cuda.synchronize()
    out = {"allocator": alloc, "batch": batch, "width": width}
    if alloc == "caching":
        torch.cuda.reset_peak_memory_stats()
        base = torch.cuda.memory_allocated()
        iteration(torch, model, x, y)
        torch.cuda.synchronize()
        out["iteration_peak_bytes"] = torch.cuda.max_memory_allocated() - base
        out["reserved_bytes"] = torch.cuda.memory_reserved()
        t0 = time.perf_counter()
        for _ in range(iters):
            iteration(torch, model, x, y)
        torch.cuda.synchronize()
        out["ms_per_iteration"] = 1e3 * (time.perf_counter() - t0) / iters
        return out
    import paper_1804_10001_b200 as mp
    import numpy as np
    # reference iteration in passthrough mode (cudaMalloc per tensor)
    ref_loss, ref_grad = iteration(torch, model, x, y)
    torch.cuda.synchronize()
    # record one iteration (profiler.py clock discipline over the hooks)
    with replay.recording():
        iteration(torch, model, x, y)
    if os.environ.get("MEMPLAN_SAVE_TRACE"):
        kinds = np.array([0 if e.kind == "alloc" else 1 for e in replay.events], np.int32)
        values = np.array([e.size if e.kind == "alloc" else e.ref for e in replay.events])
        np.savez(os.environ["MEMPLAN_SAVE_TRACE"], kinds=kinds, values=values)
    t0 = time.perf_counter()
    plan = replay.plan()  # GPU planner
    out["plan_ms"] = 1e3 * (time.perf_counter() - t0)
    inst = replay.instance
    out["trace_events"] = len(replay.events)
    out["planned_blocks"] = len(inst.blocks)
    out["plan_peak_bytes"] = plan.peak
    out["clique_lower_bound_bytes"] = mp.clique_lower_bound(inst)
    out["pool_peak_bytes"] = mp.simulate_pool(replay.events).peak
    replay.begin()
    # replay: each iteration is one epoch of the arena
    equal = True
    for _ in range(2):
        replay.new_epoch()
        lv, g = iteration(torch, model, x, y)
        torch.cuda.synchronize()
        equal = equal and bool(torch.equal(lv, ref_loss) and torch.equal(g, ref_grad))
        del lv, g
    t0 = time.perf_counter()
    for _ in range(iters):
        replay.new_epoch()
        iteration(torch, model, x, y)
    torch.cuda.synchronize()
    out["ms_per_iteration"] = 1e3 * (time.perf_counter() - t0) / iters
    st = replay.stats()
    out["requests_from_plan"] = st["n_planned"]
    out["requests_outside_plan"] = st["n_side"]
    out["epochs_off_profile"] = st["n_diverged"]
    out["replans"] = st["n_replans"]
    out["replay_bit_identical"] = equal
    replay.new_epoch()
    replay.end()
    return out


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--alloc", default="all", choices=["all", "memplan", "caching"])
    p.add_argument("--batch", type=int, default=64)
    p.add_argument("--width", type=int, default=64)
    p.add_argument("--iters", type=int, default=10)
    a = p.parse_args()
    if a.alloc != "all":
        print(json.dumps(run(a.alloc, a.batch, a.width, a.iters)), flush=True)
        return
    res = {}
    for al in ("memplan", "caching"):
        r = subprocess.run([sys.executable, os.path.abspath(__file__), "--alloc", al, "--batch",
                            str(a.batch), "--width", str(a.width), "--iters", str(a.iters)],
                           capture_output=True, text=True, timeout=900)
        lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
        res[al] = json.loads(lines[-1]) if lines else {"error": r.stderr[-800:]}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
