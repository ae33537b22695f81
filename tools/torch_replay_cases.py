"""Safety cases of the torch replay allocator (csrc/torch_alloc.cpp) on real
device memory, run in a fresh process (the pluggable allocator must be
installed before torch's first CUDA allocation).  Prints one JSON line of
named boolean checks plus the counters behind them; tests/
test_torch_replay_gpu.py asserts every check.

Cases:
  carried   a planned tensor held across an epoch boundary keeps its bytes
            while the next epoch runs (epoch reset used to let the
            next epoch's blocks overwrite it) and is freed without cudaFree
            of the region;
  growth    a request larger than planned is side-served, the next epoch
            boundary re-plans on the GPU (Arena.reoptimize, arena.py:303-322)
            into a larger region, and the grown request is then planned;
  reorder   planned [aG aA fA aB fG], run [aG(grown) aA fG aB fA]: B must not
            land on A while A is live (the grown block's free was
            never tick-checked);
  stream    a request on another stream is side-served on that stream;
  end       tensors made during replay outlive replay_end; the region is
            released only after the last of them is freed.
"""

from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

MB = 1 << 20


def main() -> None:
    import torch
    from paper_1804_10001_b200.torch_replay import TorchReplay

    rp = TorchReplay.install(alignment=512)
    dev = torch.device("cuda")
    torch.empty(1, device=dev)  # CUDA context + passthrough allocation
    torch.cuda.synchronize()
    f32 = dict(dtype=torch.float32, device=dev)
    n1 = MB // 4  # floats per MB
    out: dict = {}

    # ---------------- carried ----------------
    def step_a(v, keep=False):
        t1 = torch.full((n1,), v, **f32)
        t2 = torch.full((n1,), v + 1, **f32)
        del t1
        t3 = torch.full((n1,), v + 2, **f32)
        del t2
        if keep:
            return t3
        del t3
        return None

    with rp.recording():
        step_a(0.0)
    plan = rp.plan()
    rp.begin()
    rp.new_epoch()
    held = step_a(10.0, keep=True)
    torch.cuda.synchronize()
    held_addr = held.data_ptr()
    rp.new_epoch()
    step_a(20.0)
    extra = step_a(30.0, keep=True)  # beyond the plan: side-served extras
    torch.cuda.synchronize()
    out["carried_bytes_kept"] = bool(torch.all(held == 12.0).item())
    st = rp.stats()
    out["carried_live_counted"] = st["n_carried_live"] == 1
    del held, extra
    torch.cuda.synchronize()
    st = rp.stats()
    out["carried_released"] = st["n_carried_live"] == 0 and st["n_unknown_free"] == 0
    out["carried_plan_peak"] = plan.peak
    out["carried_addr_in_region"] = st["region_base"] <= held_addr < st["region_base"] + st["region_bytes"]
    rp.end()

    # ---------------- growth -> deferred re-plan ----------------
    rp2 = TorchReplay(alignment=512)

    def step_b(grow):
        x = torch.full((n1,), 1.0, **f32)
        y = torch.full(((2 if grow else 1) * n1,), 2.0, **f32)
        z = x + y[:n1]
        del x, y
        s = z.sum().item()
        del z
        return s

    with rp2.recording():
        step_b(False)
    p0 = rp2.plan()
    rp2.begin()
    rp2.new_epoch()
    s_grown = step_b(True)
    st1 = rp2.stats()
    rp2.new_epoch()  # re-plan here
    st2 = rp2.stats()
    side_before = st2["n_side"]
    s_again = step_b(True)
    st3 = rp2.stats()
    out["growth_side_served"] = st1["n_side"] >= 1
    out["growth_replanned"] = st2["n_replans"] == 1 and st2["plan_peak"] > p0.peak
    out["growth_region_grew"] = st2["region_bytes"] >= st2["plan_peak"] > p0.peak
    out["growth_then_planned"] = st3["n_side"] == side_before and st3["n_diverged"] == 0
    out["growth_values"] = s_grown == s_again == 3.0 * n1
    rp2.end()

    # ---------------- reorder ----------------
    rp3 = TorchReplay(alignment=512)
    with rp3.recording():
        g = torch.full((n1,), 1.0, **f32)       # aG
        a = torch.full((n1,), 2.0, **f32)       # aA
        del a                                    # fA
        b = torch.full((n1,), 3.0, **f32)       # aB (planned on A's offset)
        del g                                    # fG
        del b
    p3 = rp3.plan()
    off = p3.offsets
    out["reorder_plan_shares_offset"] = off[2] == off[3]
    rp3.begin()
    rp3.new_epoch()
    g = torch.full((2 * n1,), 1.0, **f32)       # aG, grown -> side
    a = torch.full((n1,), 7.0, **f32)           # aA (on plan)
    del g                                        # fG off its tick -> diverged
    b = torch.full((n1,), 9.0, **f32)           # aB must not alias A
    torch.cuda.synchronize()
    out["reorder_no_alias"] = bool(torch.all(a == 7.0).item()) and a.data_ptr() != b.data_ptr()
    del a, b
    out["reorder_diverged_counted"] = rp3.stats()["n_diverged"] >= 1
    rp3.end()

    # ---------------- stream ----------------
    rp4 = TorchReplay(alignment=512)

    def step_d():
        u = torch.full((n1,), 1.0, **f32)
        w = torch.full((n1,), 2.0, **f32)
        del u, w

    with rp4.recording():
        step_d()
    rp4.plan()
    rp4.begin()
    rp4.new_epoch()
    step_d()  # binds the default stream
    rp4.new_epoch()
    sd0 = rp4.stats()["n_side"]
    s2 = torch.cuda.Stream()
    with torch.cuda.stream(s2):
        step_d()
    torch.cuda.synchronize()
    out["stream_other_side_served"] = rp4.stats()["n_side"] - sd0 == 2
    rp4.end()

    # ---------------- end with live tensors ----------------
    rp5 = TorchReplay(alignment=512)
    with rp5.recording():
        step_d()
    rp5.plan()
    rp5.begin()
    rp5.new_epoch()
    keep = torch.full((n1,), 5.0, **f32)
    rp5.end()
    st = rp5.stats()
    out["end_region_retained"] = st["n_regions"] >= 1 and st["n_carried_live"] == 1
    torch.cuda.synchronize()
    out["end_tensor_intact"] = bool(torch.all(keep == 5.0).item())
    del keep
    torch.cuda.synchronize()
    st = rp5.stats()
    out["end_region_released"] = st["n_carried_live"] == 0 and st["n_unknown_free"] == 0
    out["final_stats"] = st
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
