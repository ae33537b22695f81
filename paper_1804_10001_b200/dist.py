"""Batched planning sharded over the GPUs of one node.

Traces are independent, so planning shards with no exchange: each rank
plans the traces that longest-processing-time-first (LPT) assignment gives
it, on its own GPU.  The only collective is the final gather of per-trace
offsets and peaks to rank 0 (grouped point-to-point send/recv; NCCL over
NVLink on GPUs, gloo in the CPU tests).  A single trace is never split: its
step chain is sequential ("replicas only" for single-trace planning).
"""

from __future__ import annotations

import heapq
from dataclasses import dataclass

import numpy as np


def trace_cost(n: int) -> float:
    """Planning cost estimate of an n-block trace: S ~ 3n steps, each
    touching a window that grows with n (the reference is O(n^2))."""
    return float(n) * float(n + 64)


def lpt_shards(costs, world: int) -> list:
    """Longest-processing-time-first assignment of traces to `world` ranks.
    Deterministic: ties broken by trace index, then rank index."""
    order = sorted(range(len(costs)), key=lambda t: (-costs[t], t))
    heap = [(0.0, r) for r in range(world)]
    shards = [[] for _ in range(world)]
    for t in order:
        load, r = heapq.heappop(heap)
        shards[r].append(t)
        heapq.heappush(heap, (load + costs[t], r))
    return [sorted(s) for s in shards]


@dataclass
class Batch:
    """T traces in CSR form (host int64 arrays)."""

    trace_ptr: np.ndarray
    alloc: np.ndarray
    free: np.ndarray
    size: np.ndarray

    @property
    def T(self) -> int:
        return len(self.trace_ptr) - 1

    def sizes(self) -> np.ndarray:
        return np.diff(self.trace_ptr)

    def subset(self, traces) -> "Batch":
        tp = [0]
        parts = []
        for t in traces:
            a, b = int(self.trace_ptr[t]), int(self.trace_ptr[t + 1])
            parts.append((a, b))
            tp.append(tp[-1] + (b - a))
        idx = np.concatenate([np.arange(a, b) for a, b in parts]) if parts else \
            np.zeros(0, np.int64)
        return Batch(np.asarray(tp, np.int64), self.alloc[idx], self.free[idx], self.size[idx])


def concat_batch(instances_cols) -> Batch:
    sizes = [len(c[0]) for c in instances_cols]
    tp = np.zeros(len(sizes) + 1, np.int64)
    np.cumsum(sizes, out=tp[1:])
    cat = lambda i: (np.concatenate([c[i] for c in instances_cols])  # noqa: E731
                     if instances_cols else np.zeros(0, np.int64))
    return Batch(tp, cat(0), cat(1), cat(2))


def gather_to_root(local_traces, local_offsets: np.ndarray, local_peaks: np.ndarray,
                   batch: Batch, device=None):
    """Gather every rank's per-trace results to rank 0.

    Returns (offsets CSR-aligned with `batch`, peaks[T]) on rank 0 and
    (None, None) elsewhere.  Payload = 8*sum(n_i) + 8*T bytes.  Uses
    torch.distributed point-to-point ops batched into one group call."""
    import torch
    import torch.distributed as dist

    world, rank = dist.get_world_size(), dist.get_rank()
    dev = device if device is not None else torch.device("cpu")
    counts = torch.tensor([len(local_traces), len(local_offsets)], dtype=torch.int64, device=dev)
    allc = [torch.zeros(2, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(allc, counts)
    sizes = [(int(c[0]), int(c[1])) for c in allc]
    if rank != 0:
        payload = torch.from_numpy(np.concatenate([
            np.asarray(local_traces, np.int64), local_peaks.astype(np.int64),
            local_offsets.astype(np.int64)])).to(dev)
        dist.batch_isend_irecv([dist.P2POp(dist.isend, payload, 0)])[0].wait()
        return None, None
    bufs, ops = {}, []
    for r in range(1, world):
        nt, nb = sizes[r]
        bufs[r] = torch.empty(2 * nt + nb, dtype=torch.int64, device=dev)
        ops.append(dist.P2POp(dist.irecv, bufs[r], r))
    for req in (dist.batch_isend_irecv(ops) if ops else []):
        req.wait()
    offsets = np.zeros(len(batch.alloc), np.int64)
    peaks = np.zeros(batch.T, np.int64)

    def scatter(traces, pk, off):
        pos = 0
        for i, t in enumerate(traces):
            a, b = int(batch.trace_ptr[t]), int(batch.trace_ptr[t + 1])
            offsets[a:b] = off[pos:pos + (b - a)]
            peaks[t] = pk[i]
            pos += b - a

    scatter(list(local_traces), local_peaks, local_offsets)
    for r in range(1, world):
        nt, nb = sizes[r]
        v = bufs[r].cpu().numpy()
        scatter(v[:nt].tolist(), v[nt:2 * nt], v[2 * nt:])
    return offsets, peaks


def gather_device(local_traces, d_offsets, d_peaks):
    """Device-resident gather for the benchmark/serving path: every rank's
    (trace ids, peaks, offsets) int64 tensors land on rank 0's device in one
    grouped send/recv round (NCCL over NVLink).  Returns the list of
    per-rank payload tensors on rank 0, None elsewhere."""
    import torch
    import torch.distributed as dist

    world, rank = dist.get_world_size(), dist.get_rank()
    dev = d_offsets.device
    if dist.get_backend() != "nccl":  # gloo moves host tensors
        dev = torch.device("cpu")
        d_offsets, d_peaks = d_offsets.cpu(), d_peaks.cpu()
    ids = torch.as_tensor(local_traces, dtype=torch.int64, device=dev)
    payload = torch.cat([ids, d_peaks.to(torch.int64), d_offsets.to(torch.int64)])
    n = torch.tensor([payload.numel()], dtype=torch.int64, device=dev)
    alln = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(alln, n)
    if rank != 0:
        for req in dist.batch_isend_irecv([dist.P2POp(dist.isend, payload, 0)]):
            req.wait()
        return None
    bufs = [payload] + [torch.empty(int(alln[r].item()), dtype=torch.int64, device=dev)
                        for r in range(1, world)]
    ops = [dist.P2POp(dist.irecv, bufs[r], r) for r in range(1, world)]
    for req in (dist.batch_isend_irecv(ops) if ops else []):
        req.wait()
    return bufs


def plan_sharded(batch: Batch, planner, device=None):
    """Plan `batch` across all ranks of the default process group.

    `planner(sub_batch) -> (offsets, peaks)` plans one rank's traces (the GPU
    planner in production; tests may inject a stand-in).  Every rank must
    pass the same batch.  Returns the gathered results on rank 0."""
    import torch.distributed as dist

    world, rank = dist.get_world_size(), dist.get_rank()
    shards = lpt_shards([trace_cost(int(n)) for n in batch.sizes()], world)
    mine = shards[rank]
    sub = batch.subset(mine)
    off, pk = planner(sub)
    return gather_to_root(mine, np.asarray(off), np.asarray(pk), batch, device)
