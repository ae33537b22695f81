"""Multi-process (world_size 2, gloo, CPU) tests of the batched sharding and
the final gather.  The per-rank planner is the CPU oracle standing in for
the GPU kernel (this test covers the host-side distribution logic)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as tmp

from paper_1804_10001_b200 import dist as D


def test_lpt_shards_balanced_and_deterministic():
    costs = [D.trace_cost(n) for n in [100, 5, 5, 90, 40, 40, 10, 1]]
    s = D.lpt_shards(costs, 2)
    assert sorted(sum(s, [])) == list(range(8))
    loads = [sum(costs[t] for t in x) for x in s]
    assert max(loads) <= 1.35 * min(loads)
    assert s == D.lpt_shards(costs, 2)
    assert D.lpt_shards(costs, 1) == [list(range(8))]


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _make_batch():
    rng = np.random.default_rng(7)
    cols = []
    for _ in range(9):
        n = int(rng.integers(1, 300))
        a = rng.integers(0, 500, n)
        f = a + 1 + rng.integers(0, 60, n)
        s = rng.integers(1, 1000, n)
        cols.append((a.astype(np.int64), f.astype(np.int64), s.astype(np.int64)))
    return D.concat_batch(cols)


def _oracle_planner(sub):
    import oracle
    offs, peaks = [], []
    for t in range(sub.T):
        a, b = sub.trace_ptr[t], sub.trace_ptr[t + 1]
        o, p = oracle.solve_bestfit(sub.alloc[a:b], sub.free[a:b], sub.size[a:b])
        offs.append(o)
        peaks.append(p)
    return (np.concatenate(offs) if offs else np.zeros(0, np.int64)), np.asarray(peaks, np.int64)


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    batch = _make_batch()
    off, pk = D.plan_sharded(batch, _oracle_planner)
    if rank == 0:
        np.save(out + ".off.npy", off)
        np.save(out + ".pk.npy", pk)
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_gather_world2(tmp_path):
    out = str(tmp_path / "res")
    tmp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    batch = _make_batch()
    ref_off, ref_pk = _oracle_planner(batch)
    assert np.array_equal(np.load(out + ".off.npy"), ref_off)
    assert np.array_equal(np.load(out + ".pk.npy"), ref_pk)
