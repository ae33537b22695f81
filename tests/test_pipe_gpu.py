"""PlanPipe (`mp_pipe_*`): pipelined batched planning from host arrays must
return exactly what `solve_bestfit_batched_arrays` returns for each batch
(itself pinned to the C oracle), whatever the order of waits, with
page-locked or pageable inputs, through the oversize (chunked) path, and
after a rejected submit."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _batch(rng, sizes, seed):
    from paper_1804_10001_b200.workloads import uniform_arrays
    cols = [uniform_arrays(int(n), seed + i) for i, n in enumerate(sizes)]
    cols = [(a, f, ((s + 511) // 512) * 512) for a, f, s in cols]
    tp = np.zeros(len(cols) + 1, np.int64)
    np.cumsum([len(c[0]) for c in cols], out=tp[1:])
    return (tp,) + tuple(np.concatenate([c[j] for c in cols]) for j in range(3))


def _batches():
    rng = np.random.default_rng(5)
    return [
        _batch(rng, [13] * 500, 1),                    # fused, one-warp CTAs
        _batch(rng, rng.integers(1, 3000, 60), 2),     # fused, mixed widths
        _batch(rng, [20000] * 200, 3),                 # general K0 + batched planner
        _batch(rng, [50000], 4),                       # one large trace
        _batch(rng, [0, 0, 5], 5),                     # empty traces
    ]


def test_pipe_matches_batched_call():
    from paper_1804_10001_b200.bestfit import PlanPipe, solve_bestfit_batched_arrays
    bs = _batches()
    want = [solve_bestfit_batched_arrays(*b) for b in bs]
    with PlanPipe() as pipe:
        tickets = [pipe.submit(*b) for b in bs]
        for t, (wo, wp) in zip(tickets, want):
            off, pk = pipe.wait(t)
            assert np.array_equal(off, wo) and np.array_equal(pk, wp)
        # waits out of order, batches resubmitted
        tickets = [pipe.submit(*b) for b in bs[:2]]
        for t, (wo, wp) in zip(reversed(tickets), reversed(want[:2])):
            off, pk = pipe.wait(t)
            assert np.array_equal(off, wo) and np.array_equal(pk, wp)
    # and the batched call itself agrees with the oracle on sampled traces
    tp, a, f, s = bs[1]
    for t in range(0, len(tp) - 1, 7):
        lo, hi = tp[t], tp[t + 1]
        o, p = oracle.solve_bestfit(a[lo:hi], f[lo:hi], s[lo:hi])
        assert p == want[1][1][t] and np.array_equal(o, want[1][0][lo:hi])


def test_pipe_pinned_buffers_steady_stream():
    import torch
    from paper_1804_10001_b200.bestfit import PlanPipe, solve_bestfit_batched_arrays
    tp, a, f, s = _batches()[2]
    wo, wp = solve_bestfit_batched_arrays(tp, a, f, s)
    pin = [torch.from_numpy(x).pin_memory() for x in (a, f, s)]
    outs = [(torch.empty(len(a), dtype=torch.int64).pin_memory(),
             torch.empty(len(tp) - 1, dtype=torch.int64).pin_memory()) for _ in range(2)]
    with PlanPipe() as pipe:
        pending = []
        for k in range(6):
            o, p = outs[k % 2]
            if len(pending) == 2:
                off, pk = pipe.wait(pending.pop(0))
                assert np.array_equal(off, wo) and np.array_equal(pk, wp)
            pending.append(pipe.submit(tp, *(x.numpy() for x in pin), offsets_out=o.numpy(),
                                       peaks_out=p.numpy()))
        for t in pending:
            off, pk = pipe.wait(t)
            assert np.array_equal(off, wo) and np.array_equal(pk, wp)


def test_pipe_oversize_batches_chunk(monkeypatch):
    from paper_1804_10001_b200.bestfit import PlanPipe, solve_bestfit_batched_arrays
    bs = _batches()[:2]
    want = [solve_bestfit_batched_arrays(*b) for b in bs]
    monkeypatch.setenv("MEMPLAN_MAX_BATCH_BLOCKS", "4096")
    with PlanPipe() as pipe:
        tickets = [pipe.submit(*b) for b in bs]
        for t, (wo, wp) in zip(tickets, want):
            off, pk = pipe.wait(t)
            assert np.array_equal(off, wo) and np.array_equal(pk, wp)


def test_pipe_rejects_bad_batch_and_keeps_going():
    from paper_1804_10001_b200.bestfit import PlanPipe, solve_bestfit_batched_arrays
    tp, a, f, s = _batches()[0]
    wo, wp = solve_bestfit_batched_arrays(tp, a, f, s)
    bad = tp.copy()
    bad[3] = bad[2] - 1
    with PlanPipe() as pipe:
        with pytest.raises(ValueError):
            pipe.submit(bad, a, f, s)
        off, pk = pipe.wait(pipe.submit(tp, a, f, s))
        assert np.array_equal(off, wo) and np.array_equal(pk, wp)


def test_pipe_tickets_expire():
    from paper_1804_10001_b200.bestfit import PlanPipe
    tp = np.array([0, 3], np.int64)
    a, f, s = np.array([0, 1, 2]), np.array([2, 3, 4]), np.array([512, 512, 1024])
    with PlanPipe() as pipe:
        first = pipe.submit(tp, a, f, s)
        off0, pk0 = pipe.wait(first)
        for _ in range(1030):
            t = pipe.submit(tp, a, f, s)
            off, pk = pipe.wait(t)
            assert np.array_equal(off, off0) and np.array_equal(pk, pk0)
        with pytest.raises(ValueError):
            pipe.wait(first)
        with pytest.raises(ValueError):
            pipe.wait(t + 5)
