"""Best-fit offset planning on the GPU — drop-in for ``memplan.solve_bestfit``.

The reference heuristic (bestfit.py:276-309, paper §3.2) runs as the
sm_100a planner kernels in ``csrc/plan.cu`` behind the C ABI
``mp_plan_bestfit`` / ``mp_plan_bestfit_batched``.  Results are bit-exact
with the reference: same offsets per block id, same peak.

There is no CPU path: without the built library or a CUDA device these
functions raise.
"""

from __future__ import annotations

import ctypes
from typing import Sequence

import numpy as np

from . import _native as N
from .core import DsaInstance, MemplanError, Plan, Provenance


class IllegalLift(MemplanError):
    """lift_up on the only offset line (reference bestfit.py:34-35)."""


class ContainmentViolation(MemplanError):
    """A block placed on a line that does not contain its lifetime
    (reference bestfit.py:38-39)."""


class NoDevice(MemplanError):
    """No CUDA device: the planner has no CPU fallback."""


def check(rc: int) -> None:
    """Raise the reference exception class that matches a C-ABI status."""
    if rc == N.MP_OK:
        return
    msg = N.last_error()
    from . import arena as A
    from .core import DoubleFree, UnbalancedResume
    table = {
        N.MP_ERR_INVALID: ValueError,
        N.MP_ERR_ILLEGAL_LIFT: IllegalLift,
        N.MP_ERR_NO_DEVICE: NoDevice,
        N.MP_ERR_DOUBLE_FREE: DoubleFree,
        N.MP_ERR_UNKNOWN_ID: A.UnknownId,
        N.MP_ERR_EXTRA_REQUEST: A.ExtraRequest,
        N.MP_ERR_ALLOC_AFTER_CLOSE: A.AllocAfterClose,
        N.MP_ERR_LIVE_AT_RESET: A.LiveBlocksAtReset,
        N.MP_ERR_UNBALANCED_RESUME: UnbalancedResume,
        N.MP_ERR_INVALID_PLAN: A.InvalidPlan,
        N.MP_ERR_OUT_OF_MEMORY: A.OutOfMemory,
        N.MP_ERR_NEGATIVE_SIZE: ValueError,
    }
    if rc == N.MP_ERR_LOOP_BOUND:
        raise AssertionError(msg or "best-fit loop exceeded its iteration bound")
    exc = table.get(rc)
    if exc is None:
        raise RuntimeError(f"memplan_b200 CUDA failure: {msg}")
    raise exc(msg)


def plan_info() -> dict:
    """Diagnostics of the last plan call on this thread (steps, lifts, ...)."""
    info = N.PlanInfo()
    N.lib().mp_plan_last_info(ctypes.byref(info))
    out = {name: getattr(info, name) for name, _ in N.PlanInfo._fields_
           if name not in ("diag", "cycles")}
    out["cycles"] = {"choose": info.cycles[0], "query": info.cycles[1],
                     "update": info.cycles[2], "retire": info.cycles[3],
                     "lift_steps": info.cycles[4], "place_steps": info.cycles[5]}
    out["diag"] = {"scans": info.diag[0], "passes": info.diag[1], "segments": info.diag[2],
                   "edge_rows": info.diag[3]}
    return out


def solve_bestfit_arrays(alloc, free, size, *, device: int = 0, stream: int = 0,
                         flags: int = 0) -> tuple[np.ndarray, int]:
    """Array fast path: int64 columns in id order -> (offsets[n], peak).

    Inputs must already satisfy the DsaInstance invariants (sizes >= 1 and
    aligned, 0 <= alloc < free); they are trusted like the reference's
    solver trusts its instance."""
    a, f, s = N.as_i64(alloc), N.as_i64(free), N.as_i64(size)
    n = len(a)
    if not (len(f) == n and len(s) == n):
        raise ValueError("alloc, free and size must have equal length")
    off = np.empty(n, dtype=np.int64)
    peak = np.zeros(1, dtype=np.int64)
    rc = N.lib().mp_plan_bestfit(N.ptr(a), N.ptr(f), N.ptr(s), n, N.ptr(off), N.ptr(peak),
                                 flags, device, stream or None)
    check(rc)
    return off, int(peak[0])


def solve_bestfit_device(alloc_d, free_d, size_d, offsets_d, peak_d, n: int, *,
                         device: int = 0, stream: int = 0, flags: int = 0) -> None:
    """Device-pointer path: all five arguments are device addresses (ints)
    of int64 buffers already resident in HBM."""
    rc = N.lib().mp_plan_bestfit(alloc_d, free_d, size_d, n, offsets_d, peak_d,
                                 flags | N.MP_DEVICE_PTRS, device, stream or None)
    check(rc)


def solve_bestfit(instance: DsaInstance) -> Plan:
    """Pack all blocks with the best-fit skyline heuristic on the GPU.

    Same contract as the reference: deterministic, offsets keyed by block
    id, peak = max(offset + size), provenance BESTFIT."""
    n = len(instance.blocks)
    a, f, s = instance.arrays()
    off, peak = solve_bestfit_arrays(a, f, s)
    return Plan(offsets=dict(zip(range(1, n + 1), off.tolist())), peak=peak,
                provenance=Provenance.BESTFIT)


def solve_bestfit_batched_arrays(trace_ptr, alloc, free, size, *, device: int = 0,
                                 stream: int = 0, flags: int = 0):
    """T independent traces in CSR form -> (offsets CSR-aligned, peaks[T])."""
    tp = N.as_i64(trace_ptr)
    a, f, s = N.as_i64(alloc), N.as_i64(free), N.as_i64(size)
    T = len(tp) - 1
    off = np.empty(len(a), dtype=np.int64)
    peaks = np.zeros(max(T, 0), dtype=np.int64)
    rc = N.lib().mp_plan_bestfit_batched(N.ptr(tp), N.ptr(a), N.ptr(f), N.ptr(s), T,
                                         N.ptr(off), N.ptr(peaks), flags, device,
                                         stream or None)
    check(rc)
    return off, peaks


class PlanPipe:
    """Pipelined batched planning from host arrays (`mp_pipe_*`): while the
    GPU plans batch k, batch k+1 uploads and batch k-1 downloads.  Each
    `submit` returns a ticket; `wait(ticket)` returns that batch's
    (offsets, peaks), equal to `solve_bestfit_batched_arrays` on the same
    inputs.  Inputs are kept referenced until their ticket is waited for;
    page-locked arrays (torch `pin_memory`) let the copies run
    asynchronously.  At most two batches are in flight: a third submit
    waits for the first one's results."""

    def __init__(self, device: int = 0):
        self._lib = N.lib()
        self._p = self._lib.mp_pipe_create(device)
        if not self._p:
            check(N.MP_ERR_NO_DEVICE)
        self._live = {}

    def submit(self, trace_ptr, alloc, free, size, *, offsets_out=None, peaks_out=None,
               flags: int = 0) -> int:
        tp = N.as_i64(trace_ptr)
        a, f, s = N.as_i64(alloc), N.as_i64(free), N.as_i64(size)
        T = len(tp) - 1
        off = np.empty(len(a), dtype=np.int64) if offsets_out is None else offsets_out
        pk = np.zeros(max(T, 0), dtype=np.int64) if peaks_out is None else peaks_out
        ticket = ctypes.c_int64(-1)
        rc = self._lib.mp_pipe_submit(self._p, N.ptr(tp), N.ptr(a), N.ptr(f), N.ptr(s), T,
                                      N.ptr(off), N.ptr(pk), flags, ctypes.byref(ticket))
        if ticket.value >= 0:
            self._live[ticket.value] = (tp, a, f, s, off, pk)
        check(rc)
        return ticket.value

    def wait(self, ticket: int):
        rc = self._lib.mp_pipe_wait(self._p, ticket)
        bufs = self._live.pop(ticket, None)
        check(rc)
        return bufs[4], bufs[5]

    def close(self) -> None:
        if self._p:
            self._lib.mp_pipe_destroy(self._p)
            self._p = None
            self._live.clear()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def solve_bestfit_batched(instances: Sequence[DsaInstance], *, device: int = 0) -> list[Plan]:
    """Plan many independent instances in one batched launch."""
    cols = [inst.arrays() for inst in instances]
    sizes = [len(c[0]) for c in cols]
    tp = np.zeros(len(cols) + 1, dtype=np.int64)
    np.cumsum(sizes, out=tp[1:])
    a = np.concatenate([c[0] for c in cols]) if cols else np.zeros(0, np.int64)
    f = np.concatenate([c[1] for c in cols]) if cols else np.zeros(0, np.int64)
    s = np.concatenate([c[2] for c in cols]) if cols else np.zeros(0, np.int64)
    off, peaks = solve_bestfit_batched_arrays(tp, a, f, s, device=device)
    plans = []
    for t, n in enumerate(sizes):
        seg = off[tp[t]:tp[t + 1]].tolist()
        plans.append(Plan(offsets=dict(zip(range(1, n + 1), seg)), peak=int(peaks[t]),
                          provenance=Provenance.BESTFIT))
    return plans


# host-side skyline inspection types (the reference's bestfit.py debug
# surface); the planner above never uses them
def __getattr__(name):
    if name in ("OffsetLine", "OffsetLineSet", "find_block", "_RemainingBlocks"):
        from . import skyline
        return getattr(skyline, name)
    raise AttributeError(name)
