"""Profile-guided allocation for a live PyTorch program (paper §4,
PAPER.md:400-454): record one iteration's allocation trace through the
library's ``torch.cuda.memory.CUDAPluggableAllocator`` hooks, plan it with
the GPU best-fit planner (bit-exact with ``memplan.solve_bestfit``), then
replay later iterations out of ONE cudaMalloc'd region of ``plan.peak``
bytes — request λ of an epoch gets ``region + offset[λ]``, the
``Arena.alloc`` rule (arena.py:227-254).

The reference package stops at the address arithmetic (its ``Arena`` hands
out integers); the rules that real memory adds are in
``csrc/torch_alloc.cpp``: side allocations for everything the plan does not
cover, the profile-clock guard against aliasing when a run leaves the
profiled order, blocks carried live across epoch boundaries, deferred
re-planning on growth (``Arena.reoptimize``, arena.py:303-322) at the next
epoch boundary, and one stream for planned placement.

    replay = TorchReplay.install()          # before the first CUDA allocation
    with replay.recording():
        step()                              # one profiled iteration
    plan = replay.plan()                    # GPU planner
    replay.begin()
    for _ in range(steps):
        replay.new_epoch()
        step()
    replay.end()
"""

from __future__ import annotations

import contextlib
import ctypes

import numpy as np

from . import _native as N
from .arena import Arena
from .bestfit import solve_bestfit
from .core import DsaInstance, Plan
from .profiler import alloc as ev_alloc
from .profiler import free as ev_free
from .profiler import profile_to_instance, record


def _check(rc: int) -> None:
    if rc != N.MP_OK:
        N.raise_for(rc)


class TorchReplay:
    """One process-wide replay allocator (torch has one allocator per
    process).  Use :meth:`install` to route torch's CUDA allocations through
    the hooks; it must run before torch allocates any CUDA memory."""

    _installed = None

    def __init__(self, alignment: int = 512, device: int = 0, mode: str = "lenient"):
        self.alignment = alignment
        self.device = device
        self.mode = mode
        self.events = []
        self.instance: DsaInstance | None = None
        self.arena: Arena | None = None
        self._active = False

    @classmethod
    def install(cls, alignment: int = 512, device: int = 0, mode: str = "lenient") -> "TorchReplay":
        import torch
        if cls._installed is None:
            pa = torch.cuda.memory.CUDAPluggableAllocator(N.LIB_PATH, "mp_torch_alloc",
                                                          "mp_torch_free")
            torch.cuda.memory.change_current_allocator(pa)
            cls._installed = pa
        return cls(alignment=alignment, device=device, mode=mode)

    # ---- profile (profiler.py:156-222 clock discipline over the hooks) ----
    @contextlib.contextmanager
    def recording(self):
        import torch
        lib = N.lib()
        torch.cuda.synchronize()
        _check(lib.mp_torch_set_mode(1, None))
        try:
            yield self
            torch.cuda.synchronize()
        finally:
            n = ctypes.c_int64()
            lib.mp_torch_get_trace(None, None, 0, ctypes.byref(n))
            kinds = np.zeros(n.value, np.int32)
            values = np.zeros(n.value, np.int64)
            lib.mp_torch_get_trace(N.ptr(kinds), N.ptr(values), n.value, ctypes.byref(n))
            _check(lib.mp_torch_set_mode(0, None))
        self.events = [ev_alloc(int(v)) if k == 0 else ev_free(int(v))
                       for k, v in zip(kinds.tolist(), values.tolist())]

    # ---- plan (bestfit.py:276-309 on the GPU) -----------------------------
    def plan(self) -> Plan:
        self.instance = profile_to_instance(record(self.events), alignment=self.alignment)
        plan = solve_bestfit(self.instance)
        self.arena = Arena(plan, self.instance, base=0, mode=self.mode, device=self.device)
        return plan

    # ---- replay ------------------------------------------------------------
    def begin(self) -> int:
        """Allocate the region and switch the hooks to replay; returns its base."""
        if self.arena is None:
            self.plan()
        base = ctypes.c_uint64()
        _check(N.lib().mp_torch_replay_begin(self.arena._h, self.device, ctypes.byref(base)))
        self._active = True
        return base.value

    def new_epoch(self) -> None:
        """Arena.reset (arena.py:273-291) at an iteration boundary; re-plans
        on the GPU first when the last epoch saw growth."""
        _check(N.lib().mp_torch_epoch_reset())

    def end(self) -> None:
        if self._active:
            _check(N.lib().mp_torch_replay_end())
            self._active = False

    @property
    def plan_now(self) -> Plan:
        return self.arena.plan

    def stats(self) -> dict:
        st = N.TorchStats()
        _check(N.lib().mp_torch_stats_ex(ctypes.byref(st)))
        return {k: getattr(st, k) for k, _ in N.TorchStats._fields_}
