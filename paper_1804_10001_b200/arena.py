"""Replay arena — drop-in for ``memplan.arena`` (Arena, replay_events,
PoolAllocator, simulate_pool).

The state machine lives in C++ (``csrc/arena.cpp``, C ABI ``mp_arena_*``):
the k-th monitored allocation of an epoch receives ``base + offset[k]``;
growth re-plans on the GPU (reference arena.py:303-322).  Opening an arena
verifies the plan with the GPU validator first, like arena.py:165.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N
from .core import DsaInstance, MemplanError, Plan, Provenance


class InvalidPlan(MemplanError):
    """Arena opened over a plan that fails verification."""


class ExtraRequest(MemplanError):
    """More monitored allocations than the plan covers (strict mode)."""


class AllocAfterClose(MemplanError):
    """Allocation from a closed arena."""


class LiveBlocksAtReset(MemplanError):
    """Reset with monitored blocks still live (strict mode)."""


class UnknownId(MemplanError):
    """Free of an allocation reference that was never served."""


class OutOfMemory(MemplanError):
    """Pool bump allocation beyond a finite capacity, even after a flush."""


def _check(rc: int) -> None:
    from .bestfit import check
    check(rc)


_KIND = {"alloc": 0, "free": 1, "interrupt": 2, "resume": 3}


def encode_events(events) -> tuple[np.ndarray, np.ndarray]:
    """TraceEvent list -> (kinds int32, values int64) for the C ABI."""
    n = len(events)
    kinds = np.empty(n, dtype=np.int32)
    values = np.zeros(n, dtype=np.int64)
    for i, ev in enumerate(events):
        k = _KIND.get(ev.kind)
        if k is None:
            raise MemplanError(f"unknown event kind {ev.kind!r}")
        kinds[i] = k
        values[i] = ev.size if k == 0 else ev.ref
    return kinds, values


class PoolAllocator:
    """Dynamic pool baseline (reference arena.py:59-129) backed by C++."""

    def __init__(self, capacity: int | None = None):
        self.capacity = capacity
        h = N.VP()
        _check(N.lib().mp_pool_create(-1 if capacity is None else capacity, ctypes.byref(h)))
        self._h = h
        self._owner = None

    @classmethod
    def _borrow(cls, handle, owner) -> "PoolAllocator":
        """View of a pool owned by someone else (the arena's fallback)."""
        p = cls.__new__(cls)
        p.capacity = None
        p._h = N.VP(handle)
        p._owner = owner  # keeps the owning arena alive; never destroyed here
        return p

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and getattr(self, "_owner", None) is None:
            N.lib().mp_pool_destroy(h)
        self._h = None

    def _stats(self):
        vals = [ctypes.c_int64() for _ in range(4)]
        N.lib().mp_pool_stats(self._h, *[ctypes.byref(v) for v in vals])
        return [v.value for v in vals]

    @property
    def peak(self) -> int:
        return self._stats()[0]

    @property
    def cursor(self) -> int:
        return self._stats()[1]

    @property
    def last_ref(self) -> int:
        return self._stats()[3]

    def alloc(self, size: int) -> int:
        addr, ref = ctypes.c_int64(), ctypes.c_int64()
        _check(N.lib().mp_pool_alloc(self._h, size, ctypes.byref(addr), ctypes.byref(ref)))
        return addr.value

    def free(self, ref: int) -> None:
        _check(N.lib().mp_pool_free(self._h, ref))

    def live_bytes(self) -> int:
        return self._stats()[2]


class Arena:
    """Serves one sequential request stream against a static plan.

    Same constructor, methods and attributes as the reference Arena
    (arena.py:146-322); ``mode`` is "strict" or "lenient"."""

    def __init__(self, plan: Plan, instance: DsaInstance, base: int = 0,
                 mode: str = "lenient", device: int = 0):
        if mode not in ("strict", "lenient"):
            raise ValueError(f"mode must be 'strict' or 'lenient', got {mode!r}")
        from .verifier import verify_plan
        report = verify_plan(instance, plan)
        if not report.valid:
            raise InvalidPlan(f"plan fails verification ({len(report.violations)} violations)")
        self.base = base
        self.mode = mode
        self.device = device
        n = len(instance.blocks)
        if n:
            a, f, s = instance.arrays()
        else:
            a = f = s = np.zeros(0, np.int64)
        offs = np.array([plan.offsets[b] for b in range(1, n + 1)], dtype=np.int64)
        h = N.VP()
        _check(N.lib().mp_arena_open(N.ptr(s), N.ptr(a), N.ptr(f), N.ptr(offs), n, plan.peak,
                                     base, instance.alignment, 1 if mode == "strict" else 0,
                                     device, ctypes.byref(h)))
        self._h = h
        self._plan = plan
        self._plan_version = 0
        # the arena's own pool (reference: a PoolAllocator, arena.py:172)
        self.fallback = PoolAllocator._borrow(N.lib().mp_arena_pool(h), self)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            N.lib().mp_arena_close_handle(h)
            self._h = None

    # ---- state -----------------------------------------------------------
    def _state(self) -> N.ArenaState:
        st = N.ArenaState()
        N.lib().mp_arena_get_state(self._h, ctypes.byref(st))
        return st

    def _tables(self):
        n = self._state().n_blocks
        off = np.zeros(n, np.int64)
        sz = np.zeros(n, np.int64)
        N.lib().mp_arena_get_plan(self._h, N.ptr(off), N.ptr(sz), None, None)
        return off, sz

    @property
    def plan(self) -> Plan:
        st = self._state()
        if st.plan_version != self._plan_version:
            off, _ = self._tables()
            self._plan = Plan(offsets=dict(zip(range(1, len(off) + 1), off.tolist())),
                              peak=st.plan_peak, provenance=Provenance.BESTFIT)
            self._plan_version = st.plan_version
        return self._plan

    @property
    def lam(self) -> int:
        return self._state().lam

    @property
    def interrupted_depth(self) -> int:
        return self._state().depth

    @property
    def reopt_count(self) -> int:
        return self._state().reopt_count

    @property
    def forced_closes(self) -> int:
        return self._state().forced_closes

    def live_blocks(self) -> dict:
        k = self._state().n_live
        ids = np.zeros(k, np.int64)
        addrs = np.zeros(k, np.uint64)
        sizes = np.zeros(k, np.int64)
        N.lib().mp_arena_get_live(self._h, N.ptr(ids), N.ptr(addrs), N.ptr(sizes))
        return {int(i): (int(a), int(s)) for i, a, s in zip(ids, addrs, sizes)}

    def observed_sizes(self) -> dict:
        n = self._state().n_blocks
        obs = np.zeros(n, np.int64)
        N.lib().mp_arena_get_observed(self._h, N.ptr(obs))
        return {i + 1: int(v) for i, v in enumerate(obs) if v > 0}

    def expected_sizes(self) -> dict:
        _, sz = self._tables()
        return {i + 1: int(v) for i, v in enumerate(sz)}

    def peak_usage(self) -> int:
        st = self._state()
        return st.plan_peak + st.pool_peak

    # ---- operations ------------------------------------------------------
    def interrupt(self) -> None:
        _check(N.lib().mp_arena_interrupt(self._h))

    def resume(self) -> None:
        _check(N.lib().mp_arena_resume(self._h))

    def close(self) -> None:
        _check(N.lib().mp_arena_close(self._h))

    def alloc(self, size: int) -> int:
        addr = ctypes.c_uint64()
        _check(N.lib().mp_arena_alloc(self._h, size, ctypes.byref(addr)))
        return addr.value

    def free(self, ref: int) -> None:
        _check(N.lib().mp_arena_free(self._h, ref))

    def reset(self) -> None:
        _check(N.lib().mp_arena_reset(self._h))

    def reoptimize(self) -> Plan:
        _check(N.lib().mp_arena_reoptimize(self._h))
        return self.plan

    def replay_arrays(self, kinds: np.ndarray, values: np.ndarray) -> np.ndarray:
        kinds = np.ascontiguousarray(kinds, dtype=np.int32)
        values = np.ascontiguousarray(values, dtype=np.int64)
        out = np.zeros(int((kinds == 0).sum()), dtype=np.uint64)
        got = ctypes.c_int64()
        rc = N.lib().mp_arena_replay(self._h, N.ptr(kinds), N.ptr(values), len(kinds),
                                     N.ptr(out), ctypes.byref(got))
        _check(rc)
        return out[:got.value]


def replay_events(arena: Arena, events) -> list:
    """Drive one epoch's events through the arena; addresses served to the
    allocations in order.  Does not reset (reference arena.py:325-340).
    Events before an unknown kind are applied before it raises, as in the
    reference's event-by-event loop."""
    bad = next((i for i, ev in enumerate(events) if ev.kind not in _KIND), None)
    kinds, values = encode_events(events if bad is None else events[:bad])
    out = [int(a) for a in arena.replay_arrays(kinds, values)]
    if bad is not None:
        raise MemplanError(f"unknown event kind {events[bad].kind!r}")
    return out


def simulate_pool(events, pool: PoolAllocator | None = None) -> PoolAllocator:
    """Run a trace through the pool baseline (reference arena.py:343-364)."""
    if pool is None:
        pool = PoolAllocator()
    refs = []
    for ev in events:
        if ev.kind == "alloc":
            if ev.size == 0:
                refs.append(0)
            else:
                pool.alloc(ev.size)
                refs.append(pool.last_ref)
        elif ev.kind == "free":
            if ev.ref < 1 or ev.ref > len(refs):
                raise UnknownId(f"free of unknown allocation {ev.ref}")
            if refs[ev.ref - 1]:
                pool.free(refs[ev.ref - 1])
    return pool


def simulate_pool_peak(events, capacity: int | None = None) -> int:
    """Fast path: the pool baseline's peak over a whole trace in one C call."""
    kinds, values = encode_events(events)
    peak = ctypes.c_int64()
    _check(N.lib().mp_simulate_pool(N.ptr(kinds), N.ptr(values), len(kinds),
                                    -1 if capacity is None else capacity, ctypes.byref(peak)))
    return peak.value
