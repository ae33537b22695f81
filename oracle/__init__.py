"""ORACLE — test infrastructure only; never imported by the product package.

CPU restatement of the reference `memplan` hot path (bestfit.py:276-309,
verifier.py:44-81, core.py:252-268), compiled from ``oracle/memplan_oracle.c``
into ``oracle/_build/liboracle.so``.  Only ``tests/``,
``__graft_entry__.smoke()`` (as the checker) and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module.

Parity is pinned against golden vectors produced by the reference itself
(``tests/golden/make_golden.py``; checked by ``tests/test_oracle.py``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None


class OrcStats(ctypes.Structure):
    _fields_ = [("steps", ctypes.c_int64), ("lifts", ctypes.c_int64),
                ("sum_wlive", ctypes.c_int64), ("max_lines", ctypes.c_int64)]


class OrcVerifyOut(ctypes.Structure):
    _fields_ = [("n_violations", ctypes.c_int64), ("peak", ctypes.c_int64),
                ("offsets_ok", ctypes.c_int32), ("pad", ctypes.c_int32),
                ("used_lo", ctypes.c_uint64), ("used_hi", ctypes.c_uint64)]


VIOL_DTYPE = np.dtype([("i", np.int64), ("j", np.int64),
                       ("overlap_bytes", np.int64), ("overlap_ticks", np.int64)])


def build() -> str:
    """Compile the oracle (gcc) if the shared object is missing or stale."""
    src = os.path.join(_HERE, "memplan_oracle.c")
    if (not os.path.exists(_SO)) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        l = ctypes.CDLL(_SO)
        p64 = ctypes.POINTER(ctypes.c_int64)
        l.orc_solve_bestfit.argtypes = [ctypes.c_int64, p64, p64, p64, p64, p64,
                                        ctypes.POINTER(OrcStats)]
        l.orc_solve_bestfit.restype = ctypes.c_int
        l.orc_verify.argtypes = [ctypes.c_int64, p64, p64, p64, p64,
                                 ctypes.POINTER(OrcVerifyOut), ctypes.c_void_p,
                                 ctypes.c_int64]
        l.orc_verify.restype = ctypes.c_int
        l.orc_clique_lb.argtypes = [ctypes.c_int64, p64, p64, p64]
        l.orc_clique_lb.restype = ctypes.c_int64
        _lib = l
    return _lib


def _i64(a):
    a = np.ascontiguousarray(a, dtype=np.int64)
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def solve_bestfit(alloc, free, size, with_stats: bool = False):
    """Oracle plan: (offsets int64[n] in id order, peak[, stats dict])."""
    a, pa = _i64(alloc)
    f, pf = _i64(free)
    s, ps = _i64(size)
    n = len(a)
    off = np.zeros(n, dtype=np.int64)
    peak = ctypes.c_int64(0)
    st = OrcStats()
    rc = lib().orc_solve_bestfit(n, pa, pf, ps,
                                 off.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                 ctypes.byref(peak), ctypes.byref(st))
    if rc == 1:
        raise AssertionError("best-fit loop exceeded its iteration bound")
    if rc == 2:
        raise RuntimeError("IllegalLift")
    if with_stats:
        return off, peak.value, {"steps": st.steps, "lifts": st.lifts,
                                 "sum_wlive": st.sum_wlive, "max_lines": st.max_lines}
    return off, peak.value


def verify(alloc, free, size, offsets, viol_cap: int = 1 << 16):
    """Oracle verification: dict with n_violations, violations (sorted by
    pair), peak_recomputed, offsets_ok, used (exact int)."""
    a, pa = _i64(alloc)
    f, pf = _i64(free)
    s, ps = _i64(size)
    o, po = _i64(offsets)
    out = OrcVerifyOut()
    viol = np.zeros(viol_cap, dtype=VIOL_DTYPE)
    lib().orc_verify(len(a), pa, pf, ps, po, ctypes.byref(out),
                     viol.ctypes.data_as(ctypes.c_void_p), viol_cap)
    k = min(out.n_violations, viol_cap)
    return {
        "n_violations": out.n_violations,
        "violations": [(int(v["i"]), int(v["j"]), int(v["overlap_bytes"]),
                        int(v["overlap_ticks"])) for v in viol[:k]],
        "peak_recomputed": out.peak,
        "offsets_ok": bool(out.offsets_ok),
        "used": (out.used_hi << 64) | out.used_lo,
    }


def clique_lb(alloc, free, size) -> int:
    a, pa = _i64(alloc)
    f, pf = _i64(free)
    s, ps = _i64(size)
    return int(lib().orc_clique_lb(len(a), pa, pf, ps))
