"""Plan validation on the GPU — drop-in for ``memplan.verifier``.

``verify_plan`` (reference verifier.py:44-81) runs as the K3 validator
kernel (``csrc/verify.cu``): every pair of blocks with intersecting
lifetimes is checked for address overlap on the device, the peak and the
exact 128-bit sum of size*lifetime are reduced there; utilisation is the
exact-integer ratio computed here, so it is bit-identical to the
reference's ``used / (peak * span)`` on Python ints.
"""

from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .core import DsaInstance, MemplanError, MissingOffset, Plan


class ZeroBaseline(MemplanError):
    """reduction_vs against a zero peak (reference verifier.py:24-25)."""


@dataclass(frozen=True)
class Violation:
    pair: tuple
    overlap_bytes: int
    overlap_ticks: int


@dataclass(frozen=True)
class VerifyReport:
    valid: bool
    violations: tuple
    peak_recomputed: int
    capacity_ok: bool
    utilization: float


def _plan_offsets(instance: DsaInstance, plan: Plan) -> np.ndarray:
    offs = plan.offsets
    n = len(instance.blocks)
    for bid in range(1, n + 1):
        if bid not in offs:
            raise MissingOffset(f"plan has no offset for block {bid}")
    try:
        return np.fromiter((offs[bid] for bid in range(1, n + 1)), dtype=np.int64, count=n)
    except OverflowError as exc:
        raise ValueError("offsets must fit in int64 for the GPU validator") from exc


def verify_arrays(alloc, free, size, offsets, *, viol_cap: int = 4096, device: int = 0,
                  stream: int = 0) -> dict:
    """Array fast path: returns n_violations, violations [(i, j, bytes, ticks)]
    sorted by pair, peak_recomputed, offsets_ok and the exact integer `used`."""
    a, f, s, o = N.as_i64(alloc), N.as_i64(free), N.as_i64(size), N.as_i64(offsets)
    n = len(a)
    from .bestfit import check
    while True:
        rep = N.VerifyReportC()
        buf = np.zeros(max(viol_cap, 1), dtype=N.VIOLATION_DTYPE)
        rc = N.lib().mp_verify(N.ptr(a), N.ptr(f), N.ptr(s), N.ptr(o), n, ctypes.byref(rep),
                               N.ptr(buf), viol_cap, 0, device, stream or None)
        check(rc)
        if rep.n_violations <= viol_cap:
            break
        viol_cap = int(rep.n_violations)  # second pass collects every violation
    k = int(rep.n_violations)
    return {
        "n_violations": k,
        "violations": [(int(v["i"]), int(v["j"]), int(v["overlap_bytes"]),
                        int(v["overlap_ticks"])) for v in buf[:k]],
        "peak_recomputed": int(rep.peak_recomputed),
        "offsets_ok": bool(rep.offsets_ok),
        "used": (int(rep.used_hi) << 64) | int(rep.used_lo),
    }


def verify_plan(instance: DsaInstance, plan: Plan) -> VerifyReport:
    """Re-check a plan against its instance from first principles (GPU)."""
    offsets = _plan_offsets(instance, plan)
    a, f, s = instance.arrays()
    r = verify_arrays(a, f, s, offsets)
    peak = r["peak_recomputed"]
    span = int(f.max()) - int(a.min()) if len(a) else 0
    utilization = r["used"] / (peak * span) if peak > 0 and span > 0 else 0.0
    violations = tuple(Violation((i, j), b, t) for i, j, b, t in r["violations"])
    return VerifyReport(
        valid=not violations and r["offsets_ok"] and peak == plan.peak,
        violations=violations,
        peak_recomputed=peak,
        capacity_ok=peak <= instance.capacity,
        utilization=utilization,
    )


def reduction_vs(plan_peak: int, baseline_peak: int) -> float:
    """1 - plan/baseline; negative when the plan is worse."""
    if baseline_peak == 0:
        raise ZeroBaseline("cannot compute a reduction against a zero peak")
    return 1.0 - plan_peak / baseline_peak


def report_to_json(report: VerifyReport) -> str:
    body = {
        "valid": report.valid,
        "peak_recomputed": report.peak_recomputed,
        "capacity_ok": report.capacity_ok,
        "utilization": round(report.utilization, 6),
        "violations": [{"pair": list(v.pair), "overlap_bytes": v.overlap_bytes,
                        "overlap_ticks": v.overlap_ticks} for v in report.violations],
    }
    return json.dumps(body, indent=2) + "\n"


def clique_lower_bound_arrays(alloc, free, size, *, device: int = 0, stream: int = 0) -> int:
    a, f, s = N.as_i64(alloc), N.as_i64(free), N.as_i64(size)
    out = ctypes.c_int64(0)
    from .bestfit import check
    check(N.lib().mp_clique_lower_bound(N.ptr(a), N.ptr(f), N.ptr(s), len(a),
                                        ctypes.byref(out), 0, device, stream or None))
    return int(out.value)


def _clique_lb_device(instance: DsaInstance) -> int:
    return clique_lower_bound_arrays(*instance.arrays())
