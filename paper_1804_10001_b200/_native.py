"""ctypes binding of libmemplan_b200.so (include/memplan_b200.h).

The library is built in-tree (``__graft_entry__.build()`` /
``paper_1804_10001_b200/csrc/Makefile``) into ``paper_1804_10001_b200/_lib``.
Loading fails loudly if it is missing: there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# MEMPLAN_LIB: an alternative build of the same library (A/B tuning runs)
LIB_PATH = os.environ.get("MEMPLAN_LIB") or os.path.join(_HERE, "_lib", "libmemplan_b200.so")

# status codes (include/memplan_b200.h: mp_status)
MP_OK = 0
MP_ERR_INVALID = 1
MP_ERR_LOOP_BOUND = 2
MP_ERR_ILLEGAL_LIFT = 3
MP_ERR_CUDA = 4
MP_ERR_NO_DEVICE = 5
MP_ERR_DOUBLE_FREE = 6
MP_ERR_UNKNOWN_ID = 7
MP_ERR_EXTRA_REQUEST = 8
MP_ERR_ALLOC_AFTER_CLOSE = 9
MP_ERR_LIVE_AT_RESET = 10
MP_ERR_UNBALANCED_RESUME = 11
MP_ERR_INVALID_PLAN = 12
MP_ERR_OUT_OF_MEMORY = 13
MP_ERR_NEGATIVE_SIZE = 14
MP_ERR_TRACE = 15

MP_DEVICE_PTRS = 1
MP_ASYNC = 2
MP_FORCE_GLOBAL = 4
MP_STATS = 8

P64 = ctypes.POINTER(ctypes.c_int64)
PU64 = ctypes.POINTER(ctypes.c_uint64)
P32 = ctypes.POINTER(ctypes.c_int32)
VP = ctypes.c_void_p


class PlanInfo(ctypes.Structure):
    _fields_ = [("steps", ctypes.c_int64), ("lifts", ctypes.c_int64),
                ("max_lines", ctypes.c_int64), ("prep_ms", ctypes.c_float),
                ("plan_ms", ctypes.c_float), ("kernel_ms", ctypes.c_float),
                ("engine", ctypes.c_int32), ("cluster", ctypes.c_int32),
                ("sum_wlive", ctypes.c_int64), ("launches", ctypes.c_int64),
                ("diag", ctypes.c_int64 * 4), ("cycles", ctypes.c_int64 * 6)]


class VerifyReportC(ctypes.Structure):
    _fields_ = [("n_violations", ctypes.c_int64), ("peak_recomputed", ctypes.c_int64),
                ("offsets_ok", ctypes.c_int32), ("pad", ctypes.c_int32),
                ("used_lo", ctypes.c_uint64), ("used_hi", ctypes.c_uint64)]


class ArenaState(ctypes.Structure):
    _fields_ = [(name, ctypes.c_int64) for name in (
        "lam", "reopt_count", "forced_closes", "plan_peak", "pool_peak", "n_blocks",
        "n_live", "depth", "plan_version", "pool_last_ref")]


class TorchStats(ctypes.Structure):
    """mp_torch_stats_t (include/memplan_b200.h)."""
    _fields_ = [(k, ctypes.c_int64) for k in
                ("n_planned", "n_side", "n_diverged", "n_replans", "n_carried_live",
                 "n_regions", "n_unknown_free", "n_side_live")] + \
               [("region_base", ctypes.c_uint64), ("region_bytes", ctypes.c_int64),
                ("plan_peak", ctypes.c_int64)]


class IngestInfo(ctypes.Structure):
    _fields_ = [(name, ctypes.c_int64) for name in (
        "n_blocks", "unmanaged_count", "horizon", "n_events", "err_line", "err_tok_off",
        "err_tok_len", "err_value", "err_seen")] + [("err_kind", ctypes.c_int32),
                                                     ("pad", ctypes.c_int32)]


VIOLATION_DTYPE = np.dtype([("i", np.int64), ("j", np.int64),
                            ("overlap_bytes", np.int64), ("overlap_ticks", np.int64)])

# (name, restype, argtypes) for every symbol include/memplan_b200.h declares
SIGNATURES = [
    ("mp_plan_bestfit", ctypes.c_int, [VP, VP, VP, ctypes.c_int64, VP, VP, ctypes.c_int,
                                       ctypes.c_int, VP]),
    ("mp_plan_bestfit_batched", ctypes.c_int, [VP, VP, VP, VP, ctypes.c_int64, VP, VP,
                                               ctypes.c_int, ctypes.c_int, VP]),
    ("mp_plan_last_info", ctypes.c_int, [ctypes.POINTER(PlanInfo)]),
    ("mp_pipe_create", VP, [ctypes.c_int]),
    ("mp_pipe_submit", ctypes.c_int, [VP, VP, VP, VP, VP, ctypes.c_int64, VP, VP, ctypes.c_int,
                                      P64]),
    ("mp_pipe_wait", ctypes.c_int, [VP, ctypes.c_int64]),
    ("mp_pipe_destroy", None, [VP]),
    ("mp_verify", ctypes.c_int, [VP, VP, VP, VP, ctypes.c_int64, ctypes.POINTER(VerifyReportC),
                                 VP, ctypes.c_int64, ctypes.c_int, ctypes.c_int, VP]),
    ("mp_clique_lower_bound", ctypes.c_int, [VP, VP, VP, ctypes.c_int64, P64, ctypes.c_int,
                                             ctypes.c_int, VP]),
    ("mp_ingest_trace", ctypes.c_int, [ctypes.c_char_p, ctypes.c_int64, ctypes.c_int64, VP, VP,
                                       VP, ctypes.c_int64, ctypes.POINTER(IngestInfo)]),
    ("mp_arena_open", ctypes.c_int, [VP, VP, VP, VP, ctypes.c_int64, ctypes.c_int64,
                                     ctypes.c_uint64, ctypes.c_int64, ctypes.c_int,
                                     ctypes.c_int, ctypes.POINTER(VP)]),
    ("mp_arena_close_handle", None, [VP]),
    ("mp_arena_alloc", ctypes.c_int, [VP, ctypes.c_int64, PU64]),
    ("mp_arena_free", ctypes.c_int, [VP, ctypes.c_int64]),
    ("mp_arena_reset", ctypes.c_int, [VP]),
    ("mp_arena_interrupt", ctypes.c_int, [VP]),
    ("mp_arena_resume", ctypes.c_int, [VP]),
    ("mp_arena_close", ctypes.c_int, [VP]),
    ("mp_arena_reoptimize", ctypes.c_int, [VP]),
    ("mp_arena_pool", VP, [VP]),
    ("mp_arena_get_state", ctypes.c_int, [VP, ctypes.POINTER(ArenaState)]),
    ("mp_arena_get_plan", ctypes.c_int, [VP, VP, VP, VP, VP]),
    ("mp_arena_get_live", ctypes.c_int, [VP, VP, VP, VP]),
    ("mp_arena_get_observed", ctypes.c_int, [VP, VP]),
    ("mp_arena_replay", ctypes.c_int, [VP, VP, VP, ctypes.c_int64, VP, P64]),
    ("mp_arena_bench", ctypes.c_int, [VP, VP, VP, ctypes.c_int64, ctypes.c_int64,
                                      ctypes.POINTER(ctypes.c_double)]),
    ("mp_torch_alloc", VP, [ctypes.c_size_t, ctypes.c_int, VP]),
    ("mp_torch_free", None, [VP, ctypes.c_size_t, ctypes.c_int, VP]),
    ("mp_torch_set_mode", ctypes.c_int, [ctypes.c_int, VP]),
    ("mp_torch_get_trace", ctypes.c_int, [VP, VP, ctypes.c_int64, P64]),
    ("mp_torch_epoch_reset", ctypes.c_int, []),
    ("mp_torch_replay_begin", ctypes.c_int, [VP, ctypes.c_int, PU64]),
    ("mp_torch_replay_end", ctypes.c_int, []),
    ("mp_torch_stats", ctypes.c_int, [P64, P64, P64]),
    ("mp_torch_stats_ex", ctypes.c_int, [ctypes.POINTER(TorchStats)]),
    ("mp_torch_bench", ctypes.c_int, [VP, VP, ctypes.c_int64, ctypes.c_int64,
                                      ctypes.POINTER(ctypes.c_double)]),
    ("mp_pool_create", ctypes.c_int, [ctypes.c_int64, ctypes.POINTER(VP)]),
    ("mp_pool_destroy", None, [VP]),
    ("mp_pool_alloc", ctypes.c_int, [VP, ctypes.c_int64, P64, P64]),
    ("mp_pool_free", ctypes.c_int, [VP, ctypes.c_int64]),
    ("mp_pool_stats", ctypes.c_int, [VP, P64, P64, P64, P64]),
    ("mp_simulate_pool", ctypes.c_int, [VP, VP, ctypes.c_int64, ctypes.c_int64, P64]),
    ("mp_last_error", ctypes.c_char_p, []),
    ("mp_device_count", ctypes.c_int, []),
    ("mp_version", ctypes.c_char_p, []),
]

_lib = None
_lock = threading.Lock()


class NativeLibraryMissing(ImportError):
    pass


def lib():
    """The loaded library; raises NativeLibraryMissing if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeLibraryMissing(
                    f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; "
                    "g.build()'` (there is no CPU fallback)")
            l = ctypes.CDLL(LIB_PATH)
            for name, res, args in SIGNATURES:
                fn = getattr(l, name, None)
                if fn is None:
                    continue
                fn.restype = res
                fn.argtypes = args
            _lib = l
    return _lib


def last_error() -> str:
    return lib().mp_last_error().decode(errors="replace")


def ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def as_i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)
