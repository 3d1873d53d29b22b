"""ctypes declarations of include/sinkhorn_b200.h (loads the in-tree libsinkhorn_b200.so).

Fails loudly when the library is missing: there is no CPU fallback anywhere in the
product path.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsinkhorn_b200.so")

SK_OK, SK_EINVAL, SK_ECUDA, SK_ENONFINITE, SK_ENCCL, SK_ENOMEM, SK_EUNSUPPORTED = range(7)
SK_COST_AUTO, SK_COST_ONLINE, SK_COST_STORED = 0, 1, 2
SK_SHARD_BLOCKS = 8


class SkReport(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int32), ("converged", ctypes.c_int32),
                ("marginal_error", ctypes.c_float), ("dual_objective", ctypes.c_double),
                ("init_ms", ctypes.c_double), ("build_ms", ctypes.c_double),
                ("solve_ms", ctypes.c_double)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class SkCounters(ctypes.Structure):
    _fields_ = [("kernel_launches", ctypes.c_int64), ("lse_launches", ctypes.c_int64),
                ("lse_ms", ctypes.c_double), ("lse_ex2", ctypes.c_double),
                ("lse_bytes", ctypes.c_double), ("dom_launches", ctypes.c_int64),
                ("dom_ms", ctypes.c_double), ("dom_entries", ctypes.c_double),
                ("dom_bytes", ctypes.c_double)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


EXPORTS = [
    "sk_create", "sk_set_stream", "sk_destroy", "sk_last_error", "sk_status_string", "sk_version",
    "sk_set_timing", "sk_set_relaxation", "sk_set_eps_decay", "sk_set_anderson", "sk_get_solver_options",
    "sk_set_adaptive_momentum",
    "sk_set_tuning", "sk_set_force_nccl", "sk_get_counters", "sk_reset_counters", "sk_nccl_unique_id", "sk_comm_init",
    "sk_shard_rows", "sinkhorn_sort1d_batched", "sinkhorn_soft_rank_sort", "sinkhorn_fit_gmm", "sinkhorn_vjp", "sinkhorn_init_nw1d", "sinkhorn_init_zero", "sinkhorn_init_sort1d",
    "sinkhorn_init_gaussian", "sinkhorn_init_gmm", "sinkhorn_init_subsample", "sinkhorn_solve",
    "sinkhorn_solve_sharded", "sinkhorn_solve_sharded_emulated", "sk_selftest_tc_dot",
    "sk_microbench",
]

_lib = None


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_2206_07630_b200.build` "
                           "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P, I32, I64, F, D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_double
    S = ctypes.c_int
    sig = {
        "sk_create": (S, [ctypes.POINTER(P), ctypes.c_int, P]),
        "sk_set_stream": (S, [P, P]),
        "sk_destroy": (None, [P]),
        "sk_last_error": (ctypes.c_char_p, [P]),
        "sk_status_string": (ctypes.c_char_p, [ctypes.c_int]),
        "sk_version": (I32, []),
        "sk_set_timing": (S, [P, I32]),
        "sk_set_relaxation": (S, [P, F]),
        "sk_set_eps_decay": (S, [P, F, F]),
        "sk_set_anderson": (S, [P, I32]),
        "sk_get_solver_options": (S, [P, ctypes.POINTER(F), ctypes.POINTER(F), ctypes.POINTER(F),
                                      ctypes.POINTER(I32), ctypes.POINTER(I32)]),
        "sk_set_adaptive_momentum": (S, [P, I32]),
        "sk_set_tuning": (S, [P, ctypes.c_char_p, D]),
        "sk_set_force_nccl": (S, [P, I32]),
        "sk_get_counters": (S, [P, ctypes.POINTER(SkCounters)]),
        "sk_reset_counters": (S, [P]),
        "sk_nccl_unique_id": (S, [P, P]),
        "sk_comm_init": (S, [P, P, I32, I32]),
        "sk_shard_rows": (S, [I64, I32, I32, ctypes.POINTER(I64), ctypes.POINTER(I64)]),
        "sinkhorn_sort1d_batched": (S, [P, I64, I64, P, P, P]),
        "sinkhorn_init_zero": (S, [P, I64, I64, P]),
        "sinkhorn_soft_rank_sort": (S, [P, I64, I64, I64, P, P, I32, F, P, P, P, P, P]),
        "sinkhorn_fit_gmm": (S, [P, I64, I32, P, I32, P, I32, I32, F, F, P, P, P, ctypes.POINTER(D),
                                 ctypes.POINTER(I32)]),
        "sinkhorn_init_nw1d": (S, [P, I64, I64, I64, P, P, I32, P, P, I32, P, P]),
        "sinkhorn_vjp": (S, [P, I64, I64, I32, P, P, F, P, P, P, P, F, I32, P, P, P, P, ctypes.POINTER(I32),
                             ctypes.POINTER(D)]),
        "sinkhorn_init_sort1d": (S, [P, I64, I64, I64, P, P, I32, I32, P, P, P]),
        "sinkhorn_init_gaussian": (S, [P, I64, I64, I32, P, P, P, P, F, P, ctypes.POINTER(I32)]),
        "sinkhorn_init_gmm": (S, [P, I64, I64, I32, P, P, I32, P, P, P, I32, P, P, P, F, F, I32, P,
                                  ctypes.POINTER(I32)]),
        "sinkhorn_init_subsample": (S, [P, I64, I64, I32, P, P, I64, P, I64, P, F, F, I32, P,
                                        ctypes.POINTER(I32), ctypes.POINTER(SkReport)]),
        "sinkhorn_solve": (S, [P, I64, I64, I64, I32, P, P, I32, P, P, F, F, I32, I32, ctypes.c_int,
                               P, P, P, P, ctypes.POINTER(SkReport)]),
        "sinkhorn_solve_sharded": (S, [P, I64, I64, I64, I64, I32, P, P, P, P, F, F, I32, I32,
                                       ctypes.c_int, P, P, P, ctypes.POINTER(SkReport)]),
        "sinkhorn_solve_sharded_emulated": (S, [P, I32, I64, I64, I32, P, P, P, P, F, F, I32, I32,
                                                ctypes.c_int, P, P, P, ctypes.POINTER(SkReport)]),
        "sk_selftest_tc_dot": (S, [P, I32, P, P, P]),
        "sk_microbench": (S, [P, I32, ctypes.POINTER(D)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
