"""B200-native (sm_100a) hot path of "Rethinking Initialization of the Sinkhorn Algorithm"
(Thornton & Cuturi, arXiv 2206.07630).

The compute lives in ``libsinkhorn_b200.so`` (hand-written CUDA, C ABI in
``include/sinkhorn_b200.h``).  This module only marshals arguments: torch tensors
(CUDA or CPU) are passed to the C ABI by pointer — CPU tensors are host buffers that
the library stages itself — and results come back as tensors on the inputs' device.
PyTorch provides device memory, streams and process groups; nothing here computes
any step of the method.
"""
from __future__ import annotations

import contextlib
import ctypes
from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import _lib
from ._lib import (SK_COST_AUTO, SK_COST_ONLINE, SK_COST_STORED, SK_SHARD_BLOCKS, SkCounters,
                   SkReport)

__all__ = ["Context", "SinkhornError", "sinkhorn_solve", "sinkhorn_solve_sharded",
           "sinkhorn_solve_sharded_emulated",
           "sinkhorn_init_zero", "sinkhorn_init_sort1d", "sinkhorn_init_gaussian",
           "sinkhorn_init_gmm", "sinkhorn_init_subsample", "sinkhorn_sort1d_batched",
           "shard_rows", "SK_COST_AUTO", "SK_COST_ONLINE", "SK_COST_STORED", "SK_SHARD_BLOCKS"]

_MODES = {"auto": SK_COST_AUTO, "online": SK_COST_ONLINE, "stored": SK_COST_STORED}


class SinkhornError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_lib.load().sk_status_string(status).decode()}: {msg}")
        self.status = status


class Context:
    """Owns one ``sk_ctx`` bound to a CUDA device and stream (torch's current stream by default)."""

    def __init__(self, device: int = 0, stream: Optional[torch.cuda.Stream] = None):
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2206_07630_b200 needs a CUDA device (no CPU fallback)")
        self.lib = _lib.load()
        self.device = device
        with torch.cuda.device(device):
            s = stream if stream is not None else torch.cuda.current_stream(device)
        self.stream = s
        h = ctypes.c_void_p()
        st = self.lib.sk_create(ctypes.byref(h), device, ctypes.c_void_p(s.cuda_stream))
        if st != 0:
            raise SinkhornError(st, "sk_create failed")
        self.h = h

    def check(self, st: int, allow_nonfinite: bool = False) -> int:
        if st == 0 or (allow_nonfinite and st == _lib.SK_ENONFINITE):
            return st
        raise SinkhornError(st, self.lib.sk_last_error(self.h).decode())

    def set_stream(self, stream: torch.cuda.Stream) -> None:
        self.stream = stream
        self.check(self.lib.sk_set_stream(self.h, ctypes.c_void_p(stream.cuda_stream)))

    def set_timing(self, on: bool) -> None:
        self.check(self.lib.sk_set_timing(self.h, int(on)))

    def counters(self) -> dict:
        c = SkCounters()
        self.check(self.lib.sk_get_counters(self.h, ctypes.byref(c)))
        return c.as_dict()

    def reset_counters(self) -> None:
        self.check(self.lib.sk_reset_counters(self.h))

    def microbench(self, kind: str) -> float:
        """K14 roofline denominators: 'ex2' (ex2/s), 'ffma' (FMA/s), 'hbm' (read B/s), 'tc' (fp16 MMA flop/s)."""
        k = {"ex2": 0, "ffma": 1, "hbm": 2, "tc": 3, "tc_noload": 4, "mma_f16_n128": 5, "mma_f16_n256": 6,
             "mma_tf32_n128": 7, "mma_tf32_n256": 8, "tc_clk": 9, "tc_noload_clk": 10, "tc_epi": 11, "tc_tmem": 12, "tc_math": 13, "tc_full": 14}[kind] \
            if isinstance(kind, str) else int(kind)
        v = ctypes.c_double()
        self.check(self.lib.sk_microbench(self.h, k, ctypes.byref(v)))
        return v.value

    def set_tuning(self, key: str, value: float) -> None:
        """Diagnostic kernel-variant knobs (sk_set_tuning; keys in include/sinkhorn_b200.h)."""
        self.check(self.lib.sk_set_tuning(self.h, key.encode(), float(value)))

    def set_force_nccl(self, on: bool) -> None:
        """Test hook: a 1-rank communicator takes the NCCL branch of the sharded solver."""
        self.check(self.lib.sk_set_force_nccl(self.h, int(on)))

    def solver_options(self) -> dict:
        om, di, dr = ctypes.c_float(), ctypes.c_float(), ctypes.c_float()
        am, ad = ctypes.c_int32(), ctypes.c_int32()
        self.check(self.lib.sk_get_solver_options(self.h, ctypes.byref(om), ctypes.byref(di), ctypes.byref(dr),
                                                  ctypes.byref(am), ctypes.byref(ad)))
        return {"omega": om.value, "eps_decay": (di.value, dr.value), "anderson": am.value, "adaptive": ad.value}

    def nccl_unique_id(self) -> bytes:
        buf = ctypes.create_string_buffer(128)
        self.check(self.lib.sk_nccl_unique_id(self.h, buf))
        return buf.raw

    def comm_init(self, uid: bytes, rank: int, world: int) -> None:
        buf = ctypes.create_string_buffer(uid, 128)
        self.check(self.lib.sk_comm_init(self.h, buf, rank, world))

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.sk_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------ marshalling
_REPORT_DTYPE = np.dtype({"names": [k for k, _ in SkReport._fields_],
                          "formats": ["<i4", "<i4", "<f4", "<f8", "<f8", "<f8", "<f8"],
                          "offsets": [getattr(SkReport, k).offset for k, _ in SkReport._fields_],
                          "itemsize": ctypes.sizeof(SkReport)})


class Reports(Sequence):
    """The B host reports of a batched solve: a sequence of per-problem dicts (built on access)
    over one structured array; column(name) gives a field for every problem as a numpy array
    (no per-problem Python work - a 1024-problem batch would spend ~1 ms building dicts)."""

    def __init__(self, raw):
        self.arr = np.frombuffer(raw, dtype=_REPORT_DTYPE).copy()

    def __len__(self) -> int:
        return len(self.arr)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[k] for k in range(*i.indices(len(self)))]
        r = self.arr[i]
        return {k: r[k].item() for k in self.arr.dtype.names}

    def column(self, name: str) -> np.ndarray:
        return self.arr[name]


@contextlib.contextmanager
def _solver_options(ctx: Context, omega=None, eps_decay=None, anderson=None, adaptive=None):
    """Set the given solver options on the context for one call, then restore the previous
    settings (None leaves an option as the context has it)."""
    if omega is None and eps_decay is None and anderson is None and adaptive is None:
        yield
        return
    prev = ctx.solver_options()
    try:
        if omega is not None:
            ctx.check(ctx.lib.sk_set_relaxation(ctx.h, ctypes.c_float(omega)))
        if eps_decay is not None:
            ctx.check(ctx.lib.sk_set_eps_decay(ctx.h, ctypes.c_float(eps_decay[0]), ctypes.c_float(eps_decay[1])))
        if anderson is not None:
            ctx.check(ctx.lib.sk_set_anderson(ctx.h, int(anderson)))
        if adaptive is not None:
            ctx.check(ctx.lib.sk_set_adaptive_momentum(ctx.h, int(adaptive)))
        yield
    finally:
        ctx.lib.sk_set_relaxation(ctx.h, ctypes.c_float(prev["omega"]))
        ctx.lib.sk_set_eps_decay(ctx.h, ctypes.c_float(prev["eps_decay"][0]), ctypes.c_float(prev["eps_decay"][1]))
        ctx.lib.sk_set_anderson(ctx.h, int(prev["anderson"]))
        ctx.lib.sk_set_adaptive_momentum(ctx.h, int(prev["adaptive"]))

def _ptr(t: Optional[torch.Tensor], dtype=torch.float32):
    if t is None:
        return None
    if t.dtype != dtype or not t.is_contiguous():
        raise TypeError(f"expected a contiguous {dtype} tensor, got {t.dtype} contiguous={t.is_contiguous()}")
    return ctypes.c_void_p(t.data_ptr())


def _empty(shape, like: torch.Tensor, dtype=torch.float32) -> torch.Tensor:
    if like.is_cuda:
        return torch.empty(shape, dtype=dtype, device=like.device)
    return torch.empty(shape, dtype=dtype, pin_memory=torch.cuda.is_available())


def shard_rows(n_total: int, rank: int, world: int) -> Tuple[int, int]:
    lib = _lib.load()
    r0, nl = ctypes.c_int64(), ctypes.c_int64()
    st = lib.sk_shard_rows(n_total, rank, world, ctypes.byref(r0), ctypes.byref(nl))
    if st != 0:
        raise SinkhornError(st, f"sk_shard_rows({n_total}, {rank}, {world})")
    return r0.value, nl.value


# ------------------------------------------------------------------ entries
def sinkhorn_sort1d_batched(ctx: Context, x: torch.Tensor):
    """Stable per-row sort: returns (perm, rank) int32, shape of x (B, n)."""
    B, n = (1, x.numel()) if x.dim() == 1 else (x.shape[0], x.shape[-1])
    perm, rank = _empty(x.shape, x, torch.int32), _empty(x.shape, x, torch.int32)
    ctx.check(ctx.lib.sinkhorn_sort1d_batched(ctx.h, B, n, _ptr(x), _ptr(perm, torch.int32),
                                              _ptr(rank, torch.int32)))
    return perm, rank


def sinkhorn_init_zero(ctx: Context, B: int, n: int, like: torch.Tensor) -> torch.Tensor:
    pot = _empty((B, n) if B > 1 else (n,), like)
    ctx.check(ctx.lib.sinkhorn_init_zero(ctx.h, B, n, _ptr(pot)))
    return pot


def sinkhorn_init_sort1d(ctx: Context, x: torch.Tensor, y: torch.Tensor, y_shared: bool = True,
                         dualsort_iters: int = 0, want_perm: bool = False):
    """x: (B, n) or (B, n, 1); y: (m,) shared or (B, m).  Returns pot (B, n) [, perm, rank]."""
    B = x.shape[0] if x.dim() >= 2 else 1
    n = x.shape[1] if x.dim() >= 2 else x.shape[0]
    m = y.shape[-2] if (y.dim() >= 2 and y.shape[-1] == 1) else y.shape[-1]
    pot = _empty((B, n), x)
    perm = _empty((B, n), x, torch.int32) if want_perm else None
    rank = _empty((B, n), x, torch.int32) if want_perm else None
    ctx.check(ctx.lib.sinkhorn_init_sort1d(ctx.h, B, n, m, _ptr(x), _ptr(y), int(y_shared),
                                           dualsort_iters, _ptr(pot), _ptr(perm, torch.int32),
                                           _ptr(rank, torch.int32)))
    return (pot, perm, rank) if want_perm else pot


def sinkhorn_init_gaussian(ctx: Context, x, y, a=None, b=None, ridge_rel: float = 1e-6):
    n, d = x.shape
    m = y.shape[0]
    side = ctypes.c_int32()
    pot = _empty((min(n, m) if n != m else n,), x)
    ctx.check(ctx.lib.sinkhorn_init_gaussian(ctx.h, n, m, d, _ptr(x), _ptr(a), _ptr(y), _ptr(b),
                                             float(ridge_rel), _ptr(pot), ctypes.byref(side)))
    return pot, side.value


def sinkhorn_init_gmm(ctx: Context, x, y, gx: dict, gy: dict, eps: float, inner_tol: float = 1e-9,
                      inner_max_iter: int = 100000):
    """gx/gy: {'weights': (K,), 'means': (K, d), 'covs': (K, d, d)} fp32 tensors."""
    n, d = x.shape
    m = y.shape[0]
    side = ctypes.c_int32()
    pot = _empty((min(n, m),), x)
    ctx.check(ctx.lib.sinkhorn_init_gmm(
        ctx.h, n, m, d, _ptr(x), _ptr(y), gx["weights"].shape[0], _ptr(gx["weights"]),
        _ptr(gx["means"]), _ptr(gx["covs"]), gy["weights"].shape[0], _ptr(gy["weights"]),
        _ptr(gy["means"]), _ptr(gy["covs"]), float(eps), float(inner_tol), int(inner_max_iter),
        _ptr(pot), ctypes.byref(side)))
    return pot, side.value


def sinkhorn_init_subsample(ctx: Context, x, y, idx_x, idx_y, eps: float, inner_tol: float,
                            inner_max_iter: int = 10000):
    n, d = x.shape
    m = y.shape[0]
    side = ctypes.c_int32()
    rep = SkReport()
    pot = _empty((min(n, m),), x)
    ctx.check(ctx.lib.sinkhorn_init_subsample(
        ctx.h, n, m, d, _ptr(x), _ptr(y), idx_x.numel(), _ptr(idx_x, torch.int32), idx_y.numel(),
        _ptr(idx_y, torch.int32), float(eps), float(inner_tol), int(inner_max_iter), _ptr(pot),
        ctypes.byref(side), ctypes.byref(rep)))
    return pot, side.value, rep.as_dict()


def sinkhorn_solve(ctx: Context, x, y, eps: float, tol: float = 1e-3, max_iter: int = 10000,
                   check_every: int = 1, a=None, b=None, y_shared: bool = False, mode: str = "auto",
                   f_init=None, g_init=None, f=None, g=None, allow_nonfinite: bool = False,
                   omega: Optional[float] = None, eps_decay=None, anderson: Optional[int] = None,
                   adaptive: Optional[int] = None):
    """Solve B >= 1 problems.  x: (n, d) or (B, n, d); y: (m, d) [shared] or (B, m, d).
    omega: Alg. 1's relaxation (sk_set_relaxation; 1 = plain Sinkhorn).
    eps_decay: (init, rate) for sk_set_eps_decay (e.g. (5, 0.8); (0, 1) = off).
    anderson: Anderson memory for sk_set_anderson (e.g. 5), 0 = off.
    adaptive: adaptive-momentum window for sk_set_adaptive_momentum (e.g. 10), 0 = off.
    Each option given applies to this call only (the context's previous setting is restored);
    None uses the context's setting (default: plain Sinkhorn).
    Returns (f, g, reports) with f (B, n) / g (B, m) (B dropped for a single problem)."""
    with _solver_options(ctx, omega, eps_decay, anderson, adaptive):
        return _solve(ctx, x, y, eps, tol, max_iter, check_every, a, b, y_shared, mode, f_init, g_init, f, g,
                      allow_nonfinite)


def _solve(ctx, x, y, eps, tol, max_iter, check_every, a, b, y_shared, mode, f_init, g_init, f, g,
           allow_nonfinite):
    single = x.dim() == 2
    xb = x.unsqueeze(0) if single else x
    B, n, d = xb.shape
    m = y.shape[-2]
    if f is None:
        f = _empty((B, n), x)
    if g is None:
        g = _empty((B, m), x)
    reps = (SkReport * B)()
    st = ctx.lib.sinkhorn_solve(ctx.h, B, n, m, d, _ptr(x), _ptr(y), int(y_shared), _ptr(a), _ptr(b),
                                float(eps), float(tol), int(max_iter), int(check_every), _MODES[mode],
                                _ptr(f_init), _ptr(g_init), _ptr(f), _ptr(g), reps)
    ctx.check(st, allow_nonfinite)
    if single:
        return f.view(n), g.view(m), reps[0].as_dict()
    return f, g, Reports(reps)


def sinkhorn_init_nw1d(ctx: Context, x, y, a=None, b=None, y_shared: bool = True, max_rounds: int = 0):
    """General 1D initializer (NW corner + Alg. 3/4, R-26): x (B, n) or (n,); y (m,) [shared] or
    (B, m); weights like x / y (None = uniform).  Returns (f0 like x, rounds per problem)."""
    single = x.dim() == 1
    xb = x.unsqueeze(0) if single else x
    B, n = xb.shape
    m = y.shape[-1]
    pot = _empty((B, n), x)
    rounds = torch.zeros(B, dtype=torch.int32, device=x.device) if x.is_cuda else torch.zeros(B, dtype=torch.int32)
    ctx.check(ctx.lib.sinkhorn_init_nw1d(ctx.h, B, n, m, _ptr(x), _ptr(y), int(y_shared), _ptr(a), _ptr(b),
                                         int(max_rounds), _ptr(pot), _ptr(rounds, torch.int32)))
    return (pot.view(n) if single else pot), rounds


def sinkhorn_fit_gmm(ctx: Context, x, K: int, init_idx, iters: int = 100, reg_covar: float = 1e-6,
                     kmeans_iters: int = 0, tol: float = 0.0, return_iters: bool = False):
    """EM fit of a K-component full-covariance GMM of x (n, d) (NEXT-3), started from means
    x[init_idx] (kmeans_iters = 0) or from kmeans_iters Lloyd steps from those centers (R-28);
    tol > 0 stops EM as sklearn's GaussianMixture(tol) does.
    Returns ({'weights', 'means', 'covs'} as sinkhorn_init_gmm takes them, mean log-likelihood
    [, EM steps run])."""
    n, d = x.shape
    idx = init_idx if isinstance(init_idx, torch.Tensor) else torch.as_tensor(init_idx, dtype=torch.int32)
    idx = idx.to(torch.int32).contiguous()
    w = _empty((K,), x)
    mu = _empty((K, d), x)
    cov = _empty((K, d, d), x)
    ll = ctypes.c_double()
    it = ctypes.c_int32()
    ctx.check(ctx.lib.sinkhorn_fit_gmm(ctx.h, n, d, _ptr(x), int(K), _ptr(idx, torch.int32), int(kmeans_iters),
                                       int(iters), float(tol), float(reg_covar), _ptr(w), _ptr(mu), _ptr(cov),
                                       ctypes.byref(ll), ctypes.byref(it)))
    g = {"weights": w, "means": mu, "covs": cov}
    return (g, ll.value, it.value) if return_iters else (g, ll.value)


def sinkhorn_vjp(ctx: Context, x, y, eps: float, f, g, zf, zg, cg_tol: float = 1e-6, cg_max_iter: int = 2000):
    """Implicit-differentiation VJP of the optimal potentials with cotangent (zf, zg):
    returns ({'x', 'y', 'a', 'b'} gradients, {'cg_iters', 'cg_relres'})."""
    n, d = x.shape
    m = y.shape[0]
    gx, gy, ga, gb = _empty((n, d), x), _empty((m, d), x), _empty((n,), x), _empty((m,), x)
    it, rr = ctypes.c_int32(), ctypes.c_double()
    ctx.check(ctx.lib.sinkhorn_vjp(ctx.h, n, m, d, _ptr(x), _ptr(y), float(eps), _ptr(f), _ptr(g), _ptr(zf),
                                   _ptr(zg), float(cg_tol), int(cg_max_iter), _ptr(gx), _ptr(gy), _ptr(ga), _ptr(gb),
                                   ctypes.byref(it), ctypes.byref(rr)))
    return {"x": gx, "y": gy, "a": ga, "b": gb}, {"cg_iters": it.value, "cg_relres": rr.value}


def sinkhorn_soft_rank_sort(ctx: Context, x, y, eps: float, f, g, z=None,
                            y_shared: bool = False, ranks: bool = True, sort: bool = True):
    """Soft ranks E_P[z | i] and soft sort E_P[x | j] of B 1D problems from their potentials
    (R-22).  x: (B, n) or (n,); y: (m,) [shared] or (B, m);
    f: like x, g: (B, m) or (m,).  Returns (rank, sort) (None where not requested)."""
    single = x.dim() == 1
    xb = x.unsqueeze(0) if single else x
    B, n = xb.shape
    m = y.shape[-1]
    r = _empty((B, n), x) if ranks else None
    s = _empty((B, m), x) if sort else None
    ctx.check(ctx.lib.sinkhorn_soft_rank_sort(ctx.h, B, n, m, _ptr(x), _ptr(y), int(y_shared), float(eps),
                                              _ptr(f), _ptr(g), _ptr(z), _ptr(r), _ptr(s)))
    if single:
        return (None if r is None else r.view(n)), (None if s is None else s.view(m))
    return r, s


def sinkhorn_solve_sharded_emulated(ctx: Context, world: int, x, y, eps: float, tol: float = 1e-3,
                                    max_iter: int = 10000, check_every: int = 1, a=None, b=None,
                                    mode: str = "auto", f_init=None, anderson: Optional[int] = None,
                                    omega: Optional[float] = None, eps_decay=None, adaptive: Optional[int] = None):
    """The row-sharded algorithm for `world` virtual ranks on one GPU (test entry).
    anderson / omega / eps_decay / adaptive: as sinkhorn_solve (this call only; None = the context's)."""
    with _solver_options(ctx, omega, eps_decay, anderson, adaptive):
        return _solve_sharded_emulated(ctx, world, x, y, eps, tol, max_iter, check_every, a, b, mode, f_init)


def _solve_sharded_emulated(ctx, world, x, y, eps, tol, max_iter, check_every, a, b, mode, f_init):
    n, d = x.shape
    m = y.shape[0]
    f = _empty((n,), x)
    g = _empty((m,), x)
    rep = SkReport()
    ctx.check(ctx.lib.sinkhorn_solve_sharded_emulated(
        ctx.h, world, n, m, d, _ptr(x), _ptr(y), _ptr(a), _ptr(b), float(eps), float(tol),
        int(max_iter), int(check_every), _MODES[mode], _ptr(f_init), _ptr(f), _ptr(g), ctypes.byref(rep)))
    return f, g, rep.as_dict()


def sinkhorn_solve_sharded(ctx: Context, n_total: int, row0: int, x_local, y, eps: float,
                           tol: float = 1e-3, max_iter: int = 10000, check_every: int = 1,
                           a_local=None, b=None, mode: str = "auto", f_init_local=None,
                           anderson: Optional[int] = None, omega: Optional[float] = None, eps_decay=None,
                           adaptive: Optional[int] = None):
    """Rows [row0, row0 + n_local) of an n_total-row problem on this rank (sk_comm_init first);
    anderson: Anderson memory (sk_set_anderson; one 9-double allreduce per sweep), 0 = off;
    omega: relaxation (sk_set_relaxation; one 2-double allreduce of the row terms per sweep);
    eps_decay: (init, rate); adaptive: the adaptive-momentum window.  Each applies to this call only
    (None = the context's setting)."""
    with _solver_options(ctx, omega, eps_decay, anderson, adaptive):
        return _solve_sharded(ctx, n_total, row0, x_local, y, eps, tol, max_iter, check_every, a_local, b, mode,
                              f_init_local)


def _solve_sharded(ctx, n_total, row0, x_local, y, eps, tol, max_iter, check_every, a_local, b, mode, f_init_local):
    n_local, d = x_local.shape
    m = y.shape[0]
    f = _empty((n_local,), x_local)
    g = _empty((m,), x_local)
    rep = SkReport()
    ctx.check(ctx.lib.sinkhorn_solve_sharded(
        ctx.h, n_total, row0, n_local, m, d, _ptr(x_local), _ptr(y), _ptr(a_local), _ptr(b),
        float(eps), float(tol), int(max_iter), int(check_every), _MODES[mode], _ptr(f_init_local),
        _ptr(f), _ptr(g), ctypes.byref(rep)))
    return f, g, rep.as_dict()
