"""fp64 CPU ORACLE for the hot path of arXiv 2206.07630 (Thornton & Cuturi).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  It shares no code with the CUDA path (``paper_2206_07630_b200``), and
the CUDA path never imports it.

Two layers:
  * ``sk_oracle.c`` (plain C, fp64, OpenMP over independent rows/columns only):
    cost by direct differences, soft-min, Sinkhorn (Alg. 1), the explicit
    marginal error (threshold appendix) and Eq. (2), sorting, DualSort (Alg. 2)
    and the Subsample extrapolation (Eq. 8).
  * this file (numpy fp64): the d x d linear algebra of the Gaussian (Sec. 3.2,
    Gaussian-Potential appendix) and GMM (Sec. 3.3) initializers, with matrix
    square roots by symmetric eigendecomposition (``numpy.linalg.eigh``), a
    library primitive used as one step.

Inputs are the fp32 arrays of ``workloads.gen`` promoted exactly to fp64.
Readings of the paper used here are DESIGN.md R-1..R-20.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sk_oracle.c")
_LIB_PATH = os.path.join(_HERE, "libsk_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile sk_oracle.c with gcc (-O2 -fopenmp).  Building the checker is not using it."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-fno-fast-math", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        D, I64, I = ctypes.c_double, ctypes.c_int64, ctypes.c_int
        P = ctypes.c_void_p
        lib.ora_softmin.restype = D
        lib.ora_softmin.argtypes = [I64, P, D]
        lib.ora_sinkhorn_points.restype = I
        lib.ora_sinkhorn_points.argtypes = [I64, I64, I, P, P, P, P, D, D, I, I, P, P, P, P, P, P, P]
        lib.ora_sinkhorn_points_omega.restype = I
        lib.ora_sinkhorn_points_omega.argtypes = [I64, I64, I, P, P, P, P, D, D, D, I, I, P, P, P, P, P, P, P]
        lib.ora_sinkhorn_points_decay.restype = I
        lib.ora_sinkhorn_points_decay.argtypes = [I64, I64, I, P, P, P, P, D, D, D, D, D, I, I, P, P, P, P, P, P, P]
        lib.ora_sinkhorn_points_adaptive.restype = I
        lib.ora_sinkhorn_points_adaptive.argtypes = [I64, I64, I, P, P, P, P, D, D, I, D, I, I, P, P, P, P, P, P,
                                                     P, P]
        lib.ora_sinkhorn_matrix_anderson.restype = I
        lib.ora_sinkhorn_matrix_anderson.argtypes = [I64, I64, P, P, P, D, I, D, I, I, P, P, P, P, P, P]
        lib.ora_sinkhorn_points_anderson.restype = I
        lib.ora_sinkhorn_points_anderson.argtypes = [I64, I64, I, P, P, P, P, D, I, D, I, I, P, P, P, P, P, P]
        lib.ora_sinkhorn_matrix.restype = I
        lib.ora_sinkhorn_matrix.argtypes = [I64, I64, P, P, P, D, D, I, I, P, P, P, P, P, P, P]
        lib.ora_f_update_points.argtypes = [I64, I64, I, P, P, P, P, D, P, P, I64]
        lib.ora_g_update_points.argtypes = [I64, I64, I, P, P, P, P, D, P, P, I64]
        for nm in ("ora_marginal_error_points", "ora_dual_objective_points"):
            getattr(lib, nm).restype = D
            getattr(lib, nm).argtypes = [I64, I64, I, P, P, P, P, P, P, D]
        for nm in ("ora_marginal_error_matrix", "ora_dual_objective_matrix"):
            getattr(lib, nm).restype = D
            getattr(lib, nm).argtypes = [I64, I64, P, P, P, P, P, D]
        lib.ora_plan_row_sums.argtypes = [I64, I64, I, P, P, P, P, D, P, I64, P]
        lib.ora_plan_col_sums.argtypes = [I64, I64, I, P, P, P, P, D, P, I64, P]
        lib.ora_subsample_extrapolate.argtypes = [I64, I64, I, P, P, P, D, P, P, I64]
        lib.ora_sort_rank.restype = I
        lib.ora_sort_rank.argtypes = [I64, I64, P, P, P]
        lib.ora_dualsort.restype = I
        lib.ora_dualsort.argtypes = [I64, P, P, I, P]
        lib.ora_cost_matrix.argtypes = [I64, I64, I, P, P, P]
        lib.ora_num_threads.restype = I
        lib.ora_set_num_threads.argtypes = [I]
        _lib = lib
    return _lib


def _d(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _pts(x) -> np.ndarray:
    x = _d(x)
    return x.reshape(x.shape[0], -1) if x.ndim != 1 else x.reshape(-1, 1)


def _weights(w, n) -> np.ndarray:
    return np.full(n, 1.0 / n) if w is None else _d(w)


def num_threads() -> int:
    return _L().ora_num_threads()


def set_num_threads(t: int) -> None:
    _L().ora_set_num_threads(int(t))


# ---------------------------------------------------------------- basics ---
def cost_matrix(x, y) -> np.ndarray:
    """C_ij = sum_k (x_ik - y_jk)^2 by direct differences."""
    x, y = _pts(x), _pts(y)
    C = np.empty((x.shape[0], y.shape[0]))
    _L().ora_cost_matrix(x.shape[0], y.shape[0], x.shape[1], _p(x), _p(y), _p(C))
    return C


def softmin(S_row, eps: float) -> float:
    """min_eps of one row."""
    S = _d(S_row).ravel()
    return _L().ora_softmin(S.size, _p(S), float(eps))


class Result(dict):
    __getattr__ = dict.__getitem__


def sinkhorn(x, y, eps, a=None, b=None, tol=1e-3, max_iter=10000, check_every=1,
             f0=None, trace=False, omega=1.0, eps_decay=None) -> Result:
    """Alg. 1, g-then-f, explicit stopping rule; tol<=0 = exactly max_iter sweeps.
    omega: Alg. 1's relaxation (R-1 reading): v <- (1 - omega) v + omega v_sinkhorn.
    eps_decay: (init, rate) for sweep l's eps_l = max(eps, eps init rate^(l-1)) (R-25)."""
    x, y = _pts(x), _pts(y)
    n, m, d = x.shape[0], y.shape[0], x.shape[1]
    a, b = _weights(a, n), _weights(b, m)
    f, g = np.empty(n), np.empty(m)
    it, err, E = ctypes.c_int(), ctypes.c_double(), ctypes.c_double()
    f0a = None if f0 is None else _d(f0)
    tr = np.empty(max_iter) if trace else None
    di, dr = (0.0, 1.0) if eps_decay is None else (float(eps_decay[0]), float(eps_decay[1]))
    conv = _L().ora_sinkhorn_points_decay(n, m, d, _p(x), _p(y), _p(a), _p(b), float(eps), float(omega), di, dr,
                                          float(tol), int(max_iter), int(check_every), _p(f0a), _p(f),
                                          _p(g), ctypes.byref(it), ctypes.byref(err), ctypes.byref(E), _p(tr))
    r = Result(f=f, g=g, iterations=it.value, converged=bool(conv), err=err.value, E=E.value)
    if trace:
        r["trace"] = tr[: it.value]
    return r


def sinkhorn_adaptive(x, y, eps, adapt_iters=10, a=None, b=None, tol=1e-3, max_iter=10000, check_every=1,
                      f0=None, g0=None, omega=1.0) -> Result:
    """Alg. 1 with adaptive momentum ("adapt=10"; reading R-31): plain sweeps, then
    after every window of adapt_iters sweeps (from the second on) omega = 2/(1 + sqrt(1 - rho))
    (clipped to [1, 1.95]) from the window's per-sweep error contraction rho, applied from two
    sweeps later.  adapt_iters = 0: the fixed-omega solver with an optional starting g0.
    Returns the Result of sinkhorn() plus r.omega: the omega of every sweep."""
    x, y = _pts(x), _pts(y)
    n, m, d = x.shape[0], y.shape[0], x.shape[1]
    a, b = _weights(a, n), _weights(b, m)
    f, g = np.empty(n), np.empty(m)
    it, err, E = ctypes.c_int(), ctypes.c_double(), ctypes.c_double()
    f0a = None if f0 is None else _d(f0)
    g0a = None if g0 is None else _d(g0)
    om = np.empty(max_iter)
    conv = _L().ora_sinkhorn_points_adaptive(n, m, d, _p(x), _p(y), _p(a), _p(b), float(eps), float(omega),
                                             int(adapt_iters), float(tol), int(max_iter), int(check_every), _p(f0a),
                                             _p(g0a), _p(f), _p(g), ctypes.byref(it), ctypes.byref(err),
                                             ctypes.byref(E), _p(om))
    if conv < 0:
        raise ValueError("adapt_iters must be >= 0")
    return Result(f=f, g=g, iterations=it.value, converged=bool(conv), err=err.value, E=E.value,
                  omega=om[: it.value])


def sinkhorn_anderson(x, y, eps, mem=5, a=None, b=None, tol=1e-3, max_iter=10000, check_every=1, f0=None) -> Result:
    """Alg. 1 with Anderson acceleration of memory `mem` on the sweep map (R-27):
    returns the last iterate's pair (f, g_sk(f)) with its explicit error and Eq. (2)."""
    if not 1 <= int(mem) <= 16:
        raise ValueError(f"Anderson memory must lie in [1, 16], got {mem}")
    x, y = _pts(x), _pts(y)
    n, m, d = x.shape[0], y.shape[0], x.shape[1]
    a, b = _weights(a, n), _weights(b, m)
    f, g = np.empty(n), np.empty(m)
    it, err, E = ctypes.c_int(), ctypes.c_double(), ctypes.c_double()
    f0a = None if f0 is None else _d(f0)
    conv = _L().ora_sinkhorn_points_anderson(n, m, d, _p(x), _p(y), _p(a), _p(b), float(eps), int(mem), float(tol),
                                             int(max_iter), int(check_every), _p(f0a), _p(f), _p(g),
                                             ctypes.byref(it), ctypes.byref(err), ctypes.byref(E))
    return Result(f=f, g=g, iterations=it.value, converged=bool(conv), err=err.value, E=E.value)


def sinkhorn_matrix(C, eps, a=None, b=None, tol=1e-3, max_iter=10000, check_every=1,
                    f0=None, trace=False, anderson=0) -> Result:
    C = _d(C)
    n, m = C.shape
    a, b = _weights(a, n), _weights(b, m)
    f, g = np.empty(n), np.empty(m)
    it, err, E = ctypes.c_int(), ctypes.c_double(), ctypes.c_double()
    f0a = None if f0 is None else _d(f0)
    if anderson:   # Anderson on the sweep map (R-27), as sinkhorn_anderson for a given cost matrix
        if not 1 <= int(anderson) <= 16:
            raise ValueError(f"Anderson memory must lie in [1, 16], got {anderson}")
        conv = _L().ora_sinkhorn_matrix_anderson(n, m, _p(C), _p(a), _p(b), float(eps), int(anderson), float(tol),
                                                 int(max_iter), int(check_every), _p(f0a), _p(f), _p(g),
                                                 ctypes.byref(it), ctypes.byref(err), ctypes.byref(E))
        return Result(f=f, g=g, iterations=it.value, converged=bool(conv), err=err.value, E=E.value)
    tr = np.empty(max_iter) if trace else None
    conv = _L().ora_sinkhorn_matrix(n, m, _p(C), _p(a), _p(b), float(eps), float(tol),
                                    int(max_iter), int(check_every), _p(f0a), _p(f), _p(g),
                                    ctypes.byref(it), ctypes.byref(err), ctypes.byref(E), _p(tr))
    r = Result(f=f, g=g, iterations=it.value, converged=bool(conv), err=err.value, E=E.value)
    if trace:
        r["trace"] = tr[: it.value]
    return r


def f_update(x, y, g, eps, a=None, rows=None) -> np.ndarray:
    """f_i = eps log a_i - eps LSE_j((g_j - C_ij)/eps) for the given rows (all if None)."""
    x, y, g = _pts(x), _pts(y), _d(g)
    n, m, d = x.shape[0], y.shape[0], x.shape[1]
    a = _weights(a, n)
    r = None if rows is None else np.ascontiguousarray(rows, dtype=np.int64)
    out = np.empty(n if r is None else r.size)
    _L().ora_f_update_points(n, m, d, _p(x), _p(y), _p(a), _p(g), float(eps), _p(out), _p(r),
                             0 if r is None else r.size)
    return out


def g_update(x, y, f, eps, b=None, cols=None) -> np.ndarray:
    """g_j = eps log b_j - eps LSE_i((f_i - C_ij)/eps) for the given columns (all if None)."""
    x, y, f = _pts(x), _pts(y), _d(f)
    n, m, d = x.shape[0], y.shape[0], x.shape[1]
    b = _weights(b, m)
    c = None if cols is None else np.ascontiguousarray(cols, dtype=np.int64)
    out = np.empty(m if c is None else c.size)
    _L().ora_g_update_points(n, m, d, _p(x), _p(y), _p(b), _p(f), float(eps), _p(out), _p(c),
                             0 if c is None else c.size)
    return out


def marginal_error(x, y, f, g, eps, a=None, b=None) -> float:
    x, y = _pts(x), _pts(y)
    n, m, d = x.shape[0], y.shape[0], x.shape[1]
    return _L().ora_marginal_error_points(n, m, d, _p(x), _p(y), _p(_weights(a, n)),
                                          _p(_weights(b, m)), _p(_d(f)), _p(_d(g)), float(eps))


def dual_objective(x, y, f, g, eps, a=None, b=None) -> float:
    x, y = _pts(x), _pts(y)
    n, m, d = x.shape[0], y.shape[0], x.shape[1]
    return _L().ora_dual_objective_points(n, m, d, _p(x), _p(y), _p(_weights(a, n)),
                                          _p(_weights(b, m)), _p(_d(f)), _p(_d(g)), float(eps))


def marginal_error_matrix(C, f, g, eps, a=None, b=None) -> float:
    C = _d(C)
    n, m = C.shape
    return _L().ora_marginal_error_matrix(n, m, _p(C), _p(_weights(a, n)), _p(_weights(b, m)),
                                          _p(_d(f)), _p(_d(g)), float(eps))


def dual_objective_matrix(C, f, g, eps, a=None, b=None) -> float:
    C = _d(C)
    n, m = C.shape
    return _L().ora_dual_objective_matrix(n, m, _p(C), _p(_weights(a, n)), _p(_weights(b, m)),
                                          _p(_d(f)), _p(_d(g)), float(eps))


def plan_row_sums(x, y, f, g, eps, rows) -> np.ndarray:
    x, y = _pts(x), _pts(y)
    r = np.ascontiguousarray(rows, dtype=np.int64)
    out = np.empty(r.size)
    _L().ora_plan_row_sums(x.shape[0], y.shape[0], x.shape[1], _p(x), _p(y), _p(_d(f)),
                           _p(_d(g)), float(eps), _p(r), r.size, _p(out))
    return out


def plan_col_sums(x, y, f, g, eps, cols) -> np.ndarray:
    x, y = _pts(x), _pts(y)
    c = np.ascontiguousarray(cols, dtype=np.int64)
    out = np.empty(c.size)
    _L().ora_plan_col_sums(x.shape[0], y.shape[0], x.shape[1], _p(x), _p(y), _p(_d(f)),
                           _p(_d(g)), float(eps), _p(c), c.size, _p(out))
    return out


def center(f, g=None):
    """Appendix A: potentials are unique up to (f - s, g + s); compare after centering."""
    s = float(np.mean(f))
    return (np.asarray(f) - s) if g is None else (np.asarray(f) - s, np.asarray(g) + s)


# ------------------------------------------------------------- 1D / sort ---
def sort_rank(x):
    """Stable ascending sort of each row of x (B, n) (ties by index): perm, rank (int32)."""
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    x2 = x.reshape(-1, x.shape[-1]) if x.ndim > 1 else x.reshape(1, -1)
    B, n = x2.shape
    perm = np.empty((B, n), np.int32)
    rank = np.empty((B, n), np.int32)
    if _L().ora_sort_rank(B, n, _p(x2), _p(perm), _p(rank)) != 0:
        raise ValueError("NaN in sort input")
    return perm.reshape(x.shape), rank.reshape(x.shape)


def dualsort(xs_sorted, ys_sorted, sweeps: int = 0):
    """Alg. 2 (Jacobi) on sorted supports; sweeps=0 -> fixed point.  Returns (f, sweeps_done)."""
    xs, ys = _d(xs_sorted).ravel(), _d(ys_sorted).ravel()
    f = np.empty(xs.size)
    s = _L().ora_dualsort(xs.size, _p(xs), _p(ys), int(sweeps), _p(f))
    return f, s


def init_sort1d(x, y, sweeps: int = 0) -> np.ndarray:
    """Sec. 3.1 DualSort initializer for n = m, uniform weights, cost (x - y)^2:
    sort x (sigma) and y (rho), DualSort on the sorted cost, f0_{sigma(k)} = f_k."""
    x = np.asarray(x, np.float32).ravel()
    y = np.asarray(y, np.float32).ravel()
    if x.size != y.size:
        raise ValueError("sort1d initializer needs n == m (identity matching)")
    px, _ = sort_rank(x)
    py, _ = sort_rank(y)
    fs, _ = dualsort(x[px].astype(np.float64), y[py].astype(np.float64), sweeps)
    f0 = np.empty(x.size)
    f0[px] = fs
    return f0


# ------------------------------------------------------------- Gaussian ---
def _sym_fn(M, fn):
    """Symmetric matrix function by eigendecomposition (library eigh as one step)."""
    M = 0.5 * (M + M.T)
    w, V = np.linalg.eigh(M)
    return (V * fn(w)) @ V.T


def sqrtm(M):
    return _sym_fn(M, np.sqrt)


def inv_sqrtm(M):
    return _sym_fn(M, lambda w: 1.0 / np.sqrt(w))


def moments(x, w=None, ridge_rel: float = 1e-6):
    """Weighted mean m = sum_i w_i x_i and biased covariance
    sum_i w_i (x_i - m)(x_i - m)^T + ridge_rel * tr/d * I   (reading R-11)."""
    x = _pts(x)
    n, d = x.shape
    w = _weights(w, n)
    m = (w[:, None] * x).sum(0)
    xc = x - m
    S = (w[:, None] * xc).T @ xc
    S = S + ridge_rel * np.trace(S) / d * np.eye(d)
    return m, S


def monge_A(S1, S2):
    """A = S1^{-1/2} (S1^{1/2} S2 S1^{1/2})^{1/2} S1^{-1/2}, symmetrised."""
    r = sqrtm(S1)
    ri = inv_sqrtm(S1)
    A = ri @ sqrtm(r @ S2 @ r) @ ri
    return 0.5 * (A + A.T)


def gaussian_potential(xe, m_mu, m_nu, A):
    """f*(x) = ||x||^2 - (x - m_mu)^T A (x - m_mu) - 2 m_nu^T x  (Gaussian-Potential appendix,
    P:613-615, cost ||x-y||^2; reading R-4)."""
    xe = _pts(xe)
    xc = xe - m_mu
    return (xe * xe).sum(1) - np.einsum("ij,jk,ik->i", xc, A, xc) - 2.0 * xe @ m_nu


def bures2(S1, S2):
    """B^2(S1,S2) = tr(S1 + S2 - 2 (S1^{1/2} S2 S1^{1/2})^{1/2})  (Eq. 6)."""
    r = sqrtm(S1)
    return float(np.trace(S1) + np.trace(S2) - 2.0 * np.trace(sqrtm(r @ S2 @ r)))


def w2_gaussians(m1, S1, m2, S2):
    """W_2^2 between Gaussians, Eq. (6)."""
    return float(np.sum((np.asarray(m1) - np.asarray(m2)) ** 2)) + bures2(S1, S2)


def init_gaussian(x, y, a=None, b=None, ridge_rel: float = 1e-6):
    """Gaus initializer (Sec. 3.2): moments, A, evaluate the quadratic potential on
    the smaller side (n <= m -> on x, side 0; else on y, side 1, reading R-15)."""
    x, y = _pts(x), _pts(y)
    m_mu, S_mu = moments(x, a, ridge_rel)
    m_nu, S_nu = moments(y, b, ridge_rel)
    if x.shape[0] <= y.shape[0]:
        return gaussian_potential(x, m_mu, m_nu, monge_A(S_mu, S_nu)), 0
    return gaussian_potential(y, m_nu, m_mu, monge_A(S_nu, S_mu)), 1


# ------------------------------------------------------------------ GMM ---
def gmm_log_resp(x, weights, means, covs):
    """log p_k(x) of Eq. (7): log alpha_k + log N(x; m_k, S_k), normalised by LSE over k
    (the (2 pi)^{-d/2} factor cancels).  Cholesky S_k = L L^T (library step)."""
    x = _pts(x)
    K = len(weights)
    lp = np.empty((x.shape[0], K))
    for k in range(K):
        L = np.linalg.cholesky(_d(covs[k]))
        z = np.linalg.solve(L, (x - _d(means[k])).T)
        lp[:, k] = np.log(float(weights[k])) - 0.5 * (z * z).sum(0) - np.log(np.diag(L)).sum()
    mx = lp.max(1, keepdims=True)
    return lp - (mx + np.log(np.exp(lp - mx).sum(1, keepdims=True)))


def gmm_cost(mx, cx, my, cy):
    """C~_kl = ||m_k - m'_l||^2 + B^2(S_k, S'_l)  (Eq. 6)."""
    K, L = len(mx), len(my)
    C = np.empty((K, L))
    for k in range(K):
        for l in range(L):
            C[k, l] = w2_gaussians(_d(mx[k]), _d(cx[k]), _d(my[l]), _d(cy[l]))
    return C


def gmm_dual(gx: dict, gy: dict, eps, inner_tol=1e-12, inner_max_iter=2000000):
    """The K x K problem of the GMM initializer (Sec. 3.3, "regularized K x K OT problem",
    Eq. 6 costs): plain log-domain Sinkhorn (O2, Alg. 1 with omega = 1) between the mixture
    weights at the same eps (reading R-13), to inner_tol in fp64 -> f~, returned as the
    representative with sum_k a_k f~_k = 0 (f~ is defined up to a constant, R-29)."""
    C = gmm_cost(gx["means"], gx["covs"], gy["means"], gy["covs"])
    a = _d(gx["weights"])
    r = sinkhorn_matrix(C, eps, a=a, b=_d(gy["weights"]), tol=inner_tol, max_iter=inner_max_iter)
    return r.f - (a * r.f).sum() / a.sum(), r


def init_gmm(x, y, gx: dict, gy: dict, eps, inner_tol=1e-12, inner_max_iter=2000000):
    """GMM initializer (Sec. 3.3): f~ of the K x K Bures-cost problem (gmm_dual:
    plain Sinkhorn to inner_tol 1e-12, reading R-13); f0_i = sum_k f~_k p_k(x_i) on the
    smaller side."""
    x, y = _pts(x), _pts(y)
    if x.shape[0] > y.shape[0]:
        f, _ = init_gmm(y, x, gy, gx, eps, inner_tol, inner_max_iter)
        return f, 1
    ft, _ = gmm_dual(gx, gy, eps, inner_tol, inner_max_iter)
    P = np.exp(gmm_log_resp(x, gx["weights"], gx["means"], gx["covs"]))
    return P @ ft, 0


# ------------------------------------------------------------- Subsample ---
def subsample_extrapolate(x, z, gb, eps, rows=None) -> np.ndarray:
    """Eq. (8): f0_i = -eps log (1/ms) sum_j exp((gb_j - c(x_i, z_j))/eps)."""
    x, z, gb = _pts(x), _pts(z), _d(gb)
    r = None if rows is None else np.ascontiguousarray(rows, dtype=np.int64)
    out = np.empty(x.shape[0] if r is None else r.size)
    _L().ora_subsample_extrapolate(x.shape[0], z.shape[0], x.shape[1], _p(x), _p(z), _p(gb),
                                   float(eps), _p(out), _p(r), 0 if r is None else r.size)
    return out


def init_subsample(x, y, idx_x, idx_y, eps, inner_tol, inner_max_iter=10000, rows=None):
    """Subsample initializer (Sec. 3.4): inner Sinkhorn on the uniform subsamples
    w = x[idx_x], z = y[idx_y] at the same eps (reading R-14), then Eq. (8) from g-breve.
    Side 0 (f on x) when n <= m."""
    x, y = _pts(x), _pts(y)
    if x.shape[0] > y.shape[0]:
        f, _, inner = init_subsample(y, x, idx_y, idx_x, eps, inner_tol, inner_max_iter, rows)
        return f, 1, inner
    w, z = x[np.asarray(idx_x)], y[np.asarray(idx_y)]
    inner = sinkhorn(w, z, eps, tol=inner_tol, max_iter=inner_max_iter)
    return subsample_extrapolate(x, z, inner.g, eps, rows), 0, inner


# ----------------------------------------------------------- sharded (O9) ---
def column_partials(x_rows, y, f_rows, eps):
    """Per-shard column partials of the g-pass:
    (M_j, S_j) with M_j = max_i (f_i - C_ij)/eps and S_j = sum_i exp((f_i - C_ij)/eps - M_j)
    over the shard's rows.  Plain fp64 loops over the cost matrix of the shard."""
    C = cost_matrix(x_rows, y)
    V = (_d(f_rows)[:, None] - C) / eps
    M = V.max(0)
    return M, np.exp(V - M).sum(0)


def merge_partials(parts, b, eps):
    """Stable LSE merge of shard partials in rank order -> g_j = eps log b_j - eps LSE."""
    M = np.max([p[0] for p in parts], axis=0)
    S = np.zeros_like(M)
    for Mp, Sp in parts:
        S = S + Sp * np.exp(Mp - M)
    return eps * np.log(_d(b)) - eps * (M + np.log(S))


def soft_rank_sort(x, y, f, g, eps, z=None):
    """Soft ranks and soft sort (Sec. 3.1; NEXT-2) from potentials (f, g): the plan
    P_ij = exp((f_i + g_j - (x_i - y_j)^2)/eps) of Eq. (2), then the conditional means
        rank = (P z) / (P 1),   sort = (P^T x) / (P^T 1)
    (reading R-22; the paper's n P z and n P^T x whenever P has the uniform marginals).  z
    defaults to 1, ..., m (1-based ranks).  Plain fp64 matrix products."""
    x, y, f, g = _d(x).ravel(), _d(y).ravel(), _d(f).ravel(), _d(g).ravel()
    m = len(y)
    z = np.arange(1, m + 1, dtype=np.float64) if z is None else _d(z).ravel()
    C = (x[:, None] - y[None, :]) ** 2
    P = np.exp((f[:, None] + g[None, :] - C) / eps)
    return (P @ z) / P.sum(1), (P.T @ x) / P.sum(0)


def kmeans(x, init_idx, iters):
    """Lloyd's k-means (the k-means start of the GMM fit, "sklearn"; reading R-28)
    from centers x[init_idx]: `iters` times (assign every point to its nearest center in squared
    Euclidean distance, ties to the lowest k; move each non-empty cluster's center to its mean,
    an empty cluster keeps its center), then a final assignment to the returned centers.
    Returns (centers K x d, labels n)."""
    x = _pts(x)
    c = x[np.asarray(init_idx)].copy()

    def assign(c):
        d2 = ((x[:, None, :] - c[None, :, :]) ** 2).sum(-1)
        return np.argmin(d2, axis=1)   # (first minimum: the lowest k)

    for _ in range(iters):
        lab = assign(c)
        for k in range(len(c)):
            if np.any(lab == k):
                c[k] = x[lab == k].mean(0)
    return c, assign(c)


def _gmm_mstep(x, r, reg_covar):
    """M-step: n_k = sum_i r_ik (+ 10 eps, sklearn's guard), alpha_k = n_k / n,
    m_k = sum_i r_ik x_i / n_k, S_k = sum_i r_ik (x_i - m_k)(x_i - m_k)^T / n_k + reg I."""
    n, d = x.shape
    nk = r.sum(0) + 10 * np.finfo(np.float64).eps
    weights = nk / n
    means = (r.T @ x) / nk[:, None]
    covs = np.empty((r.shape[1], d, d))
    for k in range(r.shape[1]):
        diff = x - means[k]
        covs[k] = (r[:, k, None] * diff).T @ diff / nk[k] + reg_covar * np.eye(d)
    return weights, means, covs


def gmm_fit(x, K, init_idx, iters, reg_covar=1e-6, kmeans_iters=0, tol=0.0, return_iters=False):
    """EM for a K-component full-covariance GMM (NEXT-3; "we fit first two K-component
    GMMs", done with sklearn on the CPU in the paper).  Start (R-23): kmeans_iters = 0:
    weights 1/K, means x[init_idx], covariances the biased covariance of x + reg I;
    kmeans_iters > 0 (R-28, sklearn's init_params="kmeans"): the M-step of the one-hot
    responsibilities of kmeans(x, init_idx, kmeans_iters).  Each iteration, literally:
        E-step  r_ik = alpha_k N(x_i; m_k, S_k) / sum_l alpha_l N(x_i; m_l, S_l)   (gmm_log_resp)
        M-step  (_gmm_mstep).
    tol > 0 (sklearn's convergence rule, R-28): iteration k's E-step gives the mean
    log-likelihood ll_k of the current parameters; after its M-step, stop if |ll_k - ll_{k-1}| <
    tol (ll_0 = -inf).  Returns (weights, means, covs, mean log-likelihood of the returned
    parameters[, EM iterations run])."""
    x = _pts(x)
    n, d = x.shape
    if kmeans_iters > 0:
        _, lab = kmeans(x, init_idx, kmeans_iters)
        weights, means, covs = _gmm_mstep(x, np.eye(K)[lab], reg_covar)
    else:
        means = x[np.asarray(init_idx)].copy()
        m0 = x.mean(0)
        cov0 = (x - m0).T @ (x - m0) / n + reg_covar * np.eye(d)
        covs = np.repeat(cov0[None], K, axis=0)
        weights = np.full(K, 1.0 / K)
    ll_prev, done = -np.inf, 0
    for _ in range(iters):
        ll = gmm_loglik(x, weights, means, covs)
        r = np.exp(gmm_log_resp(x, weights, means, covs))
        weights, means, covs = _gmm_mstep(x, r, reg_covar)
        done += 1
        if tol > 0 and abs(ll - ll_prev) < tol:
            break
        ll_prev = ll
    out = (weights, means, covs, gmm_loglik(x, weights, means, covs))
    return out + (done,) if return_iters else out


def gmm_loglik(x, weights, means, covs):
    """Mean over points of log sum_k alpha_k N(x_i; m_k, S_k) (Cholesky, a library step)."""
    x = _pts(x)
    n, d = x.shape
    lp = np.empty((n, len(weights)))
    for k in range(len(weights)):
        L = np.linalg.cholesky(_d(covs[k]))
        z = np.linalg.solve(L, (x - _d(means[k])).T)
        lp[:, k] = np.log(float(weights[k])) - 0.5 * (z * z).sum(0) - np.log(np.diag(L)).sum() \
            - 0.5 * d * np.log(2 * np.pi)
    mx = lp.max(1, keepdims=True)
    return float(np.mean(mx[:, 0] + np.log(np.exp(lp - mx).sum(1))))


def sinkhorn_vjp(x, y, f, g, eps, zf, zg):
    """Implicit differentiation (NEXT-4) of the optimal potentials, dense fp64:
    H(f, g) = [a - P 1; b - P^T 1] (the gradient of Eq. (2)), J_H,(f,g) = -(1/eps) M with
    M = [[diag(P 1), P], [P^T, diag(P^T 1)]], so J_F^T z = eps J_H,.^T M^+ z with z
    projected on e^perp (e = (1, -1), the shift of (f, g)) and the min-norm M^+ z (numpy lstsq,
    a library step).  For C_ij = |x_i - y_j|^2:
        grad_x_i = 2 sum_j P_ij (w_f,i + w_g,j)(x_i - y_j), grad_y_j = 2 sum_i P_ij (w_f,i + w_g,j)(y_j - x_i),
        grad_a = eps w_f, grad_b = eps w_g.   Returns (grad_x, grad_y, grad_a, grad_b)."""
    x, y, f, g = _pts(x), _pts(y), _d(f).ravel(), _d(g).ravel()
    n, m = len(f), len(g)
    C = ((x[:, None, :] - y[None, :, :]) ** 2).sum(-1)
    P = np.exp((f[:, None] + g[None, :] - C) / eps)
    M = np.block([[np.diag(P.sum(1)), P], [P.T, np.diag(P.sum(0))]])
    e = np.concatenate([np.ones(n), -np.ones(m)])
    z = np.concatenate([_d(zf).ravel(), _d(zg).ravel()])
    z = z - (z @ e) / (e @ e) * e
    w = np.linalg.lstsq(M, z, rcond=None)[0]
    w = w - (w @ e) / (e @ e) * e
    wf, wg = w[:n], w[n:]
    S = P * (wf[:, None] + wg[None, :])
    gx = 2.0 * (S[:, :, None] * (x[:, None, :] - y[None, :, :])).sum(1)
    gy = 2.0 * (S[:, :, None] * (y[None, :, :] - x[:, None, :])).sum(0)
    return gx, gy, eps * wf, eps * wg


# ------------------------------------------------ general 1D: NW corner + Alg. 3/4 (NEXT-2)
def nw_corner_support(a_sorted, b_sorted, uniform=False):
    """North-west corner solution on sorted supports: its support edges (k, l) in walk
    order and the tree id of each edge.  A tie of the cumulative masses A_k = B_l before the
    end starts a new tree (the support graph is a forest).  Reading R-26: ties are exact
    — integer k m == l n for uniform weights, else fp64 cumulative sums of the (fp32) weights."""
    n, m = len(a_sorted), len(b_sorted)
    if uniform:
        Acum = lambda k: (k + 1) * m          # (k + 1)/n scaled by n m
        Bcum = lambda l: (l + 1) * n
    else:
        A = np.cumsum(np.asarray(a_sorted, np.float64))
        B = np.cumsum(np.asarray(b_sorted, np.float64))
        Acum, Bcum = (lambda k: A[k]), (lambda l: B[l])
    edges, tree = [], []
    k = l = t = 0
    while True:
        edges.append((k, l))
        tree.append(t)
        if k == n - 1 and l == m - 1:
            break
        ak, bl = Acum(k), Bcum(l)
        if ak < bl:
            k += 1
        elif bl < ak:
            l += 1
        else:
            k += 1
            l += 1
            t += 1
    return edges, tree


def dual_from_primal(C, edges, tree, max_rounds=100000):
    """Alg. 3 (Recover dual from primal) with Alg. 4 (UpdateTree), in reading R-26:
    f = 0; repeat {
      for every tree k (the first included, from f = 0 as DualSort, R-7):
          f_{s(k)} <- min_{i in T_k, j} c_ij - c_{iota(j),j} + f_{iota(j)} - (f_i - f_{s(k)})
      (the printed line 5 is the term i = s(k); a tree's sources move together — f_i - f_{s(k)}
      is fixed by its tight edges — so every source's feasibility bounds the root);
      for every tree: UpdateTree — walk its edges in pre-order from s(k):
          a new sink t:   g_t <- c_{s,t} - f_s;    a new source s:   f_s <- c_{s,t} - g_t
    } until no root moves (a root moves only if its bound is below it by more than
    1e-12 max(1, max|C|): its own tight edges give f_{s(k)} itself up to fp64 rounding).  The walk order of the NW staircase is a pre-order traversal from
    the tree's smallest source.  With n = m uniform (n one-edge trees) this is DualSort's Jacobi
    fixed point (Alg. 2, R-5/R-7).  Returns (f, g, rounds)."""
    C = _d(C)
    n, m = C.shape
    K = tree[-1] + 1
    trees = [[e for e, t in zip(edges, tree) if t == k] for k in range(K)]
    roots = [tr[0][0] for tr in trees]
    srcs = [sorted({i for (i, _) in tr}) for tr in trees]
    iota = np.full(m, -1)
    for (i, j) in edges:
        if iota[j] < 0 or i < iota[j]:
            iota[j] = i
    f, g = np.zeros(n), np.zeros(m)

    def update_tree(tr):
        seen_s, seen_t = {tr[0][0]}, set()
        for (i, j) in tr:
            if i in seen_s and j not in seen_t:
                g[j] = C[i, j] - f[i]
                seen_t.add(j)
            elif j in seen_t and i not in seen_s:
                f[i] = C[i, j] - g[j]
                seen_s.add(i)
    for tr in trees:
        update_tree(tr)
    tol = 1e-12 * max(1.0, float(np.abs(C).max()))
    for rounds in range(1, max_rounds + 1):
        fold = f.copy()
        base = -C[iota, np.arange(m)] + fold[iota]          # -g_j of the tight edge (iota(j), j)
        moved = False
        for k in range(K):
            s = roots[k]
            v = min(np.min(C[i, :] + base - (fold[i] - fold[s])) for i in srcs[k])
            if v < fold[s] - tol:   # R-26: the tree's own tight edges give f_s to rounding
                f[s] = v
                moved = True
        if not moved:
            return f, g, rounds
        for tr in trees:
            update_tree(tr)
    return f, g, max_rounds


def init_nw1d(x, y, a=None, b=None):
    """General 1D initializer (Sec. 3.1 with any n, m and weights; NEXT-2): sort x
    (sigma) and y (rho), the NW corner plan of (a_sigma, b_rho), its eps = 0 dual by
    Alg. 3 on the sorted cost (x_sigma_k - y_rho_l)^2, f0_{sigma(k)} = f~_k."""
    x = np.asarray(x, np.float32).ravel()
    y = np.asarray(y, np.float32).ravel()
    px, _ = sort_rank(x)
    py, _ = sort_rank(y)
    uniform = a is None and b is None
    a_s = None if a is None else np.asarray(a, np.float32).ravel()[px]
    b_s = None if b is None else np.asarray(b, np.float32).ravel()[py]
    if not uniform:
        a_s = np.full(x.size, 1.0 / x.size) if a_s is None else a_s
        b_s = np.full(y.size, 1.0 / y.size) if b_s is None else b_s
    edges, tree = nw_corner_support(np.ones(x.size) if uniform else a_s, np.ones(y.size) if uniform else b_s,
                                    uniform=uniform)
    xs, ys = x[px].astype(np.float64), y[py].astype(np.float64)
    C = (xs[:, None] - ys[None, :]) ** 2
    fs, _, _ = dual_from_primal(C, edges, tree)
    f0 = np.empty(x.size)
    f0[px] = fs
    return f0
