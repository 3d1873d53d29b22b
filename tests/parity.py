"""Tolerances and comparison helpers for CUDA-vs-oracle parity (readings R-17..R-19).

These helpers hold no arithmetic of the method: centring (Appendix A), max-norm
relative errors and count tolerances only.
"""
import math

import numpy as np

POT_RTOL = 1e-4      # centred potentials, rel-inf (BJ.ns "1e-4 relative", reading R-18)
OBJ_RTOL = 1e-5      # dual objective, relative (BJ.ns)
INIT_RTOL = 1e-4     # initializer potentials after centring


def centred(f, g=None):
    f = np.asarray(f, np.float64)
    s = f.mean()
    if g is None:
        return f - s
    return f - s, np.asarray(g, np.float64) + s


def rel_inf(u, v, eps):
    """||u - v||_inf / max(||v||_inf, eps)  (R-18)."""
    u, v = np.asarray(u, np.float64), np.asarray(v, np.float64)
    return float(np.abs(u - v).max() / max(np.abs(v).max(), eps))


def count_tol(L_ora: int) -> int:
    """|L_gpu - L_ora| <= max(1, ceil(0.02 L_ora))  (BJ.ns "within 2%", R-19)."""
    return max(1, math.ceil(0.02 * L_ora))


def assert_pair_close(f, g, fo, go, eps, rtol=POT_RTOL, what=""):
    fc, gc = centred(f, g)
    foc, goc = centred(fo, go)
    ef, eg = rel_inf(fc, foc, eps), rel_inf(gc, goc, eps)
    assert ef <= rtol and eg <= rtol, f"{what}: centred potentials rel-inf f={ef:.3e} g={eg:.3e} > {rtol}"
    return ef, eg


def assert_obj_close(E, Eo, eps, rtol=OBJ_RTOL, what=""):
    r = abs(E - Eo) / max(abs(Eo), eps)
    assert r <= rtol, f"{what}: dual objective rel err {r:.3e} > {rtol} (gpu {E!r}, oracle {Eo!r})"
    return r


def plan_marginal_error(x, y, f, g, eps, a=None, b=None, chunk=2048):
    """fp64 L1 marginal error of the plan of (f, g) — a property check of CUDA outputs,
    written here (not via the oracle) so no oracle call takes a CUDA value as input."""
    x = np.asarray(x, np.float64).reshape(len(f), -1)
    y = np.asarray(y, np.float64).reshape(len(g), -1)
    f, g = np.asarray(f, np.float64), np.asarray(g, np.float64)
    n, m = len(f), len(g)
    a = np.full(n, 1.0 / n) if a is None else np.asarray(a, np.float64)
    b = np.full(m, 1.0 / m) if b is None else np.asarray(b, np.float64)
    col = np.zeros(m)
    err = 0.0
    for i0 in range(0, n, chunk):
        xi = x[i0:i0 + chunk]
        C = (xi ** 2).sum(1)[:, None] + (y ** 2).sum(1)[None, :] - 2 * xi @ y.T
        P = np.exp((f[i0:i0 + chunk, None] + g[None, :] - C) / eps)
        err += np.abs(P.sum(1) - a[i0:i0 + chunk]).sum()
        col += P.sum(0)
    return err + np.abs(col - b).sum()
