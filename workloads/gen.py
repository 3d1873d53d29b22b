"""Seeded synthetic inputs for the five BASELINE.json configs (C1..C5).

This module is shared by the oracle tests, the CUDA parity tests, ``smoke()``
and ``bench.py``.  It holds *no* arithmetic of the method (no cost matrix, no
soft-min, no potential): it only draws points, weights, subsample indices and
GMM parameters, and fixes the problem's scalar ``eps`` from the config recipe
(``eps = c * mean(C)``, the mean of the squared-L2 cost over all pairs, which is
a workload definition in BASELINE.json, evaluated in fp64 by the closed form
mean|x|^2 + mean|y|^2 - 2 <xbar, ybar> for uniform weights).

Every array is produced by ``numpy.random.default_rng(seed)`` in a fixed draw
order and returned as C-contiguous float32 (points, weights) or int32 (indices).
The recipes are the ones DESIGN.md "Input recipe" lists.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np


@dataclasses.dataclass
class Problem:
    """One OT problem instance (or a batch of B independent ones)."""
    name: str
    x: np.ndarray            # (n, d) or (B, n, d) float32
    y: np.ndarray            # (m, d) or (B, m, d) float32; shared target when y_shared
    eps: float               # fp32-representable
    a: Optional[np.ndarray] = None  # None = uniform 1/n
    b: Optional[np.ndarray] = None  # None = uniform 1/m
    tol: float = 1e-3
    max_iter: int = 10000
    y_shared: bool = False
    batch: int = 1
    extra: dict = dataclasses.field(default_factory=dict)

    @property
    def n(self) -> int:
        return self.x.shape[-2]

    @property
    def m(self) -> int:
        return self.y.shape[-2]

    @property
    def d(self) -> int:
        return self.x.shape[-1]


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


def mean_sq_cost(x: np.ndarray, y: np.ndarray) -> float:
    """Mean over all (i, j) of ||x_i - y_j||^2 for uniform weights (fp64).

    Used only to fix eps from the config recipe ("eps = 0.01*mean(C)").
    """
    x64 = np.asarray(x, np.float64).reshape(-1, x.shape[-1])
    y64 = np.asarray(y, np.float64).reshape(-1, y.shape[-1])
    return float((x64 ** 2).sum(1).mean() + (y64 ** 2).sum(1).mean()
                 - 2.0 * x64.mean(0) @ y64.mean(0))


def _eps32(v: float) -> float:
    return float(np.float32(v))


# --------------------------------------------------------------------------- C1
def c1(n: int = 256, seed: int = 0, eps_factor: float = 0.01) -> Problem:
    """BJ.cfg1: n=m=256, d=2; x~N(0,I2); y~N((1,1),S), S=LL^T+0.1I, L_ij~N(0,0.5).

    N(0,0.5) is read as variance 0.5 (reading R-20)."""
    rng = np.random.default_rng(seed)
    L = rng.normal(0.0, np.sqrt(0.5), (2, 2))
    S = L @ L.T + 0.1 * np.eye(2)
    x = rng.standard_normal((n, 2))
    y = np.array([1.0, 1.0]) + rng.standard_normal((n, 2)) @ np.linalg.cholesky(S).T
    x, y = _f32(x), _f32(y)
    eps = _eps32(eps_factor * mean_sq_cost(x, y))
    return Problem("c1", x, y, eps, extra={"S": S})


# --------------------------------------------------------------------------- C2
def c2(B: int = 1024, n: int = 1024, seed: int = 0, eps: float = 1e-3) -> Problem:
    """BJ.cfg2: B vectors of n values ~U[0,1); shared target y_j = j/(n-1); eps=1e-3."""
    rng = np.random.default_rng(seed)
    x = rng.random((B, n), dtype=np.float32).reshape(B, n, 1)
    y = (np.arange(n, dtype=np.float64) / max(n - 1, 1)).astype(np.float32).reshape(n, 1)
    return Problem("c2", _f32(x), _f32(y), _eps32(eps), y_shared=True, batch=B)


# --------------------------------------------------------------------------- C3
def gmm_params(K: int, d: int, rng) -> dict:
    """Mixture recipe of BJ.cfg3: means ~ N(0, 4I), covariances ~ Wishart(d, I/d), uniform weights."""
    means = rng.normal(0.0, 2.0, (K, d))
    covs = np.empty((K, d, d))
    for k in range(K):
        G = rng.standard_normal((d, d)) / np.sqrt(d)   # rows ~ N(0, I/d), df = d
        covs[k] = G.T @ G
    weights = np.full(K, 1.0 / K)
    return {"weights": weights, "means": means, "covs": covs}


def sample_gmm(params: dict, n: int, rng) -> np.ndarray:
    K, d = params["means"].shape
    labels = rng.choice(K, size=n, p=params["weights"])
    z = rng.standard_normal((n, d))
    out = np.empty((n, d))
    for k in range(K):
        sel = labels == k
        Lk = np.linalg.cholesky(params["covs"][k])
        out[sel] = params["means"][k] + z[sel] @ Lk.T
    return out


def c3(n: int = 16384, K: int = 8, d: int = 16, eps_factor: float = 0.01) -> Problem:
    """BJ.cfg3: d=16, x and y from independently seeded 8-component GMMs (seeds 0 and 1)."""
    rx, ry = np.random.default_rng(0), np.random.default_rng(1)
    px = gmm_params(K, d, rx)
    x = sample_gmm(px, n, rx)
    py = gmm_params(K, d, ry)
    y = sample_gmm(py, n, ry)
    x, y = _f32(x), _f32(y)
    eps = _eps32(eps_factor * mean_sq_cost(x, y))
    f32p = lambda p: {k: _f32(v) for k, v in p.items()}
    return Problem("c3", x, y, eps, extra={"gmm_x": f32p(px), "gmm_y": f32p(py)})


def gmm_start_idx(n: int, K: int, seed: int) -> np.ndarray:
    """Start indices of the device GMM fit (NEXT-3, R-23): K distinct points drawn uniformly
    without replacement (C3: seed 3 for x, seed 4 for y)."""
    return np.random.default_rng(seed).choice(n, K, replace=False).astype(np.int32)


# --------------------------------------------------------------------------- C4
def _rgb_mixture(n: int, rng, clusters: int = 12) -> np.ndarray:
    centers = rng.uniform(0.1, 0.9, (clusters, 3))
    stds = rng.uniform(0.03, 0.15, clusters)
    w = rng.dirichlet(np.full(clusters, 2.0))
    labels = rng.choice(clusters, size=n, p=w)
    pts = centers[labels] + rng.standard_normal((n, 3)) * stds[labels, None]
    return np.clip(pts, 0.0, 1.0)


def c4(n: int = 262144, ns: int = 4096, eps: float = 1e-2) -> Problem:
    """BJ.cfg4: RGB-pixel-shaped points in [0,1]^3 from 12-cluster mixtures (x: seed 0, y: seed 1);
    subsample indices (seed 2) of size ns per side without replacement."""
    x = _rgb_mixture(n, np.random.default_rng(0))
    y = _rgb_mixture(n, np.random.default_rng(1))
    r2 = np.random.default_rng(2)
    ns = min(ns, n)
    idx_x = np.sort(r2.choice(n, ns, replace=False)).astype(np.int32)
    idx_y = np.sort(r2.choice(n, ns, replace=False)).astype(np.int32)
    return Problem("c4", _f32(x), _f32(y), _eps32(eps),
                   extra={"idx_x": idx_x, "idx_y": idx_y})


# --------------------------------------------------------------------------- C5
def c5(n: int = 65536, d: int = 64, eps_factor: float = 1e-2) -> Problem:
    """BJ.cfg5: x ~ N(0, diag(k^-1)), y ~ N(0.5*1, diag(k^-1)), k=1..d, then L2-normalised rows."""
    rng = np.random.default_rng(0)
    sd = 1.0 / np.sqrt(np.arange(1, d + 1, dtype=np.float64))
    x = rng.standard_normal((n, d)) * sd
    y = 0.5 + rng.standard_normal((n, d)) * sd
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    y /= np.linalg.norm(y, axis=1, keepdims=True)
    x, y = _f32(x), _f32(y)
    eps = _eps32(eps_factor * mean_sq_cost(x, y))
    return Problem("c5", x, y, eps)


CONFIGS = {"c1": c1, "c2": c2, "c3": c3, "c4": c4, "c5": c5}


def random_weights(n: int, rng) -> np.ndarray:
    """Positive weights summing to 1 (fp32), for non-uniform parity cases."""
    w = rng.uniform(0.5, 1.5, n)
    return _f32(w / w.sum())
