"""Device GMM fitting by EM (K16) through the C ABI (-m gpu):
parameters vs the oracle's EM (itself pinned to sklearn), the fitted GMM initializer end to end
at C3, and argument errors."""
import numpy as np
import pytest
import torch

from parity import centred, rel_inf
from workloads import gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2206_07630_b200 as sk
    return sk.Context(0)


def _close(gpu, ora, tol):
    g = gpu.cpu().numpy().astype(np.float64)
    return np.abs(g - ora).max() <= tol * max(1.0, np.abs(ora).max())


@pytest.mark.parametrize("n,d,K,iters", [(900, 3, 3, 12), (2500, 7, 5, 30), (16384, 16, 8, 20)])
def test_fit_parity(O, ctx, n, d, K, iters):
    import paper_2206_07630_b200 as sk
    if n == 16384:
        x = gen.c3().x
    else:
        rng = np.random.default_rng(n + d)
        cents = rng.standard_normal((K, d)) * 3
        x = (cents[rng.integers(0, K, n)] + rng.standard_normal((n, d)) * 0.7).astype(np.float32)
    idx = gen.gmm_start_idx(len(x), K, seed=n)
    g, ll = sk.sinkhorn_fit_gmm(ctx, torch.from_numpy(x).cuda(), K, idx, iters=iters)
    w, m, S, llo = O.gmm_fit(x, K, idx, iters, 1e-6)
    # fp64 on both sides (summation order differs); outputs are fp32 casts
    assert _close(g["weights"], w, 1e-6) and _close(g["means"], m, 1e-6) and _close(g["covs"], S, 1e-6)
    assert abs(ll - llo) <= 1e-9 * max(1.0, abs(llo))


@pytest.mark.parametrize("n,d,K,km,iters", [(900, 3, 3, 4, 0), (2500, 7, 5, 10, 8), (16384, 16, 8, 10, 20),
                                             (1000, 2, 6, 30, 3)])
def test_fit_kmeans_start_parity(O, ctx, n, d, K, km, iters):
    """R-28: Lloyd steps (hard assignments decided in fp64 on both sides) then the one-hot
    M-step and EM; iters = 0 checks the k-means start itself."""
    import paper_2206_07630_b200 as sk
    if n == 16384:
        x = gen.c3().x
    else:
        rng = np.random.default_rng(n + d + km)
        cents = rng.standard_normal((K, d)) * 3
        x = (cents[rng.integers(0, K, n)] + rng.standard_normal((n, d)) * 0.9).astype(np.float32)
    idx = gen.gmm_start_idx(len(x), K, seed=n + 1)
    g, ll = sk.sinkhorn_fit_gmm(ctx, torch.from_numpy(x).cuda(), K, idx, iters=iters, kmeans_iters=km)
    w, m, S, llo = O.gmm_fit(x, K, idx, iters, 1e-6, kmeans_iters=km)
    assert _close(g["weights"], w, 1e-6) and _close(g["means"], m, 1e-6) and _close(g["covs"], S, 1e-6)
    assert abs(ll - llo) <= 1e-9 * max(1.0, abs(llo))


@pytest.mark.parametrize("n,d,K,tol", [(2500, 7, 5, 1e-3), (16384, 16, 8, 1e-3), (3000, 4, 6, 1e-5)])
def test_fit_tol_stops_like_the_oracle(O, ctx, n, d, K, tol):
    """sklearn's convergence rule on the device (flags set by the M-step, later EM kernels
    return at once): the same EM step count and parameters as the oracle (itself pinned to
    sklearn's n_iter_)."""
    import paper_2206_07630_b200 as sk
    if n == 16384:
        x = gen.c3().x
    else:
        rng = np.random.default_rng(n + K)
        cents = rng.standard_normal((K, d)) * 3
        x = (cents[rng.integers(0, K, n)] + rng.standard_normal((n, d)) * 0.9).astype(np.float32)
    idx = gen.gmm_start_idx(len(x), K, seed=n + 2)
    g, ll, it = sk.sinkhorn_fit_gmm(ctx, torch.from_numpy(x).cuda(), K, idx, iters=100, kmeans_iters=10, tol=tol,
                                    return_iters=True)
    w, m, S, llo, ito = O.gmm_fit(x, K, idx, 100, 1e-6, kmeans_iters=10, tol=tol, return_iters=True)
    assert it == ito, (it, ito)
    assert _close(g["weights"], w, 1e-6) and _close(g["means"], m, 1e-6) and _close(g["covs"], S, 1e-6)
    assert abs(ll - llo) <= 1e-9 * max(1.0, abs(llo))


def test_fitted_gmm_initializer_c3(O, ctx):
    """The paper's GMM initializer with GMMs fitted on the device: f0 vs the oracle's
    initializer evaluated with the oracle's own fitted mixtures."""
    import paper_2206_07630_b200 as sk
    p = gen.c3()
    xd, yd = torch.from_numpy(p.x).cuda(), torch.from_numpy(p.y).cuda()
    ix, iy = gen.gmm_start_idx(p.n, 8, 3), gen.gmm_start_idx(p.m, 8, 4)
    gx, _ = sk.sinkhorn_fit_gmm(ctx, xd, 8, ix, iters=25)
    gy, _ = sk.sinkhorn_fit_gmm(ctx, yd, 8, iy, iters=25)
    pot, side = sk.sinkhorn_init_gmm(ctx, xd, yd, gx, gy, p.eps)
    ox = O.gmm_fit(p.x, 8, ix, 25, 1e-6)
    oy = O.gmm_fit(p.y, 8, iy, 25, 1e-6)
    f32 = lambda t: {"weights": t[0].astype(np.float32), "means": t[1].astype(np.float32),
                     "covs": t[2].astype(np.float32)}
    fo, so = O.init_gmm(p.x, p.y, f32(ox), f32(oy), p.eps)
    assert side == so
    assert rel_inf(centred(pot.cpu().numpy()), centred(fo), p.eps) <= 1e-4


def test_fit_errors(ctx):
    import paper_2206_07630_b200 as sk
    x = torch.rand(100, 4, device="cuda")
    with pytest.raises(sk.SinkhornError):
        sk.sinkhorn_fit_gmm(ctx, x, 3, [1, 1, 2])          # duplicate start
    with pytest.raises(sk.SinkhornError):
        sk.sinkhorn_fit_gmm(ctx, x, 3, [1, 2, 100])        # out of range
    with pytest.raises(sk.SinkhornError):
        sk.sinkhorn_fit_gmm(ctx, torch.rand(100, 257, device="cuda"), 2, [0, 1])   # d > 256
    with pytest.raises(sk.SinkhornError):
        sk.sinkhorn_fit_gmm(ctx, x, 2, [0, 1], kmeans_iters=-1)
    with pytest.raises(sk.SinkhornError):
        sk.sinkhorn_fit_gmm(ctx, x, 2, [0, 1], tol=-1.0)
    bad = x.clone(); bad[5, 1] = float("inf")
    with pytest.raises(sk.SinkhornError):
        sk.sinkhorn_fit_gmm(ctx, bad, 2, [0, 1])


@pytest.mark.parametrize("n,d,K,km,iters,tol", [(3000, 50, 10, 10, 6, 0.0), (2000, 40, 5, 0, 8, 0.0),
                                                (4000, 64, 8, 10, 100, 1e-3), (1200, 130, 3, 5, 4, 0.0)])
def test_fit_wide_parity(O, ctx, n, d, K, km, iters, tol):
    """d > 32 (the wide path: per-component Cholesky CTAs, responsibilities per point, the
    x x^T statistics by 64 x 64 tiles; P:388's word-embedding mixtures are d = 50, K up to 50)
    against the oracle's EM, k-means start and stopping rule included."""
    import paper_2206_07630_b200 as sk
    rng = np.random.default_rng(n + d)
    cents = rng.standard_normal((K, d)) * 2
    x = (cents[rng.integers(0, K, n)] + rng.standard_normal((n, d)) * 0.9).astype(np.float32)
    idx = gen.gmm_start_idx(n, K, seed=n + 3)
    g, ll, it = sk.sinkhorn_fit_gmm(ctx, torch.from_numpy(x).cuda(), K, idx, iters=iters, kmeans_iters=km, tol=tol,
                                    return_iters=True)
    w, m, S, llo, ito = O.gmm_fit(x, K, idx, iters, 1e-6, kmeans_iters=km, tol=tol, return_iters=True)
    assert it == ito, (it, ito)
    assert _close(g["weights"], w, 1e-6) and _close(g["means"], m, 1e-6) and _close(g["covs"], S, 1e-6)
    assert abs(ll - llo) <= 1e-9 * max(1.0, abs(llo))
