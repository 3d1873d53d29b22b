"""d in (64, 256] (only d > 256 is SK_EINVAL), -m gpu, through the C ABI:
the K-chunked tensor-core pass (K3, KC = 2..4 chunks of K = 64), the wide FFMA pass (K2 with
the output point's coordinates in shared memory), the stored cost build (K4) and the subsample
initializer's extension pass, each against the fp64 oracle on the same seeded inputs."""
import ctypes

import numpy as np
import pytest
import torch

from parity import INIT_RTOL, assert_obj_close, assert_pair_close, centred, count_tol, rel_inf
from workloads import gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2206_07630_b200 as sk
    return sk.Context(0)


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("d,sx,sy", [(65, 1, 1), (100, 1, 1), (128, 1, 1), (129, 1, 1), (192, 1, 1), (200, 1, 1),
                                     (256, 1, 1), (256, 1e4, 1e-3), (160, 1e30, 1e-30)])
def test_tc_tile_product_k_chunks(ctx, d, sx, sy):
    """The raw 128 x 128 tile product of the K-chunked images against fp64 (as at d <= 64)."""
    rng = np.random.default_rng(d)
    x = (rng.standard_normal((128, d)) * sx).astype(np.float32)
    y = (rng.standard_normal((128, d)) * sy).astype(np.float32)
    out = torch.empty((128, 128), dtype=torch.float32, device="cuda")
    xd, yd = _cuda(x), _cuda(y)
    ctx.check(ctx.lib.sk_selftest_tc_dot(ctx.h, d, ctypes.c_void_p(xd.data_ptr()), ctypes.c_void_p(yd.data_ptr()),
                                         ctypes.c_void_p(out.data_ptr())))
    ref = x.astype(np.float64) @ y.astype(np.float64).T
    scale = np.abs(x).astype(np.float64) @ np.abs(y).astype(np.float64).T
    err = np.abs(out.cpu().numpy() - ref) / scale
    assert err.max() < 4e-6, err.max()


def _problem(n, m, d, eps_factor, seed=0):
    p = gen.c5(n=max(n, m), d=d, eps_factor=eps_factor)
    x, y = p.x[:n].copy(), p.y[:m].copy()
    return x, y, float(np.float32(eps_factor * gen.mean_sq_cost(x, y)))


@pytest.mark.parametrize("n,m,d,tc", [(1100, 1300, 128, 1), (700, 515, 96, 1), (900, 1000, 256, 1), (1000, 777, 65, 1),
                                      (1100, 1300, 128, 0), (600, 700, 200, 0), (513, 515, 256, 0), (1100, 2100, 128, 0),
                                      (3000, 5000, 100, 0)])
def test_wide_solve_parity(O, ctx, n, m, d, tc):
    """Solve to tol (count within 2 %, P1) and lockstep potentials / objective (P2): tc = 1 the
    K-chunked tensor-core pass, tc = 0 the wide FFMA pass."""
    import paper_2206_07630_b200 as sk
    x, y, eps = _problem(n, m, d, 2e-2)
    c = sk.Context(0)
    c.set_tuning("tc", tc)
    f, g, rep = sk.sinkhorn_solve(c, _cuda(x), _cuda(y), eps, mode="online")
    c.close()
    ref = O.sinkhorn(x, y, eps)
    assert rep["converged"] and abs(rep["iterations"] - ref.iterations) <= count_tol(ref.iterations)
    lock = O.sinkhorn(x, y, eps, tol=0, max_iter=rep["iterations"])
    assert_pair_close(f.cpu().numpy(), g.cpu().numpy(), lock.f, lock.g, eps)
    assert_obj_close(rep["dual_objective"], lock.E, eps)


def test_wide_tc_matches_ffma(ctx):
    """The same d = 160 problem through K3 (3 chunks) and the wide K2: same count, potentials
    within fp32 noise."""
    import paper_2206_07630_b200 as sk
    x, y, eps = _problem(1536, 1536, 160, 1e-2)
    outs = []
    for tc in (1, 0):
        c = sk.Context(0)
        c.set_tuning("tc", tc)
        f, g, r = sk.sinkhorn_solve(c, _cuda(x), _cuda(y), eps, mode="online")
        outs.append((f.cpu().numpy(), r["iterations"]))
        c.close()
    (fa, ia), (fb, ib) = outs
    assert abs(ia - ib) <= 1
    fa, fb = fa - fa.mean(), fb - fb.mean()
    assert np.abs(fa - fb).max() <= 1e-4 * max(np.abs(fb).max(), 1e-3)


def test_wide_seeded_fallback_and_column_redo(O):
    """K3 at d = 128 with a 300 log2-unit seed margin: every seeded partial underflows, so every
    row is recomputed exactly in the merge and every seeded column pass is redone exactly."""
    import paper_2206_07630_b200 as sk
    x, y, eps = _problem(700, 1100, 128, 2e-2)
    c = sk.Context(0)
    c.set_tuning("tc_margin", 300)
    f, g, r = sk.sinkhorn_solve(c, _cuda(x), _cuda(y), eps, mode="online")
    c.close()
    assert r["iterations"] > 3
    lock = O.sinkhorn(x, y, eps, tol=0, max_iter=r["iterations"])
    assert_pair_close(f.cpu().numpy(), g.cpu().numpy(), lock.f, lock.g, eps)
    assert_obj_close(r["dual_objective"], lock.E, eps)


@pytest.mark.parametrize("d", [256, 100])
def test_wide_stored_parity(O, ctx, d):
    """Stored mode: K4's chunked cost build and the stored sweep at d > 64 (m % 4 == 0)."""
    import paper_2206_07630_b200 as sk
    x, y, eps = _problem(1000, 1200, d, 5e-2)
    f, g, rep = sk.sinkhorn_solve(ctx, _cuda(x), _cuda(y), eps, mode="stored")
    ref = O.sinkhorn(x, y, eps)
    assert rep["converged"] and abs(rep["iterations"] - ref.iterations) <= count_tol(ref.iterations)
    lock = O.sinkhorn(x, y, eps, tol=0, max_iter=rep["iterations"])
    assert_pair_close(f.cpu().numpy(), g.cpu().numpy(), lock.f, lock.g, eps)
    assert_obj_close(rep["dual_objective"], lock.E, eps)


@pytest.mark.parametrize("mode,d,tc", [("online", 128, 1), ("online", 256, 1), ("online", 200, 0), ("stored", 200, 1)])
def test_wide_sharded_bit_identical(O, ctx, mode, d, tc):
    """Row-sharded (emulated W = 1, 2, 4) at d > 64 on the tensor-core pass (tc = 1) and on the
    wide FFMA pass with its fused premerge (tc = 0): bit-identical across world sizes and with the
    unsharded entry; lockstep vs the oracle."""
    import paper_2206_07630_b200 as sk
    x, y, eps = _problem(6000, 2100, d, 3e-2)
    xd, yd = _cuda(x), _cuda(y)
    c = sk.Context(0)
    c.set_tuning("tc", tc)
    outs = {W: sk.sinkhorn_solve_sharded_emulated(c, W, xd, yd, eps, mode=mode) for W in (1, 2, 4)}
    f1, g1, r1 = outs[1]
    for W in (2, 4):
        f, g, r = outs[W]
        assert torch.equal(f, f1) and torch.equal(g, g1) and r["iterations"] == r1["iterations"], W
    fu, gu, ru = sk.sinkhorn_solve(c, xd, yd, eps, mode=mode)
    c.close()
    if mode == "online":
        assert ru["iterations"] == r1["iterations"] and torch.equal(fu, f1) and torch.equal(gu, g1)
    else:   # (the unsharded stored sweep recomputes a failing column in its merge: fp32 rounding)
        assert abs(ru["iterations"] - r1["iterations"]) <= 1
    lock = O.sinkhorn(x, y, eps, tol=0, max_iter=r1["iterations"])
    assert_pair_close(f1.cpu().numpy(), g1.cpu().numpy(), lock.f, lock.g, eps)


@pytest.mark.parametrize("d", [128, 256])
def test_wide_subsample_init(O, ctx, d):
    """Subsample initializer at d > 64: inner solve (K3 / wide K2) in lockstep, the Eq. (8)
    extension pass (wide K2) against the oracle's extrapolation from the lockstep g~."""
    import paper_2206_07630_b200 as sk
    x, y, eps = _problem(2600, 3000, d, 2e-2)
    rng = np.random.default_rng(d)
    ix = np.sort(rng.choice(2600, 400, replace=False)).astype(np.int32)
    iy = np.sort(rng.choice(3000, 300, replace=False)).astype(np.int32)
    tol = 1e-4
    pot, side, inner = sk.sinkhorn_init_subsample(ctx, _cuda(x), _cuda(y), _cuda(ix), _cuda(iy), eps, tol)
    assert side == 0
    w, z = x[ix], y[iy]
    ref_in = O.sinkhorn(w, z, eps, tol=tol)
    assert abs(inner["iterations"] - ref_in.iterations) <= count_tol(ref_in.iterations)
    lock = O.sinkhorn(w, z, eps, tol=0, max_iter=inner["iterations"])
    ref = O.subsample_extrapolate(x, z, lock.g, eps)
    got = pot.cpu().numpy()
    assert rel_inf(got - got.mean(), ref - ref.mean(), eps) <= INIT_RTOL


@pytest.mark.parametrize("n,m,d", [(1500, 1600, 65), (2000, 1900, 128), (3000, 3100, 256), (700, 800, 200)])
def test_wide_gaussian_init(O, ctx, n, m, d):
    """Gaussian initializer at d > 64 (moments by 64 x 64 output tiles, the Newton-Schulz square
    roots over the whole grid in one cooperative launch, the potential with A in L2) against
    the oracle; correlated x, shifted y, non-uniform a; n > m swaps the side."""
    import paper_2206_07630_b200 as sk
    rng = np.random.default_rng(d + n)
    G = rng.standard_normal((d, d)) / np.sqrt(d)
    x = (rng.standard_normal((n, d)) @ G.T).astype(np.float32)
    y = (rng.standard_normal((m, d)) * 0.7 + 0.4).astype(np.float32)
    a = gen.random_weights(n, rng)
    pot, side = sk.sinkhorn_init_gaussian(ctx, _cuda(x), _cuda(y), a=_cuda(a))
    ref, so = O.init_gaussian(x, y, a=a)
    assert side == so
    eps = 0.01 * gen.mean_sq_cost(x, y)
    assert rel_inf(centred(pot.cpu().numpy()), centred(ref), eps) <= INIT_RTOL


def test_wide_gaussian_init_then_solve(O, ctx):
    """End to end at d = 128: the Gaussian potential seeds the K-chunked tensor-core solve; fewer
    sweeps than the zero init, lockstep vs the oracle from the same f0."""
    import paper_2206_07630_b200 as sk
    x, y, eps = _problem(2048, 2048, 128, 1e-2)
    f0, side = sk.sinkhorn_init_gaussian(ctx, _cuda(x), _cuda(y))
    f, g, rep = sk.sinkhorn_solve(ctx, _cuda(x), _cuda(y), eps, f_init=f0, mode="online")
    _, _, rz = sk.sinkhorn_solve(ctx, _cuda(x), _cuda(y), eps, mode="online")
    assert rep["converged"] and rep["iterations"] < rz["iterations"]
    lock = O.sinkhorn(x, y, eps, tol=0, max_iter=rep["iterations"], f0=f0.cpu().numpy())
    assert_pair_close(f.cpu().numpy(), g.cpu().numpy(), lock.f, lock.g, eps)


def _mixture(rng, K, d, shift):
    """K components: weights, means N(shift, 4 I), covariances A A^T / d + 0.2 I (fp32)."""
    w = rng.uniform(0.5, 1.5, K)
    mu = shift + 2.0 * rng.standard_normal((K, d))
    A = rng.standard_normal((K, d, d))
    cov = np.einsum("kij,klj->kil", A, A) / d + 0.2 * np.eye(d)
    return {"weights": (w / w.sum()).astype(np.float32), "means": mu.astype(np.float32),
            "covs": cov.astype(np.float32)}


def _sample(rng, g, n):
    K, d = g["means"].shape
    w = g["weights"].astype(np.float64)
    comp = rng.choice(K, n, p=w / w.sum())
    L = np.linalg.cholesky(g["covs"].astype(np.float64))
    z = rng.standard_normal((n, d))
    return (g["means"][comp] + np.einsum("nij,nj->ni", L[comp], z)).astype(np.float32)


@pytest.mark.parametrize("d,Kx,Ky,n,m", [(96, 4, 3, 1500, 1700), (256, 3, 4, 1200, 1100)])
def test_wide_gmm_init(O, ctx, d, Kx, Ky, n, m):
    """GMM initializer at d > 64 with given mixtures (Eq. 6 Bures costs from per-pair Newton-Schulz
    square roots, the K x K problem, Cholesky responsibilities) against the oracle; n > m swaps."""
    import paper_2206_07630_b200 as sk
    rng = np.random.default_rng(d)
    gx, gy = _mixture(rng, Kx, d, 0.0), _mixture(rng, Ky, d, 0.5)
    x, y = _sample(rng, gx, n), _sample(rng, gy, m)
    eps = float(np.float32(0.05 * gen.mean_sq_cost(x, y)))
    pot, side = sk.sinkhorn_init_gmm(ctx, _cuda(x), _cuda(y), {k: _cuda(v) for k, v in gx.items()},
                                     {k: _cuda(v) for k, v in gy.items()}, eps)
    ref, so = O.init_gmm(x, y, gx, gy, eps)
    assert side == so
    assert rel_inf(centred(pot.cpu().numpy()), centred(ref), eps) <= INIT_RTOL


def test_wide_error_contract(ctx):
    """d = 257 is SK_EINVAL."""
    import paper_2206_07630_b200 as sk
    x = torch.rand(64, 257, device="cuda")
    with pytest.raises(sk.SinkhornError, match="SK_EINVAL"):
        sk.sinkhorn_solve(ctx, x, x, 0.1)
    with pytest.raises(sk.SinkhornError, match="SK_EINVAL"):
        sk.sinkhorn_init_gaussian(ctx, x, x)


def _lse_rows(Z):
    mx = Z.max(1, keepdims=True)
    return (mx + np.log(np.exp(Z - mx).sum(1, keepdims=True))).ravel()


@pytest.mark.parametrize("d", [256, 160])
def test_wide_tc_full_launch_first_sweep_sampled(O, ctx, d):
    """K3 with K chunks at a launch size with many tiles per item (n = m = 16384, BJ.cfg5 recipe
    at d): the first sweep from f0 = 0 — g1 on 256 sampled columns and f1 (from the returned g1)
    on 256 sampled rows — against fp64 log-sum-exps of the exact costs."""
    import paper_2206_07630_b200 as sk
    p = gen.c5(n=16384, d=d, eps_factor=1e-2)
    n = p.x.shape[0]
    f, g, rep = sk.sinkhorn_solve(ctx, _cuda(p.x), _cuda(p.y), p.eps, tol=1e-12, max_iter=1, mode="online")
    f, g = f.cpu().numpy().astype(np.float64), g.cpu().numpy().astype(np.float64)
    X, Y, eps = p.x.astype(np.float64), p.y.astype(np.float64), float(p.eps)
    rng = np.random.default_rng(d)
    cols = rng.choice(n, 256, replace=False)
    rows = rng.choice(n, 256, replace=False)
    x2, y2 = (X ** 2).sum(1), (Y ** 2).sum(1)
    g_ref = O.g_update(p.x, p.y, np.zeros(n), eps, cols=cols)
    C2 = x2[rows, None] + y2[None, :] - 2 * X[rows] @ Y.T         # sampled rows x all columns
    f_ref = eps * np.log(1.0 / n) - eps * _lse_rows((g[None, :] - C2) / eps)
    scale = max(np.abs(g_ref).max(), eps)
    assert np.abs(g[cols] - g_ref).max() <= 1e-4 * scale, np.abs(g[cols] - g_ref).max() / scale
    assert np.abs(f[rows] - f_ref).max() <= 1e-4 * max(np.abs(f_ref).max(), eps)


def test_wide_relaxation_and_adaptive(O, ctx):
    """The accelerations on the K-chunked tensor-core path (d = 128): relaxation omega = 1.2 and
    adaptive momentum (window 10) against the oracle's counts and lockstep pairs."""
    import paper_2206_07630_b200 as sk
    x, y, eps = _problem(1100, 1300, 128, 2e-2)
    f, g, rep = sk.sinkhorn_solve(ctx, _cuda(x), _cuda(y), eps, mode="online", omega=1.2)
    ref = O.sinkhorn(x, y, eps, omega=1.2)
    assert rep["converged"] and abs(rep["iterations"] - ref.iterations) <= count_tol(ref.iterations)
    lock = O.sinkhorn(x, y, eps, tol=0, max_iter=rep["iterations"], omega=1.2)
    assert_pair_close(f.cpu().numpy(), g.cpu().numpy(), lock.f, lock.g, eps)
    f, g, rep = sk.sinkhorn_solve(ctx, _cuda(x), _cuda(y), eps, mode="online", adaptive=10)
    ref = O.sinkhorn_adaptive(x, y, eps, adapt_iters=10)
    assert rep["converged"] and abs(rep["iterations"] - ref.iterations) <= count_tol(ref.iterations)
    lock = O.sinkhorn_adaptive(x, y, eps, adapt_iters=10, tol=0, max_iter=rep["iterations"])
    assert_pair_close(f.cpu().numpy(), g.cpu().numpy(), lock.f, lock.g, eps)
