"""Implicit differentiation (K17) through the C ABI (-m gpu):
GPU VJP vs the oracle's dense VJP on the oracle's own converged potentials (fp32 cast), the
envelope closed form at a larger size on the GPU's own solve, and argument errors."""
import numpy as np
import pytest
import torch

from workloads import gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2206_07630_b200 as sk
    return sk.Context(0)


def _c(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def _rel(u, v):
    u, v = np.asarray(u, np.float64), np.asarray(v, np.float64)
    return np.abs(u - v).max() / max(np.abs(v).max(), 1e-12)


@pytest.mark.parametrize("n,m,d,epsf", [(40, 33, 2, 0.05), (256, 256, 2, 0.01), (200, 150, 16, 0.05),
                                        (64, 70, 64, 0.1), (1, 5, 3, 0.1), (90, 77, 100, 0.1), (70, 65, 256, 0.1)])
def test_vjp_parity_on_oracle_potentials(O, ctx, n, m, d, epsf):
    import paper_2206_07630_b200 as sk
    rng = np.random.default_rng(n * 3 + d)
    x = rng.standard_normal((n, d)).astype(np.float32)
    y = (rng.standard_normal((m, d)) * 0.8 + 0.4).astype(np.float32)
    eps = float(np.float32(epsf * gen.mean_sq_cost(x, y)))
    r = O.sinkhorn(x, y, eps, tol=1e-7, max_iter=200000)
    f32, g32 = r.f.astype(np.float32), r.g.astype(np.float32)
    zf = rng.standard_normal(n).astype(np.float32)
    zg = rng.standard_normal(m).astype(np.float32)
    grads, info = sk.sinkhorn_vjp(ctx, _c(x), _c(y), eps, _c(f32), _c(g32), _c(zf), _c(zg), cg_tol=1e-7)
    gx, gy, ga, gb = O.sinkhorn_vjp(x, y, f32, g32, eps, zf, zg)
    assert info["cg_relres"] <= 1e-7
    # fp32 plan entries (relative ~kappa ulp(f + g)) propagate through the solve: 1e-4 relative
    assert _rel(grads["x"].cpu().numpy(), gx) <= 1e-4, _rel(grads["x"].cpu().numpy(), gx)
    assert _rel(grads["y"].cpu().numpy(), gy) <= 1e-4
    assert _rel(grads["a"].cpu().numpy(), ga) <= 1e-4 and _rel(grads["b"].cpu().numpy(), gb) <= 1e-4


def test_vjp_envelope_at_scale(ctx):
    """z = (a, b) on the GPU's own C4-shaped solve (n = m = 4096, d = 3): the VJP must equal the
    envelope gradient 2 sum_j P_ij (x_i - y_j), recomputed here in fp64 from the returned pair."""
    import paper_2206_07630_b200 as sk
    p = gen.c4(n=4096)
    x, y = _c(p.x), _c(p.y)
    f, g, rep = sk.sinkhorn_solve(ctx, x, y, p.eps, tol=1e-6, mode="online")
    n = p.n
    grads, info = sk.sinkhorn_vjp(ctx, x, y, p.eps, f, g, torch.full((n,), 1 / n, device="cuda"),
                                  torch.full((n,), 1 / n, device="cuda"), cg_tol=1e-8)
    X, Y = p.x.astype(np.float64), p.y.astype(np.float64)
    F, G = f.cpu().numpy().astype(np.float64), g.cpu().numpy().astype(np.float64)
    env = np.zeros_like(X)
    for i0 in range(0, n, 512):
        C = ((X[i0:i0 + 512, None] - Y[None]) ** 2).sum(-1)
        P = np.exp((F[i0:i0 + 512, None] + G[None] - C) / p.eps)
        env[i0:i0 + 512] = 2 * (P.sum(1)[:, None] * X[i0:i0 + 512] - P @ Y)
    assert _rel(grads["x"].cpu().numpy(), env) <= 1e-3, _rel(grads["x"].cpu().numpy(), env)


def test_vjp_envelope_wide(ctx):
    """The envelope check at d = 128 (the wide plan pass, n = m = 2048, BJ.cfg5-shaped points) on
    the GPU's own K-chunked tensor-core solve."""
    import paper_2206_07630_b200 as sk
    p = gen.c5(n=2048, d=128, eps_factor=5e-2)
    x, y = _c(p.x), _c(p.y)
    f, g, rep = sk.sinkhorn_solve(ctx, x, y, p.eps, tol=1e-6, mode="online")
    n = p.x.shape[0]
    grads, info = sk.sinkhorn_vjp(ctx, x, y, p.eps, f, g, torch.full((n,), 1 / n, device="cuda"),
                                  torch.full((n,), 1 / n, device="cuda"), cg_tol=1e-8)
    X, Y = p.x.astype(np.float64), p.y.astype(np.float64)
    F, G = f.cpu().numpy().astype(np.float64), g.cpu().numpy().astype(np.float64)
    C = ((X[:, None] - Y[None]) ** 2).sum(-1)
    P = np.exp((F[:, None] + G[None] - C) / p.eps)
    env = 2 * (P.sum(1)[:, None] * X - P @ Y)
    assert _rel(grads["x"].cpu().numpy(), env) <= 1e-3, _rel(grads["x"].cpu().numpy(), env)


def test_vjp_errors(ctx):
    import paper_2206_07630_b200 as sk
    x, y = torch.rand(10, 2, device="cuda"), torch.rand(9, 2, device="cuda")
    f, g = torch.zeros(10, device="cuda"), torch.zeros(9, device="cuda")
    with pytest.raises(sk.SinkhornError):
        sk.sinkhorn_vjp(ctx, x, y, 0.0, f, g, f, g)
    with pytest.raises(sk.SinkhornError):
        sk.sinkhorn_vjp(ctx, torch.rand(10, 257, device="cuda"), torch.rand(9, 257, device="cuda"), 0.1, f, g, f, g)
