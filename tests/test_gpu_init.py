"""Initializer parity (-m gpu): Gaussian (Sec. 3.2), GMM (Sec. 3.3), Subsample (Sec. 3.4)."""
import numpy as np
import pytest
import torch

from parity import INIT_RTOL, centred, rel_inf
from workloads import gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2206_07630_b200 as sk
    return sk.Context(0)


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("n,m,d", [(256, 256, 2), (5000, 3000, 3), (2000, 2100, 16), (1500, 1600, 64)])
def test_gaussian_init(O, ctx, n, m, d):
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


def test_gaussian_special_cases(ctx):
    import paper_2206_07630_b200 as sk
    rng = np.random.default_rng(3)
    x = rng.standard_normal((400, 3)).astype(np.float32)
    pot, _ = sk.sinkhorn_init_gaussian(ctx, _cuda(x), _cuda(x))
    assert float(pot.max() - pot.min()) < 1e-4       # equal moments -> A = I -> constant


def test_gmm_init_c3_shape(O, ctx):
    import paper_2206_07630_b200 as sk
    p = gen.c3(n=2048)
    gx = {k: _cuda(v) for k, v in p.extra["gmm_x"].items()}
    gy = {k: _cuda(v) for k, v in p.extra["gmm_y"].items()}
    pot, side = sk.sinkhorn_init_gmm(ctx, _cuda(p.x), _cuda(p.y), gx, gy, p.eps)
    ref, so = O.init_gmm(p.x, p.y, p.extra["gmm_x"], p.extra["gmm_y"], p.eps)
    assert side == so == 0
    assert rel_inf(centred(pot.cpu().numpy()), centred(ref), p.eps) <= INIT_RTOL


def test_gmm_single_component_constant(ctx):
    import paper_2206_07630_b200 as sk
    rng = np.random.default_rng(4)
    x = rng.standard_normal((100, 2)).astype(np.float32)
    y = rng.standard_normal((120, 2)).astype(np.float32)
    g1 = {"weights": _cuda(np.ones(1, np.float32)), "means": _cuda(np.zeros((1, 2), np.float32)),
          "covs": _cuda(np.eye(2, dtype=np.float32)[None])}
    pot, _ = sk.sinkhorn_init_gmm(ctx, _cuda(x), _cuda(y), g1, g1, 0.5)
    assert float(pot.max() - pot.min()) == 0.0


@pytest.mark.parametrize("n,ns", [(20000, 1500), (3000, 3000), (5000, 1)])
def test_subsample_init(O, ctx, n, ns):
    import paper_2206_07630_b200 as sk
    p = gen.c4(n=n, ns=ns)
    tol = 1e-4
    pot, side, inner = sk.sinkhorn_init_subsample(ctx, _cuda(p.x), _cuda(p.y), _cuda(p.extra["idx_x"]),
                                                  _cuda(p.extra["idx_y"]), p.eps, tol)
    _, so, rin = O.init_subsample(p.x, p.y, p.extra["idx_x"], p.extra["idx_y"], p.eps, tol)
    assert side == so == 0
    from parity import count_tol
    assert abs(inner["iterations"] - rin.iterations) <= count_tol(rin.iterations)
    # lockstep: the oracle's inner solve replays exactly the GPU's inner sweep count, then Eq. (8)
    w, z = p.x[p.extra["idx_x"]], p.y[p.extra["idx_y"]]
    lock = O.sinkhorn(w, z, p.eps, tol=0, max_iter=inner["iterations"])
    ref = O.subsample_extrapolate(p.x, z, lock.g, p.eps)
    assert rel_inf(centred(pot.cpu().numpy()), centred(ref), p.eps) <= INIT_RTOL


@pytest.mark.parametrize("n,m,d,ns,ms,eps_f,cap,shift", [(7000, 9000, 3, 1500, 1100, 0.01, 0, 0.0),
                                                          (6000, 6000, 2, 700, 800, 0.003, 60, 1.0),
                                                          (8000, 9000, 4, 1200, 3100, 0.05, 0, 0.0),
                                                          (5000, 5000, 1, 600, 4737, 0.05, 0, 0.0)])
def test_subsample_inner_grid_solver(O, ctx, n, m, d, ns, ms, eps_f, cap, shift):
    """K20 (the grid-persistent inner solve), side 0 (n <= m): ragged ns != ms, d = 1..4, point
    counts past the one-round-per-CTA limit (4737 > 32 x 148), and a small eps whose first seeded
    sweeps move the LSEs by more than the seeded range (the exact redo of a point group) - run for
    `cap` sweeps on clouds shifted apart (on overlapping clouds the centred potentials span only
    ~0.01 of max |q|^2, so fp32's ulp(|q|^2) / eps rounding alone is 1.3e-4 of them after 60
    sweeps on both paths, tools/k20_check.py).  The inner report (L, err, E) against the oracle's inner solve, the potential in
    lockstep, and the same through the multi-kernel path (sk_set_tuning grid_solver 0)."""
    import paper_2206_07630_b200 as sk
    from parity import assert_obj_close, count_tol
    rng = np.random.default_rng(n + d)
    x = rng.random((n, d)).astype(np.float32)
    y = (rng.random((m, d)) * 0.9 + 0.05 + shift).astype(np.float32)
    ix = np.sort(rng.choice(n, ns, replace=False)).astype(np.int32)
    iy = np.sort(rng.choice(m, ms, replace=False)).astype(np.int32)
    eps = float(np.float32(eps_f * gen.mean_sq_cost(x, y)))
    tol, max_iter = (1e-12, cap) if cap else (1e-4, 10000)
    w, z = x[ix], y[iy]
    ref = None if cap else O.sinkhorn(w, z, eps, tol=tol)
    for gs in (1, 0):
        ctx.set_tuning("grid_solver", gs)
        try:
            pot, side, inner = sk.sinkhorn_init_subsample(ctx, _cuda(x), _cuda(y), _cuda(ix), _cuda(iy), eps, tol,
                                                         inner_max_iter=max_iter)
        finally:
            ctx.set_tuning("grid_solver", 1)
        assert side == 0, (gs, side)
        if cap:
            assert inner["iterations"] == cap and not inner["converged"], (gs, inner)
        else:
            assert inner["converged"], (gs, inner)
            assert abs(inner["iterations"] - ref.iterations) <= count_tol(ref.iterations), (gs, inner, ref.iterations)
        lock = O.sinkhorn(w, z, eps, tol=0, max_iter=inner["iterations"])
        assert_obj_close(inner["dual_objective"], lock.E, eps, what=f"grid_solver={gs}")
        # the reported err_L is formed from fp32 potentials at the scale of |q|^2: ~4 ulp(max |q|^2) /
        # eps of noise per term (as test_gpu_adaptive)
        scale = max(float((w.astype(np.float64) ** 2).sum(-1).max()), float((z.astype(np.float64) ** 2).sum(-1).max()))
        slack = 4 * 2.0 ** -24 * scale / eps
        assert abs(inner["marginal_error"] - lock.err) <= 0.02 * lock.err + slack + 1e-7, (gs, inner, lock.err, slack)
        ex = O.subsample_extrapolate(x, z, lock.g, eps)
        assert rel_inf(centred(pot.cpu().numpy()), centred(ex), eps) <= INIT_RTOL, gs
    # a capped inner solve: max_iter sweeps, not converged
    _, _, capped = sk.sinkhorn_init_subsample(ctx, _cuda(x), _cuda(y), _cuda(ix), _cuda(iy), eps, 1e-12,
                                             inner_max_iter=5)
    assert capped["iterations"] == 5 and not capped["converged"]
    lock5 = O.sinkhorn(w, z, eps, tol=0, max_iter=5)
    assert_obj_close(capped["dual_objective"], lock5.E, eps, what="capped")


def test_initializer_argument_errors(ctx):
    import paper_2206_07630_b200 as sk
    x = _cuda(np.random.default_rng(0).random((10, 2)).astype(np.float32))
    y = _cuda(np.random.default_rng(1).random((12, 2)).astype(np.float32))
    # sort1d needs n == m (general NW + Alg. 3 is a later row) -> SK_EUNSUPPORTED
    with pytest.raises(sk.SinkhornError) as e:
        sk.sinkhorn_init_sort1d(ctx, x[:, :1].contiguous().view(1, 10), y[:, 0].contiguous(), y_shared=True)
    assert e.value.status == 6
    # subsample: repeated / out-of-range indices -> SK_EINVAL
    ix = _cuda(np.array([0, 1, 1], np.int32))
    iy = _cuda(np.array([0, 2, 3], np.int32))
    with pytest.raises(sk.SinkhornError) as e:
        sk.sinkhorn_init_subsample(ctx, x, y, ix, iy, 0.1, 1e-3)
    assert e.value.status == 1
    with pytest.raises(sk.SinkhornError):
        sk.sinkhorn_init_subsample(ctx, x, y, _cuda(np.array([0, 10], np.int32)), iy, 0.1, 1e-3)
    # GMM: a non-SPD covariance -> SK_EINVAL; zero mixture weight -> SK_EINVAL
    g_bad = {"weights": _cuda(np.ones(1, np.float32)), "means": _cuda(np.zeros((1, 2), np.float32)),
             "covs": _cuda(np.array([[[1.0, 2.0], [2.0, 1.0]]], np.float32))}
    g_ok = {"weights": _cuda(np.ones(1, np.float32)), "means": _cuda(np.zeros((1, 2), np.float32)),
            "covs": _cuda(np.eye(2, dtype=np.float32)[None])}
    with pytest.raises(sk.SinkhornError):
        sk.sinkhorn_init_gmm(ctx, x, y, g_bad, g_ok, 0.5)
    g_zero = dict(g_ok, weights=_cuda(np.zeros(1, np.float32)))
    with pytest.raises(sk.SinkhornError) as e:
        sk.sinkhorn_init_gmm(ctx, x, y, g_zero, g_ok, 0.5)
    assert e.value.status == 1
    # Gaussian: NaN input -> SK_EINVAL
    xn = x.clone()
    xn[3, 0] = float("nan")
    with pytest.raises(sk.SinkhornError) as e:
        sk.sinkhorn_init_gaussian(ctx, xn, y)
    assert e.value.status == 1


def test_gaussian_side_swap_matches_oracle(O, ctx):
    """n > m: the potential lives on y and equals the oracle's swapped evaluation."""
    import paper_2206_07630_b200 as sk
    rng = np.random.default_rng(9)
    x = rng.standard_normal((900, 3)).astype(np.float32)
    y = (rng.standard_normal((400, 3)) * 1.3 + 0.2).astype(np.float32)
    pot, side = sk.sinkhorn_init_gaussian(ctx, _cuda(x), _cuda(y))
    ref, so = O.init_gaussian(x, y)
    assert side == so == 1 and pot.numel() == 400
    assert rel_inf(centred(pot.cpu().numpy()), centred(ref), 0.01) <= INIT_RTOL
