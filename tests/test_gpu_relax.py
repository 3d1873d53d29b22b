"""Alg. 1 with relaxation omega != 1 (reading R-1; P:73 / P:230
"fixed momentum"), CUDA vs the oracle through the C ABI (-m gpu): the same protocol as
test_gpu_solve (stop-rule counts, lockstep potentials and E, an fp64 property check of the
marginal error) on every solver path: on-chip batched (K13), online FFMA (K2), tensor-core
(K3) and stored (K4/K5, where omega != 1 takes the separate row/column passes)."""
import numpy as np
import pytest
import torch

from parity import assert_obj_close, assert_pair_close, count_tol, plan_marginal_error
from workloads import gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2206_07630_b200 as sk
    return sk.Context(0)


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def check_relaxed(O, sk, ctx, x, y, eps, omega, f0=None, a=None, mode="auto", tol=1e-3, what="", decay=None):
    f, g, rep = sk.sinkhorn_solve(ctx, _cuda(x), _cuda(y), eps, tol=tol, mode=mode, omega=omega,
                                  a=None if a is None else _cuda(a), eps_decay=decay,
                                  f_init=None if f0 is None else _cuda(np.asarray(f0, np.float32)))
    f, g = f.cpu().numpy(), g.cpu().numpy()
    L = rep["iterations"]
    ref = O.sinkhorn(x, y, eps, a=a, tol=tol, omega=omega, f0=f0, eps_decay=decay)
    assert abs(L - ref.iterations) <= count_tol(ref.iterations), (what, L, ref.iterations)
    lock = O.sinkhorn(x, y, eps, a=a, tol=0, max_iter=L, omega=omega, f0=f0, eps_decay=decay)
    assert_pair_close(f, g, lock.f, lock.g, eps, what=what)
    assert_obj_close(rep["dual_objective"], lock.E, eps, what=what)
    assert rep["converged"] and rep["marginal_error"] < tol
    # the error includes the row term: recomputed in fp64 from the returned pair
    assert plan_marginal_error(x, y, f, g, eps, a) <= 1.05 * tol + 2e-5, what
    return rep


@pytest.mark.parametrize("omega", [1.05, 1.5, 0.8])
def test_relaxed_onchip_c1(O, ctx, omega):
    import paper_2206_07630_b200 as sk
    p = gen.c1()
    rep = check_relaxed(O, sk, ctx, p.x, p.y, p.eps, omega, what=f"c1 omega={omega}")
    if omega == 1.5:   # the over-relaxed iteration is the faster one on C1 (oracle: 50 vs 165)
        _, _, r1 = sk.sinkhorn_solve(ctx, _cuda(p.x), _cuda(p.y), p.eps)
        assert rep["iterations"] < r1["iterations"]


def test_relaxed_onchip_gaussian_init(O, ctx):
    import paper_2206_07630_b200 as sk
    p = gen.c1(seed=1)
    pot, _ = sk.sinkhorn_init_gaussian(ctx, _cuda(p.x), _cuda(p.y))
    check_relaxed(O, sk, ctx, p.x, p.y, p.eps, 1.4, f0=pot.cpu().numpy(), what="c1 gaussian omega=1.4")


@pytest.mark.parametrize("mode,n,m,d,omega", [("online", 3000, 2600, 3, 1.5), ("online", 1500, 1300, 40, 1.3),
                                              ("stored", 2000, 1024, 16, 1.6), ("online", 2100, 1800, 8, 0.9)])
def test_relaxed_multikernel(O, ctx, mode, n, m, d, omega):
    import paper_2206_07630_b200 as sk
    rng = np.random.default_rng(n + d)
    x = rng.random((n, d)).astype(np.float32)
    y = (rng.random((m, d)) * 0.9 + 0.05).astype(np.float32)
    a = gen.random_weights(n, rng)
    eps = float(np.float32(0.03 * gen.mean_sq_cost(x, y)))
    check_relaxed(O, sk, ctx, x, y, eps, omega, a=a, mode=mode, what=f"{mode} {n}x{m}x{d} omega={omega}")


def test_relaxed_batched_sort1d(O, ctx):
    """A C2-shaped batch (8 problems of 256) with the sorted closed-form init and omega = 1.5."""
    import paper_2206_07630_b200 as sk
    c2 = gen.c2(B=8, n=256)
    xb, yb = _cuda(c2.x), _cuda(c2.y)
    pot = sk.sinkhorn_init_sort1d(ctx, xb.view(8, 256), yb.view(-1))
    f, g, reps = sk.sinkhorn_solve(ctx, xb, yb, c2.eps, y_shared=True, f_init=pot, omega=1.5)
    for k in (0, 5):
        L = reps[k]["iterations"]
        f0 = pot[k].cpu().numpy()
        ref = O.sinkhorn(c2.x[k], c2.y, c2.eps, f0=f0, omega=1.5)
        assert abs(L - ref.iterations) <= count_tol(ref.iterations)
        lock = O.sinkhorn(c2.x[k], c2.y, c2.eps, tol=0, max_iter=L, f0=f0, omega=1.5)
        assert_pair_close(f[k].cpu().numpy(), g[k].cpu().numpy(), lock.f, lock.g, c2.eps)
        assert_obj_close(reps[k]["dual_objective"], lock.E, c2.eps)


def test_relaxation_argument_errors(ctx):
    import ctypes
    import paper_2206_07630_b200 as sk
    for bad in (0.0, -1.0, 2.0, float("nan")):
        assert ctx.lib.sk_set_relaxation(ctx.h, ctypes.c_float(bad)) == 1   # SK_EINVAL


@pytest.mark.parametrize("world,mode,d,omega", [(2, "online", 3, 1.5), (4, "online", 40, 1.3), (8, "stored", 16, 1.4),
                                              (2, "online", 8, 0.8)])
def test_relaxed_sharded_emulated(O, ctx, world, mode, d, omega):
    """omega != 1 with rows sharded over `world` emulated ranks: the row terms of err_l and of
    sum P (E) are summed over the shards (over ranks: one 2-double allreduce per sweep)."""
    import paper_2206_07630_b200 as sk
    rng = np.random.default_rng(60 + world + d)
    n, m = 6000, 1600
    x = rng.random((n, d)).astype(np.float32)
    y = rng.random((m, d)).astype(np.float32)
    a = gen.random_weights(n, rng)
    eps = float(np.float32(0.04 * gen.mean_sq_cost(x, y)))
    f, g, rep = sk.sinkhorn_solve_sharded_emulated(ctx, world, _cuda(x), _cuda(y), eps, a=_cuda(a), mode=mode,
                                                   omega=omega)
    L = rep["iterations"]
    ref = O.sinkhorn(x, y, eps, a=a, omega=omega)
    assert abs(L - ref.iterations) <= count_tol(ref.iterations), (L, ref.iterations)
    lock = O.sinkhorn(x, y, eps, a=a, tol=0, max_iter=L, omega=omega)
    assert_pair_close(f.cpu().numpy(), g.cpu().numpy(), lock.f, lock.g, eps, what=f"relaxed x{world} {mode}")
    assert_obj_close(rep["dual_objective"], lock.E, eps)
    assert rep["converged"] and plan_marginal_error(x, y, f.cpu().numpy(), g.cpu().numpy(), eps, a) <= 1.05e-3 + 2e-5


# ------------------------------------------------------------- eps-decay (NEXT-1, R-25)
@pytest.mark.parametrize("omega", [1.0, 1.5])
def test_eps_decay_onchip_c1(O, ctx, omega):
    import paper_2206_07630_b200 as sk
    p = gen.c1()
    check_relaxed(O, sk, ctx, p.x, p.y, p.eps, omega, decay=(5.0, 0.8), what=f"c1 decay omega={omega}")


@pytest.mark.parametrize("mode,n,m,d", [("online", 3000, 2600, 3), ("online", 1500, 1300, 40), ("stored", 2000, 1024, 16)])
def test_eps_decay_multikernel(O, ctx, mode, n, m, d):
    import paper_2206_07630_b200 as sk
    rng = np.random.default_rng(n + 2 * d)
    x = rng.random((n, d)).astype(np.float32)
    y = (rng.random((m, d)) * 0.9 + 0.05).astype(np.float32)
    eps = float(np.float32(0.03 * gen.mean_sq_cost(x, y)))
    check_relaxed(O, sk, ctx, x, y, eps, 1.0, mode=mode, decay=(5.0, 0.8), what=f"{mode} decay {n}x{m}x{d}")


def test_eps_decay_batched_and_errors(O, ctx):
    import ctypes
    import paper_2206_07630_b200 as sk
    c2 = gen.c2(B=4, n=1024)   # (the C2 shape: ~30 sweeps; long trajectories of this 1D problem at
    xb, yb = _cuda(c2.x), _cuda(c2.y)   # eps = 1e-3 drift past 1e-4 in fp32 with or without decay)
    pot = sk.sinkhorn_init_sort1d(ctx, xb.view(4, 1024), yb.view(-1))
    f, g, reps = sk.sinkhorn_solve(ctx, xb, yb, c2.eps, y_shared=True, f_init=pot, eps_decay=(5.0, 0.8))
    k = 2
    f0 = pot[k].cpu().numpy()
    ref = O.sinkhorn(c2.x[k], c2.y, c2.eps, f0=f0, eps_decay=(5.0, 0.8))
    assert abs(reps[k]["iterations"] - ref.iterations) <= count_tol(ref.iterations)
    lock = O.sinkhorn(c2.x[k], c2.y, c2.eps, tol=0, max_iter=reps[k]["iterations"], f0=f0, eps_decay=(5.0, 0.8))
    assert_pair_close(f[k].cpu().numpy(), g[k].cpu().numpy(), lock.f, lock.g, c2.eps)
    assert ctx.lib.sk_set_eps_decay(ctx.h, ctypes.c_float(5.0), ctypes.c_float(1.5)) == 1   # SK_EINVAL
    x = _cuda(np.random.default_rng(1).random((3000, 3)).astype(np.float32))
    with pytest.raises(sk.SinkhornError):   # multi-kernel: decay with omega != 1 is unsupported
        sk.sinkhorn_solve(ctx, x, x, 0.01, mode="online", omega=1.3, eps_decay=(5.0, 0.8))


def test_eps_decay_max_iter_inside_the_decay(ctx):
    """max_iter <= T: the on-chip solver stops at max_iter (no sweep is checked) instead of looping."""
    import paper_2206_07630_b200 as sk
    p = gen.c1()
    f, g, rep = sk.sinkhorn_solve(ctx, _cuda(p.x), _cuda(p.y), p.eps, max_iter=3, eps_decay=(5.0, 0.8))
    assert rep["iterations"] == 3 and not rep["converged"]


@pytest.mark.parametrize("world,mode,d", [(2, "online", 3), (4, "stored", 16)])
def test_eps_decay_sharded_emulated(O, ctx, world, mode, d):
    """eps-decay (R-25) with rows sharded over emulated ranks: the decay sweeps are chained
    one-sweep solves through each shard's f, as on the unsharded multi-kernel path."""
    import paper_2206_07630_b200 as sk
    rng = np.random.default_rng(70 + world + d)
    n, m = 6000, 1600
    x = rng.random((n, d)).astype(np.float32)
    y = rng.random((m, d)).astype(np.float32)
    eps = float(np.float32(0.03 * gen.mean_sq_cost(x, y)))
    f, g, rep = sk.sinkhorn_solve_sharded_emulated(ctx, world, _cuda(x), _cuda(y), eps, mode=mode,
                                                   eps_decay=(5.0, 0.8))
    L = rep["iterations"]
    ref = O.sinkhorn(x, y, eps, eps_decay=(5.0, 0.8))
    assert abs(L - ref.iterations) <= count_tol(ref.iterations), (L, ref.iterations)
    lock = O.sinkhorn(x, y, eps, tol=0, max_iter=L, eps_decay=(5.0, 0.8))
    assert_pair_close(f.cpu().numpy(), g.cpu().numpy(), lock.f, lock.g, eps, what=f"decay x{world} {mode}")
    assert_obj_close(rep["dual_objective"], lock.E, eps)
