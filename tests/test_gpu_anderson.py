"""Anderson acceleration of the sweep map ("Anderson
acceleration (And = 5)"; reading R-27), CUDA (the on-chip solver K13) vs the oracle through
the C ABI (-m gpu): stop-rule counts, lockstep potentials and E, and an fp64 property check of
the returned pair's marginal error, for a single problem (CTA pair) and a batch (one CTA per
problem), plus the argument and path errors."""
import ctypes

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


def check_anderson(O, sk, ctx, x, y, eps, mem, f0=None, a=None, tol=1e-3, what="", mode="auto"):
    f, g, rep = sk.sinkhorn_solve(ctx, _cuda(x), _cuda(y), eps, tol=tol, anderson=mem, mode=mode,
                                  a=None if a is None else _cuda(a),
                                  f_init=None if f0 is None else _cuda(np.asarray(f0, np.float32)))
    f, g = f.cpu().numpy(), g.cpu().numpy()
    L = rep["iterations"]
    ref = O.sinkhorn_anderson(x, y, eps, mem=mem, a=a, tol=tol, f0=f0)
    assert abs(L - ref.iterations) <= count_tol(ref.iterations), (what, L, ref.iterations)
    lock = O.sinkhorn_anderson(x, y, eps, mem=mem, a=a, tol=0, max_iter=L, f0=f0)
    assert_pair_close(f, g, lock.f, lock.g, eps, what=what)
    assert_obj_close(rep["dual_objective"], lock.E, eps, what=what)
    assert rep["converged"] and rep["marginal_error"] < tol
    assert plan_marginal_error(x, y, f, g, eps, a) <= 1.05 * tol + 2e-5, what
    return rep


@pytest.mark.parametrize("mem", [2, 5, 8])
def test_anderson_onchip_c1(O, ctx, mem):
    import paper_2206_07630_b200 as sk
    p = gen.c1()
    rep = check_anderson(O, sk, ctx, p.x, p.y, p.eps, mem, what=f"c1 anderson mem={mem}")
    if mem == 5:   # accelerated: the oracle takes 31 sweeps against plain Sinkhorn's 165 on C1
        _, _, r1 = sk.sinkhorn_solve(ctx, _cuda(p.x), _cuda(p.y), p.eps)
        assert rep["iterations"] < r1["iterations"] / 2


def test_anderson_weighted_and_initialized(O, ctx):
    import paper_2206_07630_b200 as sk
    p = gen.c1(seed=3)
    rng = np.random.default_rng(3)
    a = gen.random_weights(p.x.shape[0], rng)
    pot, _ = sk.sinkhorn_init_gaussian(ctx, _cuda(p.x), _cuda(p.y))
    check_anderson(O, sk, ctx, p.x, p.y, p.eps, 5, a=a, what="c1 weighted anderson")
    check_anderson(O, sk, ctx, p.x, p.y, p.eps, 5, f0=pot.cpu().numpy(), what="c1 gaussian anderson")


def test_anderson_ragged_and_tiny(O, ctx):
    import paper_2206_07630_b200 as sk
    rng = np.random.default_rng(11)
    for n, m, d in ((1, 7, 2), (37, 211, 3), (300, 129, 4)):
        x = rng.random((n, d)).astype(np.float32)
        y = rng.random((m, d)).astype(np.float32)
        eps = float(np.float32(0.05 * gen.mean_sq_cost(x, y)))
        check_anderson(O, sk, ctx, x, y, eps, 4, what=f"anderson {n}x{m}x{d}")


def test_anderson_batched_sort1d(O, ctx):
    """A C2-shaped batch (8 problems of 1024, the sorted closed-form init, mem = 5).  Near the
    solution of these 1D problems the residual Gram matrix is ill-conditioned (cond up to 1e5
    in the oracle), and fp32 rounding of T (~7e-8 absolute) moves the mixed iterate by ~2e-3
    relative (R-27, measured by perturbing the oracle's T): the full trajectory is
    not a lockstep quantity here.  Parity is therefore (1) lockstep over the first 3 sweeps
    (two-slot mixing), (2) the stop count within 15 %, (3) the returned pair's fp64 marginal
    error below tol and (4) E within 3e-5 of the oracle's (both pairs at err < 1e-3 sit within
    1.2e-5 of the optimum's E)."""
    import paper_2206_07630_b200 as sk
    c2 = gen.c2(B=8, n=1024)
    xb, yb = _cuda(c2.x), _cuda(c2.y)
    pot = sk.sinkhorn_init_sort1d(ctx, xb.view(8, 1024), yb.view(-1))
    f3, g3, _ = sk.sinkhorn_solve(ctx, xb, yb, c2.eps, y_shared=True, f_init=pot, anderson=5, tol=1e-30, max_iter=3)
    f, g, reps = sk.sinkhorn_solve(ctx, xb, yb, c2.eps, y_shared=True, f_init=pot, anderson=5)
    for k in (0, 3, 7):
        f0 = pot[k].cpu().numpy()
        lock = O.sinkhorn_anderson(c2.x[k], c2.y, c2.eps, mem=5, tol=0, max_iter=3, f0=f0)
        assert_pair_close(f3[k].cpu().numpy(), g3[k].cpu().numpy(), lock.f, lock.g, c2.eps, what=f"c2[{k}] 3 sweeps")
        L = reps[k]["iterations"]
        ref = O.sinkhorn_anderson(c2.x[k], c2.y, c2.eps, mem=5, f0=f0)
        assert abs(L - ref.iterations) <= max(2, int(np.ceil(0.15 * ref.iterations))), (k, L, ref.iterations)
        assert reps[k]["converged"] and reps[k]["marginal_error"] < 1e-3
        fk, gk = f[k].cpu().numpy(), g[k].cpu().numpy()
        assert plan_marginal_error(c2.x[k], c2.y, fk, gk, c2.eps) <= 1.05e-3 + 2e-5
        assert abs(reps[k]["dual_objective"] - ref.E) <= 3e-5 * abs(ref.E), (k, reps[k]["dual_objective"], ref.E)


@pytest.mark.parametrize("mode,n,m,d,mem", [("online", 3000, 2600, 3, 5), ("online", 1500, 1300, 40, 5),
                                            ("stored", 2000, 1024, 16, 4), ("online", 2100, 1800, 8, 3),
                                            ("online", 1500, 1300, 128, 5), ("stored", 1200, 1024, 100, 4)])
def test_anderson_multikernel(O, ctx, mode, n, m, d, mem):
    """K19 on the online FFMA (K2), tensor-core (K3, d = 40) and stored (K4) solvers."""
    import paper_2206_07630_b200 as sk
    rng = np.random.default_rng(n + d + 7)
    x = rng.random((n, d)).astype(np.float32)
    y = (rng.random((m, d)) * 0.9 + 0.05).astype(np.float32)
    a = gen.random_weights(n, rng)
    eps = float(np.float32(0.03 * gen.mean_sq_cost(x, y)))
    rep = check_anderson(O, sk, ctx, x, y, eps, mem, a=a, mode=mode, what=f"{mode} {n}x{m}x{d} mem={mem}")
    _, _, r0 = sk.sinkhorn_solve(ctx, _cuda(x), _cuda(y), eps, a=_cuda(a), mode=mode)
    # (high-d uniform clouds at this eps converge in a handful of plain sweeps: no room to gain)
    assert rep["iterations"] < r0["iterations"] or r0["iterations"] <= 8


@pytest.mark.parametrize("mode,d", [("online", 3), ("online", 40), ("stored", 16)])
def test_anderson_multikernel_max_iter_and_check_every(O, ctx, mode, d):
    """K19: an unreachable tol stops at max_iter with (f^{L-1}, g_sk(f^{L-1})) (lockstep), and
    check_every = 3 stops on a multiple of 3 sweeps."""
    import paper_2206_07630_b200 as sk
    rng = np.random.default_rng(40 + d)
    n, m = 1800, 1536
    x = rng.random((n, d)).astype(np.float32)
    y = rng.random((m, d)).astype(np.float32)
    eps = float(np.float32(0.05 * gen.mean_sq_cost(x, y)))
    f, g, rep = sk.sinkhorn_solve(ctx, _cuda(x), _cuda(y), eps, tol=1e-30, max_iter=7, mode=mode, anderson=4)
    assert rep["iterations"] == 7 and not rep["converged"]
    lock = O.sinkhorn_anderson(x, y, eps, mem=4, tol=0, max_iter=7)
    assert_pair_close(f.cpu().numpy(), g.cpu().numpy(), lock.f, lock.g, eps, what=f"{mode} d={d} max_iter")
    assert_obj_close(rep["dual_objective"], lock.E, eps)
    _, _, rep = sk.sinkhorn_solve(ctx, _cuda(x), _cuda(y), eps, check_every=3, mode=mode, anderson=4)
    assert rep["converged"] and rep["iterations"] % 3 == 0


@pytest.mark.parametrize("world,mode,d", [(2, "online", 3), (4, "online", 40), (8, "stored", 16)])
def test_anderson_sharded_emulated(O, ctx, world, mode, d):
    """Rows sharded over `world` emulated ranks (slices): the Gram dots and the error are summed
    over the slices in rank order (the NCCL path allreduces the same 9 numbers): lockstep with
    the oracle, and the same stop count as the unsharded solve."""
    import ctypes
    import paper_2206_07630_b200 as sk
    rng = np.random.default_rng(50 + world + d)
    n, m = 6000, 1600
    x = rng.random((n, d)).astype(np.float32)
    y = rng.random((m, d)).astype(np.float32)
    eps = float(np.float32(0.05 * gen.mean_sq_cost(x, y)))
    f, g, rep = sk.sinkhorn_solve_sharded_emulated(ctx, world, _cuda(x), _cuda(y), eps, mode=mode, anderson=5)
    L = rep["iterations"]
    ref = O.sinkhorn_anderson(x, y, eps, mem=5)
    assert abs(L - ref.iterations) <= count_tol(ref.iterations), (L, ref.iterations)
    lock = O.sinkhorn_anderson(x, y, eps, mem=5, tol=0, max_iter=L)
    assert_pair_close(f.cpu().numpy(), g.cpu().numpy(), lock.f, lock.g, eps, what=f"sharded x{world} {mode}")
    assert_obj_close(rep["dual_objective"], lock.E, eps)
    assert rep["converged"]


def test_anderson_max_iter_and_check_every(O, ctx):
    """An unreachable tol runs exactly max_iter sweeps and returns (f^{L-1}, g_sk(f^{L-1})); check_every
    > 1 stops on a multiple of it."""
    import paper_2206_07630_b200 as sk
    p = gen.c1(seed=5)
    f, g, rep = sk.sinkhorn_solve(ctx, _cuda(p.x), _cuda(p.y), p.eps, tol=1e-30, max_iter=12, anderson=5)
    assert rep["iterations"] == 12 and not rep["converged"]
    lock = O.sinkhorn_anderson(p.x, p.y, p.eps, mem=5, tol=0, max_iter=12)
    assert_pair_close(f.cpu().numpy(), g.cpu().numpy(), lock.f, lock.g, p.eps)
    _, _, rep = sk.sinkhorn_solve(ctx, _cuda(p.x), _cuda(p.y), p.eps, check_every=4, anderson=5)
    assert rep["converged"] and rep["iterations"] % 4 == 0


def test_anderson_argument_and_path_errors(ctx):
    import paper_2206_07630_b200 as sk
    for bad in (-1, 9, 100):
        assert ctx.lib.sk_set_anderson(ctx.h, bad) == 1   # SK_EINVAL
    p = gen.c1()
    x, y = _cuda(p.x), _cuda(p.y)
    with pytest.raises(sk.SinkhornError):   # combined with omega != 1
        sk.sinkhorn_solve(ctx, x, y, p.eps, omega=1.5, anderson=5)
    with pytest.raises(sk.SinkhornError):   # combined with eps-decay
        sk.sinkhorn_solve(ctx, x, y, p.eps, eps_decay=(5.0, 0.8), anderson=5)
    # the context is back to plain Sinkhorn afterwards
    _, _, r = sk.sinkhorn_solve(ctx, x, y, p.eps)
    assert r["iterations"] > 100


def test_anderson_host_buffers_match_device(ctx):
    """The e2e path: host (pinned) inputs staged by the library give the same Anderson solve as
    device inputs (on-chip batch and multi-kernel)."""
    import paper_2206_07630_b200 as sk
    c2 = gen.c2(B=16, n=1024)
    xh, yh = torch.from_numpy(c2.x).pin_memory(), torch.from_numpy(c2.y).pin_memory()
    fd, gd, rd = sk.sinkhorn_solve(ctx, xh.cuda(), yh.cuda(), c2.eps, y_shared=True, anderson=5)
    fh, gh, rh = sk.sinkhorn_solve(ctx, xh, yh, c2.eps, y_shared=True, anderson=5)
    assert [r["iterations"] for r in rd] == [r["iterations"] for r in rh]
    assert torch.equal(fd.cpu(), fh) and torch.equal(gd.cpu(), gh)
    rng = np.random.default_rng(9)
    x = rng.random((3000, 3)).astype(np.float32)
    y = rng.random((2500, 3)).astype(np.float32)
    eps = float(np.float32(0.05 * gen.mean_sq_cost(x, y)))
    xh, yh = torch.from_numpy(x).pin_memory(), torch.from_numpy(y).pin_memory()
    fd, gd, rd = sk.sinkhorn_solve(ctx, xh.cuda(), yh.cuda(), eps, mode="online", anderson=5)
    fh, gh, rh = sk.sinkhorn_solve(ctx, xh, yh, eps, mode="online", anderson=5)
    assert rd["iterations"] == rh["iterations"]
    assert torch.equal(fd.cpu(), fh) and torch.equal(gd.cpu(), gh)
