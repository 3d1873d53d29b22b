"""CUDA-vs-oracle parity of the Sinkhorn solve through the C ABI (-m gpu).

Protocol: (P1) stop-rule parity of iteration counts,
(P2) lockstep parity — the oracle replays exactly L_gpu sweeps from the same f0 —
of centred potentials (1e-4 rel-inf) and the dual objective (1e-5 rel),
(P4) an fp64 property check of the GPU plan's marginal error.
"""
import numpy as np
import pytest
import torch

from parity import (assert_obj_close, assert_pair_close, count_tol, plan_marginal_error)
from workloads import gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2206_07630_b200 as sk
    return sk.Context(0)


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def check_solve(O, sk, ctx, x, y, eps, tol=1e-3, f0=None, a=None, b=None, mode="auto",
                max_iter=10000, check_every=1, what=""):
    f, g, rep = sk.sinkhorn_solve(ctx, _cuda(x), _cuda(y), eps, tol=tol, max_iter=max_iter,
                                  check_every=check_every, a=None if a is None else _cuda(a),
                                  b=None if b is None else _cuda(b), mode=mode,
                                  f_init=None if f0 is None else _cuda(np.asarray(f0, np.float32)))
    f, g = f.cpu().numpy(), g.cpu().numpy()
    L = rep["iterations"]
    ref = O.sinkhorn(x, y, eps, a=a, b=b, tol=tol, max_iter=max_iter, check_every=check_every,
                     f0=None if f0 is None else np.asarray(f0, np.float32))
    assert abs(L - ref.iterations) <= count_tol(ref.iterations), (what, L, ref.iterations)
    lock = O.sinkhorn(x, y, eps, a=a, b=b, tol=0, max_iter=L,
                      f0=None if f0 is None else np.asarray(f0, np.float32))
    assert_pair_close(f, g, lock.f, lock.g, eps, what=what)
    assert_obj_close(rep["dual_objective"], lock.E, eps, what=what)
    if rep["converged"]:
        assert rep["marginal_error"] < tol
        assert plan_marginal_error(x, y, f, g, eps, a, b) <= 1.05 * tol + 2e-5, what
    return rep


# ------------------------------------------------------------------ C1 (BJ.cfg1)
@pytest.mark.parametrize("init", ["zero", "gaussian"])
def test_c1_parity(O, ctx, init):
    import paper_2206_07630_b200 as sk
    p = gen.c1()
    f0 = None
    if init == "gaussian":
        pot, side = sk.sinkhorn_init_gaussian(ctx, _cuda(p.x), _cuda(p.y))
        fo, so = O.init_gaussian(p.x, p.y)
        assert side == so == 0
        pot = pot.cpu().numpy()
        from parity import centred, rel_inf
        assert rel_inf(centred(pot), centred(fo), p.eps) <= 1e-4
        f0 = pot
    rep = check_solve(O, sk, ctx, p.x, p.y, p.eps, f0=f0, what=f"c1-{init}")
    assert rep["converged"]


# ------------------------------------------------------------- on-chip solver edges
@pytest.mark.parametrize("n,m,d", [(1, 1, 1), (1, 7, 2), (13, 1, 3), (37, 53, 2), (300, 211, 4)])
def test_onchip_ragged_and_degenerate(O, ctx, n, m, d):
    import paper_2206_07630_b200 as sk
    rng = np.random.default_rng(n * 1000 + m)
    x = rng.standard_normal((n, d)).astype(np.float32)
    y = (rng.standard_normal((m, d)) + 0.3).astype(np.float32)
    a = gen.random_weights(n, rng)
    b = gen.random_weights(m, rng)
    eps = float(np.float32(0.05 * max(gen.mean_sq_cost(x, y), 1e-3)))
    check_solve(O, sk, ctx, x, y, eps, a=a, b=b, what=f"onchip {n}x{m}x{d}")


def test_single_atom_closed_form(ctx):
    import paper_2206_07630_b200 as sk
    f, g, rep = sk.sinkhorn_solve(ctx, _cuda(np.zeros((1, 1), np.float32)),
                                  _cuda(np.full((1, 1), 2.0, np.float32)), 0.3)
    assert rep["iterations"] == 1 and rep["converged"]
    assert abs(float(f[0] + g[0]) - 4.0) < 1e-5
    assert abs(rep["dual_objective"] - 3.7) < 1e-5


def test_check_every_and_max_iter(O, ctx):
    import paper_2206_07630_b200 as sk
    p = gen.c1(n=64, seed=3)
    for k in (1, 3, 7):
        check_solve(O, sk, ctx, p.x, p.y, p.eps, check_every=k, what=f"k={k}")
    # non-convergence is not an error: converged = 0, L = max_iter
    f, g, rep = sk.sinkhorn_solve(ctx, _cuda(p.x), _cuda(p.y), p.eps, tol=1e-9, max_iter=5)
    assert rep["iterations"] == 5 and not rep["converged"]
    lock = O.sinkhorn(p.x, p.y, p.eps, tol=0, max_iter=5)
    assert_pair_close(f.cpu().numpy(), g.cpu().numpy(), lock.f, lock.g, p.eps)
    assert abs(rep["marginal_error"] - lock.err) <= 1e-4 * max(lock.err, 1e-3)


def test_g_init_transposed(O, ctx):
    import paper_2206_07630_b200 as sk
    rng = np.random.default_rng(5)
    x = rng.standard_normal((40, 2)).astype(np.float32)
    y = rng.standard_normal((30, 2)).astype(np.float32)
    eps = 0.2
    g0 = rng.standard_normal(30).astype(np.float32) * 0.1
    f, g, rep = sk.sinkhorn_solve(ctx, _cuda(x), _cuda(y), eps, g_init=_cuda(g0))
    ref = O.sinkhorn(y, x, eps, tol=0, max_iter=rep["iterations"], f0=g0)   # transposed problem
    assert_pair_close(g.cpu().numpy(), f.cpu().numpy(), ref.f, ref.g, eps)


def test_host_buffers_roundtrip(O, ctx):
    """Host (CPU) arrays go through the C ABI's own staging (the e2e path)."""
    import paper_2206_07630_b200 as sk
    p = gen.c1(n=96, seed=7)
    f, g, rep = sk.sinkhorn_solve(ctx, torch.from_numpy(p.x), torch.from_numpy(p.y), p.eps)
    assert not f.is_cuda
    fd, gd, repd = sk.sinkhorn_solve(ctx, _cuda(p.x), _cuda(p.y), p.eps)
    assert rep["iterations"] == repd["iterations"]
    assert torch.equal(f, fd.cpu()) and torch.equal(g, gd.cpu())


def test_determinism(ctx):
    import paper_2206_07630_b200 as sk
    p = gen.c1()
    r1 = sk.sinkhorn_solve(ctx, _cuda(p.x), _cuda(p.y), p.eps)
    r2 = sk.sinkhorn_solve(ctx, _cuda(p.x), _cuda(p.y), p.eps)
    assert torch.equal(r1[0], r2[0]) and torch.equal(r1[1], r2[1])
    assert r1[2]["iterations"] == r2[2]["iterations"]


def test_invalid_arguments(ctx):
    import paper_2206_07630_b200 as sk
    x = _cuda(np.zeros((4, 2), np.float32))
    y = _cuda(np.ones((5, 2), np.float32))
    for kw in ({"eps": 0.0}, {"eps": float("nan")}, {"eps": 1.0, "tol": 0.0},
               {"eps": 1.0, "max_iter": 0}, {"eps": 1.0, "check_every": 0}):
        with pytest.raises(sk.SinkhornError) as e:
            sk.sinkhorn_solve(ctx, x, y, **kw)
        assert e.value.status == 1
    bad = x.clone()
    bad[1, 1] = float("inf")
    with pytest.raises(sk.SinkhornError):
        sk.sinkhorn_solve(ctx, bad, y, 1.0)
    a0 = _cuda(np.array([0.5, 0.5, 0.0, 0.0], np.float32))   # zero weights rejected
    with pytest.raises(sk.SinkhornError):
        sk.sinkhorn_solve(ctx, x, y, 1.0, a=a0)
    with pytest.raises(sk.SinkhornError):
        sk.sinkhorn_solve(ctx, x, y, 1.0, f_init=_cuda(np.zeros(4, np.float32)),
                          g_init=_cuda(np.zeros(5, np.float32)))


# -------------------------------------------------------- multi-kernel online path
@pytest.mark.parametrize("n,m,d", [(2500, 1999, 3), (1100, 1300, 16), (777, 900, 2), (600, 520, 64)])
def test_online_multikernel_parity(O, ctx, n, m, d):
    import paper_2206_07630_b200 as sk
    rng = np.random.default_rng(n + m + d)
    x = rng.random((n, d)).astype(np.float32)
    y = (rng.random((m, d)) * 0.9 + 0.05).astype(np.float32)
    eps = float(np.float32(0.03 * gen.mean_sq_cost(x, y)))
    check_solve(O, sk, ctx, x, y, eps, mode="online", what=f"online {n}x{m}x{d}")


@pytest.mark.parametrize("n,m,d", [(1536, 1024, 16), (700, 900, 8)])
def test_stored_parity(O, ctx, n, m, d):
    import paper_2206_07630_b200 as sk
    rng = np.random.default_rng(n * 7 + d)
    x = rng.standard_normal((n, d)).astype(np.float32)
    y = (rng.standard_normal((m, d)) + 0.5).astype(np.float32)
    eps = float(np.float32(0.05 * gen.mean_sq_cost(x, y)))
    a = gen.random_weights(n, rng)
    check_solve(O, sk, ctx, x, y, eps, a=a, mode="stored", what=f"stored {n}x{m}x{d}")


@pytest.mark.parametrize("n,m,d,eps_f", [(1003, 16384, 5, 0.1), (257, 12, 3, 0.05), (3000, 4100, 16, 0.02)])
def test_stored_fused_sweep_parity(O, ctx, n, m, d, eps_f):
    """The fused single-read stored sweep (one exponential per entry, scaled column sums) at the
    widest row it supports (m = 16384), a tiny row and a ragged split, against the oracle."""
    import paper_2206_07630_b200 as sk
    rng = np.random.default_rng(n + m)
    x = rng.standard_normal((n, d)).astype(np.float32)
    y = (rng.standard_normal((m, d)) * 0.8 + 0.3).astype(np.float32)
    eps = float(np.float32(eps_f * gen.mean_sq_cost(x, y)))
    check_solve(O, sk, ctx, x, y, eps, mode="stored", what=f"fused {n}x{m}x{d}")


def test_stored_fused_column_fallback(O, ctx):
    """A column of weight 1e-32 drives its scaled column mass below 2^-100 every sweep: the merge
    must detect it and redo the column pass exactly (status colfail path)."""
    import paper_2206_07630_b200 as sk
    rng = np.random.default_rng(5)
    n, m, d = 900, 1024, 8
    x = rng.standard_normal((n, d)).astype(np.float32)
    y = (rng.standard_normal((m, d)) + 0.25).astype(np.float32)
    b = np.full(m, 1.0, np.float64)
    b[0] = 1e-32
    b = (b / b.sum()).astype(np.float32)
    eps = float(np.float32(0.05 * gen.mean_sq_cost(x, y)))
    check_solve(O, sk, ctx, x, y, eps, b=b, mode="stored", what="fused colfail")


def test_onchip_cta_pair_variant_is_bit_identical(O, ctx):
    """sk_set_tuning("batched_cl", 2) (a CTA pair per problem, DSMEM exchange) computes every
    point's LSE with the same arithmetic: the same potentials and counts as one CTA per problem."""
    import paper_2206_07630_b200 as sk
    c2 = gen.c2(B=16, n=1024)
    outs = []
    for cl in (1, 2):
        c = sk.Context(0)
        c.set_tuning("batched_cl", cl)
        xb, yb = torch.from_numpy(c2.x).cuda(), torch.from_numpy(c2.y).cuda()
        pot = sk.sinkhorn_init_sort1d(c, xb.view(16, 1024), yb.view(-1))
        f, g, r = sk.sinkhorn_solve(c, xb, yb, c2.eps, y_shared=True, f_init=pot)
        outs.append((f.cpu().numpy(), g.cpu().numpy(), [q["iterations"] for q in r]))
        c.close()
    assert outs[0][2] == outs[1][2]
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("entry", ["solve", "anderson", "onchip", "onchip_anderson", "sharded2", "sharded2_anderson"])
def test_nonfinite_potentials_are_reported(ctx, entry):
    """Error contract (include/sinkhorn_b200.h): finite inputs whose squared norms
    overflow fp32 make the potentials non-finite in the first sweep -> SK_ENONFINITE (never SK_OK
    with a NaN error), and f, g hold the last finite iterate (here f^(0) = 0, g^(0) = 0)."""
    import paper_2206_07630_b200 as sk
    from paper_2206_07630_b200 import _lib
    rng = np.random.default_rng(21)
    n, m = (256, 256) if entry.startswith("onchip") else (3000, 2500)
    x = torch.from_numpy(rng.uniform(1e19, 2e19, (n, 1)).astype(np.float32)).cuda()
    y = torch.from_numpy(rng.uniform(-2e19, -1e19, (m, 1)).astype(np.float32)).cuda()
    kw = {"anderson": 5} if "anderson" in entry else {}
    with pytest.raises(sk.SinkhornError) as ei:
        if entry.startswith("sharded2"):
            sk.sinkhorn_solve_sharded_emulated(ctx, 2, x, y, 1.0, mode="online", **kw)
        elif entry.startswith("onchip"):
            f = torch.full((2, n), 7.0, device="cuda")
            g = torch.full((2, m), 7.0, device="cuda")
            sk.sinkhorn_solve(ctx, torch.stack([x, x]), torch.stack([y, y]), 1.0, f=f, g=g, **kw)
        else:
            f = torch.full((1, n), 7.0, device="cuda")
            g = torch.full((1, m), 7.0, device="cuda")
            sk.sinkhorn_solve(ctx, x, y, 1.0, mode="online", f=f, g=g, **kw)
    assert ei.value.status == _lib.SK_ENONFINITE, str(ei.value)
    if not entry.startswith("sharded2"):
        assert bool(torch.isfinite(f).all()) and bool(torch.isfinite(g).all())
