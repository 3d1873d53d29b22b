"""Tensor-core (tcgen05 kind::f16, 3-product hi/lo split) cross term, -m gpu: the raw 128x128 tile product against fp64,
and the d > 16 solve through the tensor-core pass against the oracle and the FFMA kernel."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from parity import assert_obj_close, assert_pair_close, count_tol
from workloads import gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2206_07630_b200 as sk
    return sk.Context(0)


@pytest.mark.parametrize("d,sx,sy", [(64, 1, 1), (48, 1, 1), (33, 1, 1), (32, 1, 1), (20, 1, 1), (16, 1, 1), (3, 1, 1),
                                     (64, 1e4, 1e-3), (40, 3e-6, 7e5), (64, 1e30, 1e-30)])
def test_tc_tile_product_is_fp32_accurate(ctx, d, sx, sy):
    """Any magnitude: the operands are scaled by exact powers of two before the fp16 split."""
    import ctypes
    import paper_2206_07630_b200 as sk
    rng = np.random.default_rng(d)
    x = (rng.standard_normal((128, d)) * sx).astype(np.float32)
    y = (rng.standard_normal((128, d)) * sy).astype(np.float32)
    out = torch.empty((128, 128), dtype=torch.float32, device="cuda")
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    ctx.check(ctx.lib.sk_selftest_tc_dot(ctx.h, d, ctypes.c_void_p(xd.data_ptr()), ctypes.c_void_p(yd.data_ptr()),
                                         ctypes.c_void_p(out.data_ptr())))
    ref = x.astype(np.float64) @ y.astype(np.float64).T
    scale = np.abs(x).astype(np.float64) @ np.abs(y).astype(np.float64).T
    err = np.abs(out.cpu().numpy() - ref) / scale
    # hi/lo fp16 split, 3 products: ~2^-22 relative to sum |x_k y_k| (one fp16 product: ~2^-11)
    assert err.max() < 4e-6, err.max()


@pytest.mark.parametrize("n,m,d,eps_factor", [(1000, 1300, 64, 1e-2), (700, 515, 40, 5e-2), (2048, 2048, 64, 1e-1),
                                               (1024, 1024, 64, 1e-3)])
def test_tc_solve_parity(O, ctx, n, m, d, eps_factor):
    """K3 solves to tol vs the oracle: counts (P1) and lockstep (P2).  eps = 1e-3 x mean(C) is
    the smallest of BJ.cfg5's sweep (the largest fp16 fold scale, ~450 sweeps): from the
    Gaussian initializer as in the bench."""
    import paper_2206_07630_b200 as sk
    p = gen.c5(n=max(n, m), d=d, eps_factor=eps_factor)
    x, y = p.x[:n].copy(), p.y[:m].copy()
    eps = p.eps
    f0 = None
    if eps_factor == 1e-3:
        f0, _ = sk.sinkhorn_init_gaussian(ctx, torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())
        f0 = f0.cpu().numpy()
    f, g, rep = sk.sinkhorn_solve(ctx, torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), eps, mode="online",
                                  f_init=None if f0 is None else torch.from_numpy(f0).cuda())
    ref = O.sinkhorn(x, y, eps, f0=f0)
    assert rep["converged"] and abs(rep["iterations"] - ref.iterations) <= count_tol(ref.iterations)
    lock = O.sinkhorn(x, y, eps, tol=0, max_iter=rep["iterations"], f0=f0)
    assert_pair_close(f.cpu().numpy(), g.cpu().numpy(), lock.f, lock.g, eps)
    assert_obj_close(rep["dual_objective"], lock.E, eps)


def test_tc_matches_ffma_kernel():
    """Same problem through the tcgen05 pass and (sk_set_tuning("tc", 0)) the FFMA pass: same
    iteration count, potentials within fp32 noise of each other."""
    import paper_2206_07630_b200 as sk
    p = gen.c5(n=1536, eps_factor=1e-2)
    outs = []
    for tc in (1, 0):
        ctx = sk.Context(0)
        ctx.set_tuning("tc", tc)
        f, g, r = sk.sinkhorn_solve(ctx, torch.from_numpy(p.x).cuda(), torch.from_numpy(p.y).cuda(), p.eps,
                                    mode="online")
        outs.append((f.cpu().numpy(), r["iterations"]))
        ctx.close()
    (fa, ia), (fb, ib) = outs
    assert abs(ia - ib) <= 1
    fa, fb = fa - fa.mean(), fb - fb.mean()
    assert np.abs(fa - fb).max() <= 1e-4 * max(np.abs(fb).max(), 1e-3)


@pytest.mark.parametrize("d", [48, 3])
def test_seeded_exact_fallback_and_column_redo(O, d):
    """The seeded passes (fixed shift = previous LSE + margin) with a margin of 300 log2 units:
    every partial sum underflows, so k_merge must recompute every row exactly and every seeded
    column pass must be redone exactly (the colfail redo, K3 at d = 48 / K2 at d = 3); the
    result must still match the oracle in lockstep."""
    import paper_2206_07630_b200 as sk
    if d == 48:
        p = gen.c5(n=1100, d=48, eps_factor=2e-2)
        x, y, eps = p.x[:700].copy(), p.y[:1100].copy(), p.eps
    else:
        rng = np.random.default_rng(3)
        x = rng.random((5000, 3)).astype(np.float32)
        y = rng.random((4100, 3)).astype(np.float32)
        eps = float(np.float32(0.03 * gen.mean_sq_cost(x, y)))
    ctx = sk.Context(0)
    ctx.set_tuning("tc_margin" if d == 48 else "lse_margin", 300)
    f, g, r = sk.sinkhorn_solve(ctx, torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), eps, mode="online")
    ctx.close()
    it = r["iterations"]
    assert it > 3   # seeded passes (sweep >= 2) ran
    lock = O.sinkhorn(x, y, eps, tol=0, max_iter=it)
    assert_pair_close(f.cpu().numpy(), g.cpu().numpy(), lock.f, lock.g, eps)
    assert_obj_close(r["dual_objective"], lock.E, eps)
