"""Soft ranks / soft sort (Sec. 3.1; K15) through the C ABI (-m gpu).

(1) Kernel parity on the ORACLE's potentials (fp64 solve, cast to fp32 — never a CUDA value
as an oracle input): GPU K15 vs oracle.soft_rank_sort on the same (x, y, f, g).
(2) End to end: GPU sort1d init + solve + K15 vs the oracle replaying the same number of
sweeps from the same initial potential.  (3) Edges: n = 1, ragged sizes, n != m, weights, z,
host buffers, invalid arguments."""
import numpy as np
import pytest
import torch

from parity import centred, rel_inf
from workloads import gen

pytestmark = pytest.mark.gpu
RTOL_KERNEL = 2e-5   # fp32 exponents of magnitude ~kappa |f| (R-22)
RTOL_E2E = 1e-4      # the potentials' own lockstep bar (R-18)


@pytest.fixture(scope="module")
def ctx():
    import paper_2206_07630_b200 as sk
    return sk.Context(0)


def _c(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


@pytest.mark.parametrize("n,m,weights,zgiven", [(512, 512, False, False), (300, 211, True, True),
                                                (1, 1, False, False), (1, 9, True, False), (37, 1024, False, True)])
def test_kernel_parity_on_oracle_potentials(O, ctx, n, m, weights, zgiven):
    """(weights only shape the potentials; the outputs are conditional means under P, R-22)"""
    import paper_2206_07630_b200 as sk
    rng = np.random.default_rng(n * 7 + m)
    B = 3
    x = rng.random((B, n)).astype(np.float32)
    y = np.sort(rng.random(m)).astype(np.float32)
    a = np.stack([gen.random_weights(n, rng) for _ in range(B)]) if weights else None
    b = np.stack([gen.random_weights(m, rng) for _ in range(B)]) if weights else None
    z = (rng.random(m) * 5 - 1).astype(np.float32) if zgiven else None
    eps = 2e-3
    F, G, R, S = [], [], [], []
    for k in range(B):
        r = O.sinkhorn(x[k][:, None], y[:, None], eps, a=None if a is None else a[k],
                       b=None if b is None else b[k], tol=0, max_iter=30)
        f32, g32 = r.f.astype(np.float32), r.g.astype(np.float32)
        rk, st = O.soft_rank_sort(x[k], y, f32, g32, eps, z=z)
        F.append(f32); G.append(g32); R.append(rk); S.append(st)
    rk_g, st_g = sk.sinkhorn_soft_rank_sort(ctx, _c(x), _c(y), eps, _c(np.stack(F)), _c(np.stack(G)),
                                            z=None if z is None else _c(z), y_shared=True)
    for k in range(B):
        assert rel_inf(rk_g[k].cpu().numpy(), R[k], 1.0) <= RTOL_KERNEL, k
        assert rel_inf(st_g[k].cpu().numpy(), S[k], 1e-3) <= RTOL_KERNEL, k


@pytest.mark.parametrize("B,n,m", [(2, 8000, 12000), (1, 30000, 2000)])
def test_large_problems_global_kernel(O, ctx, B, n, m):
    """2n + 3m floats beyond shared memory: the global-memory K15 variant against the oracle's
    fp64 conditional means, on arbitrary finite potentials."""
    import paper_2206_07630_b200 as sk
    rng = np.random.default_rng(n + m)
    eps = 1e-2
    x = rng.random((B, n)).astype(np.float32)
    y = np.sort(rng.random(m)).astype(np.float32)
    f = (rng.standard_normal((B, n)) * eps).astype(np.float32)
    g = (rng.standard_normal((B, m)) * eps).astype(np.float32)
    rk_g, st_g = sk.sinkhorn_soft_rank_sort(ctx, _c(x), _c(y), eps, _c(f), _c(g), y_shared=True)
    for k in range(B):
        rk, st = O.soft_rank_sort(x[k], y, f[k], g[k], eps)
        assert rel_inf(rk_g[k].cpu().numpy(), rk, 1.0) <= RTOL_KERNEL, k
        assert rel_inf(st_g[k].cpu().numpy(), st, 1e-3) <= RTOL_KERNEL, k


def test_end_to_end_c2_batch(O, ctx):
    """A C2-shaped batch (BJ.cfg2 recipe, 16 problems of 1024): sort1d init -> solve -> K15,
    against the oracle replaying L_gpu sweeps from the same f0 (sampled problems)."""
    import paper_2206_07630_b200 as sk
    c2 = gen.c2(B=16, n=1024)
    xb, yb = torch.from_numpy(c2.x).cuda(), torch.from_numpy(c2.y).cuda()
    pot = sk.sinkhorn_init_sort1d(ctx, xb.view(16, 1024), yb.view(-1))
    f, g, reps = sk.sinkhorn_solve(ctx, xb, yb, c2.eps, y_shared=True, f_init=pot)
    rk, st = sk.sinkhorn_soft_rank_sort(ctx, xb.view(16, 1024), yb.view(-1), c2.eps, f, g, y_shared=True)
    for k in (0, 9):
        f0 = pot[k].cpu().numpy()
        lock = O.sinkhorn(c2.x[k], c2.y, c2.eps, tol=0, max_iter=reps[k]["iterations"], f0=f0)
        rko, sto = O.soft_rank_sort(c2.x[k].ravel(), c2.y.ravel(), lock.f, lock.g, c2.eps)
        # the outputs are weighted means under P, whose weights move by exp(dlt/eps) - 1 when the
        # potentials move by dlt (centred, f + g): |d rank| <= 2 dlt/eps (m - 1), |d sort| <= 2 dlt/eps
        fc, gc = centred(f[k].cpu().numpy(), g[k].cpu().numpy())
        foc, goc = centred(lock.f, lock.g)
        dlt = np.abs(fc - foc).max() + np.abs(gc - goc).max()
        assert rel_inf(fc, foc, c2.eps) <= RTOL_E2E and rel_inf(gc, goc, c2.eps) <= RTOL_E2E
        amp = np.expm1(2 * dlt / c2.eps)
        assert np.abs(rk[k].cpu().numpy() - rko).max() <= amp * 1023 + 1e-3
        assert np.abs(st[k].cpu().numpy() - sto).max() <= amp * 1.0 + 1e-5
        # properties of the outputs: exp(2 x y / eps) is totally positive, so the soft rank is
        # non-decreasing in x; and sum_i a_i rank_i = sum_j (column mass)_j z_j ~ (m + 1) / 2
        r_sorted = rk[k].cpu().numpy()[np.argsort(c2.x[k].ravel(), kind="stable")]
        # (up to the fp32 jitter of the weights, ~kappa ulp(f + g))
        assert np.all(np.diff(r_sorted) >= -0.01), np.diff(r_sorted).min()
        assert abs(rk[k].cpu().numpy().mean() - 1025 / 2) <= 1e-3 * 1024


def test_host_buffers_and_errors(O, ctx):
    import paper_2206_07630_b200 as sk
    rng = np.random.default_rng(3)
    x = torch.from_numpy(rng.random(64).astype(np.float32))
    y = torch.from_numpy(np.linspace(0, 1, 64).astype(np.float32))
    r = O.sinkhorn(x.numpy()[:, None], y.numpy()[:, None], 0.01, tol=0, max_iter=20)
    f = torch.from_numpy(r.f.astype(np.float32))
    g = torch.from_numpy(r.g.astype(np.float32))
    rk, st = sk.sinkhorn_soft_rank_sort(ctx, x, y, 0.01, f, g, y_shared=True)   # host arrays
    rko, sto = O.soft_rank_sort(x.numpy(), y.numpy(), f.numpy(), g.numpy(), 0.01)
    assert rel_inf(rk.numpy(), rko, 1.0) <= RTOL_KERNEL and rel_inf(st.numpy(), sto, 1e-3) <= RTOL_KERNEL
    with pytest.raises(sk.SinkhornError):
        sk.sinkhorn_soft_rank_sort(ctx, x.cuda(), y.cuda(), 0.0, f.cuda(), g.cuda(), y_shared=True)
    with pytest.raises(sk.SinkhornError):
        bad = f.clone(); bad[3] = float("nan")
        sk.sinkhorn_soft_rank_sort(ctx, x.cuda(), y.cuda(), 0.01, bad.cuda(), g.cuda(), y_shared=True)


def test_full_c2_batch_sampled(O, ctx):
    """The bench's launch configuration (BJ.cfg2: 1024 problems of 1024, the default step's solve
    then K15 on the whole batch): sampled problems against the oracle's soft rank/sort of the
    oracle's lockstep potentials, with the derived amplification bound of the e2e test."""
    import paper_2206_07630_b200 as sk
    c2 = gen.c2()
    xb, yb = torch.from_numpy(c2.x).cuda(), torch.from_numpy(c2.y).cuda()
    pot = sk.sinkhorn_init_sort1d(ctx, xb.view(1024, 1024), yb.view(-1))
    f, g, reps = sk.sinkhorn_solve(ctx, xb, yb, c2.eps, y_shared=True, f_init=pot)
    rk, st = sk.sinkhorn_soft_rank_sort(ctx, xb.view(1024, 1024), yb.view(-1), c2.eps, f, g, y_shared=True)
    for k in (0, 511, 1023):
        lock = O.sinkhorn(c2.x[k], c2.y, c2.eps, tol=0, max_iter=reps[k]["iterations"], f0=pot[k].cpu().numpy())
        rko, sto = O.soft_rank_sort(c2.x[k].ravel(), c2.y.ravel(), lock.f, lock.g, c2.eps)
        fc, gc = centred(f[k].cpu().numpy(), g[k].cpu().numpy())
        foc, goc = centred(lock.f, lock.g)
        amp = np.expm1(2 * (np.abs(fc - foc).max() + np.abs(gc - goc).max()) / c2.eps)
        assert np.abs(rk[k].cpu().numpy() - rko).max() <= amp * 1023 + 1e-3, k
        assert np.abs(st[k].cpu().numpy() - sto).max() <= amp + 1e-5, k
