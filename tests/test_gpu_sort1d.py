"""1D path parity (BJ.cfg2 and ragged variants), -m gpu: bit-exact sort/rank, the DualSort
initializer (closed-form fixed point and paper mode) and the batched on-chip solve."""
import numpy as np
import pytest
import torch

from parity import (assert_obj_close, assert_pair_close, centred, count_tol, rel_inf, INIT_RTOL)
from workloads import gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2206_07630_b200 as sk
    return sk.Context(0)


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("B,n", [(1024, 1024), (3, 1), (5, 1000), (2, 4097), (1, 8192), (2, 8193), (3, 20000),
                                 (1, 100000)])
def test_sort_rank_bit_exact(O, ctx, B, n):
    import paper_2206_07630_b200 as sk
    rng = np.random.default_rng(B + n)
    x = rng.random((B, n), dtype=np.float32)
    x[:, ::7] = np.round(x[:, ::7] * 16) / 16      # ties
    if n > 2:
        x[0, 1], x[0, 2] = -0.0, 0.0                  # -0.0 == +0.0 -> index order
    perm, rank = sk.sinkhorn_sort1d_batched(ctx, _cuda(x))
    po, ro = O.sort_rank(x)
    assert np.array_equal(perm.cpu().numpy(), po) and np.array_equal(rank.cpu().numpy(), ro)


def test_sort_rejects_nan(ctx):
    import paper_2206_07630_b200 as sk
    x = np.zeros((2, 5), np.float32)
    x[1, 3] = np.nan
    with pytest.raises(sk.SinkhornError):
        sk.sinkhorn_sort1d_batched(ctx, _cuda(x))


@pytest.fixture(scope="module")
def c2():
    return gen.c2()


def test_c2_init_closed_form_full_batch(O, ctx, c2):
    """Closed-form O(n) dual == the oracle's Alg. 2 Jacobi fixed point, on sampled problems of
    the full launch (B=1024, n=1024); ranks bit-exact on all problems."""
    import paper_2206_07630_b200 as sk
    x = c2.x.reshape(c2.batch, c2.n)
    y = c2.y.reshape(-1)
    pot, perm, rank = sk.sinkhorn_init_sort1d(ctx, _cuda(x), _cuda(y), y_shared=True, want_perm=True)
    po, ro = O.sort_rank(x)
    assert np.array_equal(perm.cpu().numpy(), po) and np.array_equal(rank.cpu().numpy(), ro)
    pot = pot.cpu().numpy()
    for b in (0, 511, 1023):
        f0 = O.init_sort1d(x[b], y)
        assert rel_inf(centred(pot[b]), centred(f0), c2.eps) <= INIT_RTOL, b
        # and uncentred: the fixed point itself (f <= 0, max = 0) is reproduced
        assert np.abs(pot[b] - f0).max() <= 1e-6


@pytest.mark.parametrize("L", [1, 3])
def test_sort1d_paper_mode(O, ctx, L):
    import paper_2206_07630_b200 as sk
    rng = np.random.default_rng(L)
    x = rng.random((4, 300), dtype=np.float32)
    y = (np.arange(300) / 299).astype(np.float32)
    pot = sk.sinkhorn_init_sort1d(ctx, _cuda(x), _cuda(y), y_shared=True, dualsort_iters=L).cpu().numpy()
    for b in range(4):
        f0 = O.init_sort1d(x[b], y, sweeps=L)
        assert np.abs(pot[b] - f0).max() <= 1e-6


@pytest.mark.parametrize("B,n,shared", [(1, 5000, False), (1, 8300, True)])
def test_sort1d_large_n_vs_oracle(O, ctx, B, n, shared):
    """n > 4096: the closed-form scans in workspace (and, n > 8192, the global bitonic sort)
    against the oracle's Alg. 2 Jacobi fixed point."""
    import paper_2206_07630_b200 as sk
    rng = np.random.default_rng(n)
    x = rng.random((B, n), dtype=np.float32)
    y = (np.arange(n) / (n - 1)).astype(np.float32) if shared else rng.random((B, n), dtype=np.float32)
    pot = sk.sinkhorn_init_sort1d(ctx, _cuda(x), _cuda(y), y_shared=shared).cpu().numpy()
    for b in range(B):
        f0 = O.init_sort1d(x[b], y if shared else y[b])
        assert np.abs(pot[b] - f0).max() <= 1e-6, b


def test_sort1d_fixed_point_at_scale(O, ctx):
    """n = 200000 (one problem): the returned dual is the fixed point of Alg. 2 on the sorted
    supports — f_i = min_j (c_ij - c_jj + f_j) — checked on 512 sampled rows over all j in fp64,
    with f <= 0 and max f = 0 (the fixed point from f = 0)."""
    import paper_2206_07630_b200 as sk
    n = 200000
    rng = np.random.default_rng(5)
    x = rng.random((1, n), dtype=np.float32)
    y = rng.standard_normal(n).astype(np.float32)
    pot, perm, _ = sk.sinkhorn_init_sort1d(ctx, _cuda(x), _cuda(y), y_shared=True, want_perm=True)
    pot, perm = pot.cpu().numpy()[0].astype(np.float64), perm.cpu().numpy()[0]
    assert np.array_equal(perm, O.sort_rank(x)[0][0])
    xs = x[0][perm].astype(np.float64)
    ys = np.sort(y).astype(np.float64)
    fs = pot[perm]
    cjj = (xs - ys) ** 2
    scale = max(1.0, np.abs(fs).max())
    assert fs.max() <= 1e-6 * scale and abs(fs.max()) <= 1e-6 * scale
    for i in np.sort(rng.choice(n, 512, replace=False)):
        best = np.min((xs[i] - ys) ** 2 - cjj + fs)
        assert abs(best - fs[i]) <= 1e-5 * scale, (i, best, fs[i])


def test_sort1d_unshared_targets(O, ctx):
    import paper_2206_07630_b200 as sk
    rng = np.random.default_rng(11)
    x = rng.random((3, 129), dtype=np.float32)
    y = rng.random((3, 129), dtype=np.float32)
    pot = sk.sinkhorn_init_sort1d(ctx, _cuda(x), _cuda(y), y_shared=False).cpu().numpy()
    for b in range(3):
        assert np.abs(pot[b] - O.init_sort1d(x[b], y[b])).max() <= 1e-6


@pytest.mark.parametrize("init", ["sort1d", "zero"])
def test_c2_batched_solve_full_launch(O, ctx, c2, init):
    """The bench's launch configuration (B=1024 on-chip solver); sampled problems vs the oracle."""
    import paper_2206_07630_b200 as sk
    x = c2.x.reshape(c2.batch, c2.n)
    y = c2.y.reshape(-1)
    xs, ys = _cuda(c2.x), _cuda(c2.y)
    f0 = sk.sinkhorn_init_sort1d(ctx, _cuda(x), _cuda(y), y_shared=True) if init == "sort1d" else None
    f, g, reps = sk.sinkhorn_solve(ctx, xs, ys, c2.eps, tol=c2.tol, y_shared=True, f_init=f0)
    f, g = f.cpu().numpy(), g.cpu().numpy()
    f0n = None if f0 is None else f0.cpu().numpy()
    assert all(r["converged"] for r in reps)
    samples = (0, 777) if init == "sort1d" else (5,)
    for b in samples:
        fi = None if f0n is None else f0n[b]
        L = reps[b]["iterations"]
        ref = O.sinkhorn(c2.x[b], c2.y, c2.eps, tol=c2.tol, f0=fi)
        assert abs(L - ref.iterations) <= count_tol(ref.iterations), (b, L, ref.iterations)
        lock = O.sinkhorn(c2.x[b], c2.y, c2.eps, tol=0, max_iter=L, f0=fi)
        assert_pair_close(f[b], g[b], lock.f, lock.g, c2.eps, what=f"c2[{b}]")
        assert_obj_close(reps[b]["dual_objective"], lock.E, c2.eps, what=f"c2[{b}]")
    if init == "sort1d":
        its = np.array([r["iterations"] for r in reps])
        assert its.max() < 200, its.max()   # the eps=0 dual start is close (Sec. 3.1)


@pytest.mark.parametrize("kw", [{}, {"omega": 1.3}, {"adaptive": 10}])
def test_c2_park_resume_scheduler_is_bit_identical(kw):
    """K13's park / resume scheduler (sk_set_tuning batched_park: a problem runs at most k sweeps
    per turn, parks its state and re-queues by predicted remaining sweeps) changes only which CTA
    runs which sweeps: the full C2 batch's potentials, counts, errors and objectives are
    bit-identical to one turn per problem (batched_park = 0), for plain, relaxed and adaptive."""
    import paper_2206_07630_b200 as sk
    p = gen.c2()
    outs = []
    for park in (8, 3, 0):
        c = sk.Context(0)
        c.set_tuning("batched_park", park)
        x, y = torch.from_numpy(p.x).cuda(), torch.from_numpy(p.y).cuda()
        f0 = sk.sinkhorn_init_sort1d(c, x.view(1024, 1024), y.view(1024), y_shared=True)
        f, g, reps = sk.sinkhorn_solve(c, x, y, p.eps, y_shared=True, f_init=f0, **kw)
        outs.append((f.cpu(), g.cpu(), [(r["iterations"], r["marginal_error"], r["dual_objective"]) for r in reps]))
        c.close()
    for f, g, r in outs[:2]:
        assert torch.equal(f, outs[2][0]) and torch.equal(g, outs[2][1]) and r == outs[2][2]
    assert max(it for it, _, _ in outs[2][2]) > 8   # problems did park
