"""General 1D initializer (K18: NW corner + Alg. 3/4 in reading R-26) through the
C ABI (-m gpu): f0 vs the oracle (which is pinned to the LP optimum and to DualSort), batches,
non-shared targets, and its use in a solve."""
import numpy as np
import pytest
import torch

from parity import assert_obj_close, assert_pair_close, centred, count_tol, rel_inf
from workloads import gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2206_07630_b200 as sk
    return sk.Context(0)


def _c(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


@pytest.mark.parametrize("n,m,weights", [(300, 200, False), (256, 384, True), (1000, 1024, False),
                                         (512, 512, True), (64, 64, False), (1, 7, True), (9, 1, False)])
def test_nw1d_parity(O, ctx, n, m, weights):
    import paper_2206_07630_b200 as sk
    rng = np.random.default_rng(n + 7 * m)
    B = 3
    x = rng.random((B, n)).astype(np.float32)
    y = np.sort(rng.random(m)).astype(np.float32)
    a = np.stack([gen.random_weights(n, rng) for _ in range(B)]) if weights else None
    b = gen.random_weights(m, rng) if weights else None
    f0, rounds = sk.sinkhorn_init_nw1d(ctx, _c(x), _c(y), a=None if a is None else _c(a),
                                       b=None if b is None else _c(b), y_shared=True)
    for k in range(B):
        fo = O.init_nw1d(x[k], y, None if a is None else a[k], b)
        # the eps = 0 dual is unique up to the tree structure's freedom; the fixed point is exact
        # arithmetic in fp64 on both sides: compare to rounding
        assert np.abs(f0[k].cpu().numpy() - fo).max() <= 1e-6 * max(1.0, np.abs(fo).max()), k


@pytest.mark.parametrize("n,m,weights", [(5000, 7000, True), (9000, 3000, True)])
def test_nw1d_beyond_shared_memory(O, ctx, n, m, weights):
    """Problems whose arrays exceed shared memory keep them in a global slot (one CTA each; the
    n = 9000 side also takes the global-memory sort)."""
    import paper_2206_07630_b200 as sk
    rng = np.random.default_rng(n + m)
    B = 2
    x = rng.random((B, n)).astype(np.float32)
    y = np.sort(rng.random(m)).astype(np.float32)
    a = np.stack([gen.random_weights(n, rng) for _ in range(B)]) if weights else None
    b = gen.random_weights(m, rng) if weights else None
    f0, rounds = sk.sinkhorn_init_nw1d(ctx, _c(x), _c(y), a=None if a is None else _c(a),
                                       b=None if b is None else _c(b), y_shared=True)
    for k in range(B):
        fo = O.init_nw1d(x[k], y, None if a is None else a[k], b)
        assert np.abs(f0[k].cpu().numpy() - fo).max() <= 1e-6 * max(1.0, np.abs(fo).max()), k


def test_nw1d_batched_targets_and_solve(O, ctx):
    """Non-shared targets (B x m), then a solve from f0 with n != m: oracle parity, and fewer sweeps
    than the zero start (the point of the initializer)."""
    import paper_2206_07630_b200 as sk
    rng = np.random.default_rng(5)
    B, n, m = 2, 700, 500
    x = rng.random((B, n)).astype(np.float32)
    y = rng.random((B, m)).astype(np.float32)
    f0, _ = sk.sinkhorn_init_nw1d(ctx, _c(x), _c(y), y_shared=False)
    for k in range(B):
        fo = O.init_nw1d(x[k], y[k])
        assert np.abs(f0[k].cpu().numpy() - fo).max() <= 1e-6 * max(1.0, np.abs(fo).max())
    eps = 2e-3
    xk, yk = x[0][:, None].copy(), y[0][:, None].copy()
    f, g, rep = sk.sinkhorn_solve(ctx, _c(xk), _c(yk), eps, f_init=f0[0].contiguous())
    _, _, rep0 = sk.sinkhorn_solve(ctx, _c(xk), _c(yk), eps)
    assert rep["converged"] and rep["iterations"] < rep0["iterations"]
    ref = O.sinkhorn(xk, yk, eps, f0=f0[0].cpu().numpy())
    assert abs(rep["iterations"] - ref.iterations) <= count_tol(ref.iterations)
    lock = O.sinkhorn(xk, yk, eps, tol=0, max_iter=rep["iterations"], f0=f0[0].cpu().numpy())
    assert_pair_close(f.cpu().numpy(), g.cpu().numpy(), lock.f, lock.g, eps)
    assert_obj_close(rep["dual_objective"], lock.E, eps)
