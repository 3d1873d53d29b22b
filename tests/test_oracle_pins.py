"""Pins for the fp64 oracle (-m "not gpu"): closed forms, invariants, brute force and
independent library routines — never a retyped copy of the oracle's own formula.

Each test names the passage (PAPER.md line, "P:n") or DESIGN.md reading it checks.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

from workloads import gen

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "analytic_cases.json")))


def rand_cloud(rng, n, d, shift=0.0):
    return (rng.standard_normal((n, d)) + shift).astype(np.float32)


# ------------------------------------------------------------------ cost / soft-min
def test_cost_analytic_and_invariants(O):
    assert O.cost_matrix([[0.0]], [[3.0]])[0, 0] == 9.0
    rng = np.random.default_rng(1)
    x = rand_cloud(rng, 7, 3)
    C = O.cost_matrix(x, x)
    assert np.all(np.diag(C) == 0) and np.array_equal(C, C.T)
    t = np.array([0.5, -2.0, 1.25], np.float32)
    y = rand_cloud(rng, 5, 3)
    assert np.allclose(O.cost_matrix(x + t, y + t), O.cost_matrix(x, y), atol=1e-9)


def test_softmin_closed_form_and_limits(O):
    g = GOLD["softmin_two_zeros"]
    assert abs(O.softmin(g["S"], g["eps"]) - g["value"]) < 1e-15
    rng = np.random.default_rng(2)
    S = rng.uniform(0, 3, 9)
    # eps -> 0 gives the hard minimum (P:49 limit)
    assert abs(O.softmin(S, 1e-9) - S.min()) < 1e-6
    # brute-force exactly-rounded summation (math.fsum) without max shift
    eps = 0.7
    ref = -eps * math.log(math.fsum(math.exp(-s / eps) for s in S))
    assert abs(O.softmin(S, eps) - ref) < 1e-12
    # max shift: no overflow for huge costs
    assert np.isfinite(O.softmin(S + 1e5, 1e-3))


# ------------------------------------------------------------------ Sinkhorn + Eq. (2)
def test_single_atom_forced_coupling(O):
    g = GOLD["single_atom"]
    r = O.sinkhorn(g["x"], g["y"], g["eps"], tol=1e-12, max_iter=5)
    assert r.iterations == 1 and r.converged
    assert abs(r.f[0] + r.g[0] - g["f_plus_g"]) < 1e-12
    assert abs(r.E - g["E"]) < 1e-12


def test_zero_potentials_objective(O):
    E = O.dual_objective([[0.0]], [[0.0]], [0.0], [0.0], 1.0)
    assert E == GOLD["zero_potentials_zero_cost"]["E"]


def test_symmetric_two_point_problem(O):
    # C = [[0,1],[1,0]], eps=1 (SPEC-style symmetry case): marginals (1/2,1/2), f ~ g
    x = y = np.array([[0.0], [1.0]], np.float32)
    r = O.sinkhorn(x, y, 1.0, tol=1e-13, max_iter=1000)
    C = O.cost_matrix(x, y)
    P = np.exp((r.f[:, None] + r.g[None, :] - C) / 1.0)
    assert np.allclose(P.sum(1), 0.5, atol=1e-12) and np.allclose(P.sum(0), 0.5, atol=1e-12)
    fc, gc = r.f - r.f.mean(), r.g - r.g.mean()
    assert np.allclose(fc, gc, atol=1e-12)


def test_dual_ascent_monotone_and_identity(O):
    # Each half-update is an exact block maximisation of Eq. (2): E nondecreasing.
    rng = np.random.default_rng(3)
    x, y = rand_cloud(rng, 16, 2), rand_cloud(rng, 19, 2, 0.5)
    a = rng.uniform(0.5, 1.5, 16); a /= a.sum()
    b = rng.uniform(0.5, 1.5, 19); b /= b.sum()
    r = O.sinkhorn(x, y, 0.1, a=a, b=b, tol=0, max_iter=60, trace=True)
    assert np.all(np.diff(r.trace) >= -1e-12)
    # After an f-update the row sums of P equal a exactly, so E = <f,a> + <g,b> - eps sum(a)
    assert abs(r.E - (r.f @ a + r.g @ b - 0.1 * a.sum())) < 1e-12


def test_shift_invariance_and_weak_strong_duality(O):
    rng = np.random.default_rng(4)
    n, m, eps = 8, 8, 0.1
    x, y = rand_cloud(rng, n, 2), rand_cloud(rng, m, 2, 0.3)
    a, b = np.full(n, 1 / n), np.full(m, 1 / m)
    C = O.cost_matrix(x, y)
    f, g = rng.standard_normal(n), rng.standard_normal(m)
    # shift invariance (BJ.ns)
    E0 = O.dual_objective(x, y, f, g, eps)
    assert abs(O.dual_objective(x, y, f + 0.37, g - 0.37, eps) - E0) < 1e-14 * abs(E0)

    def primal(P):  # Eq. (1) with the + entropy sign (reading R-3)
        return float((P * C).sum() + eps * (P * (np.log(P) - 1)).sum())

    # weak duality: any (f,g) is below the primal value of any feasible P (here a b^T)
    for _ in range(20):
        f, g = rng.standard_normal(n), rng.standard_normal(m)
        assert O.dual_objective(x, y, f, g, eps) <= primal(np.outer(a, b)) + 1e-12
    # strong duality at convergence: E* = primal(P*)
    eps = 1.0
    r = O.sinkhorn(x, y, eps, tol=1e-13, max_iter=100000)
    assert r.converged
    P = np.exp((r.f[:, None] + r.g[None, :] - C) / eps)
    assert abs(r.E - primal(P)) < 1e-9
    # the printed "-eps" sign of Eq. (1) does NOT give strong duality (why R-3 is needed)
    assert abs(r.E - float((P * C).sum() - eps * (P * (np.log(P) - 1)).sum())) > 1e-3


def test_converged_plan_meets_both_marginals_independently(O):
    rng = np.random.default_rng(5)
    x, y = rand_cloud(rng, 30, 3), rand_cloud(rng, 25, 3, 1.0)
    eps = 0.05 * float(O.cost_matrix(x, y).mean())
    r = O.sinkhorn(x, y, eps, tol=1e-3)
    assert r.converged
    C = ((x[:, None, :].astype(np.float64) - y[None, :, :]) ** 2).sum(-1)
    P = np.exp((r.f[:, None] + r.g[None, :] - C) / eps)
    err = np.abs(P.sum(1) - 1 / 30).sum() + np.abs(P.sum(0) - 1 / 25).sum()
    assert err < 1e-3 and abs(err - r.err) < 1e-12


def test_warm_start_from_solution(O):
    rng = np.random.default_rng(6)
    x, y = rand_cloud(rng, 20, 2), rand_cloud(rng, 20, 2, 0.5)
    r = O.sinkhorn(x, y, 0.2, tol=1e-10, max_iter=100000)
    r2 = O.sinkhorn(x, y, 0.2, tol=1e-9, f0=r.f)
    assert r2.iterations == 1


def test_fused_error_identity(O):
    # err_l from the next g-update: sum_j b_j |expm1((g^l - g^{l+1})/eps)| (H5)
    rng = np.random.default_rng(7)
    x, y = rand_cloud(rng, 24, 2), rand_cloud(rng, 17, 2, 0.4)
    eps = 0.3
    r = O.sinkhorn(x, y, eps, tol=0, max_iter=7)
    g_next = O.g_update(x, y, r.f, eps)
    fused = float((np.full(17, 1 / 17) * np.abs(np.expm1((r.g - g_next) / eps))).sum())
    assert abs(fused - r.err) < 1e-13


def test_sampled_updates_match_full(O):
    rng = np.random.default_rng(8)
    x, y = rand_cloud(rng, 40, 3), rand_cloud(rng, 33, 3)
    g = rng.standard_normal(33)
    full = O.f_update(x, y, g, 0.4)
    rows = np.array([0, 5, 39, 17])
    assert np.array_equal(O.f_update(x, y, g, 0.4, rows=rows), full[rows])
    # one f-update makes the row marginals exact
    rs = O.plan_row_sums(x, y, full, g, 0.4, np.arange(40))
    assert np.allclose(rs, 1 / 40, rtol=1e-12)


# ------------------------------------------------------------------ 1D: sort, eps->0
def test_sort_rank_stable_ties(O):
    x = np.array([[0.5, -0.0, 0.1, 0.0, 0.5, -1.0]], np.float32)
    perm, rank = O.sort_rank(x)
    assert perm.tolist() == [[5, 1, 3, 2, 0, 4]]   # -0.0 == +0.0 -> index order
    assert np.array_equal(rank[0][perm[0]], np.arange(6))
    rng = np.random.default_rng(9)
    xb = rng.integers(0, 50, (64, 200)).astype(np.float32)  # heavy ties
    perm, rank = O.sort_rank(xb)
    assert np.array_equal(perm, np.argsort(xb, axis=1, kind="stable"))
    with pytest.raises(ValueError):
        O.sort_rank(np.array([1.0, np.nan], np.float32))


def brute_assignment(C):
    n = C.shape[0]
    return min(sum(C[i, p[i]] for i in range(n)) for p in itertools.permutations(range(n))) / n


@pytest.mark.parametrize("n", [2, 3, 4, 5, 6])
def test_1d_eps0_limit_sorted_matching_is_lp_optimum(O, n):
    rng = np.random.default_rng(10 + n)
    for _ in range(5):
        x, y = rng.normal(size=n).astype(np.float32), rng.normal(size=n).astype(np.float32)
        C = O.cost_matrix(x.reshape(-1, 1), y.reshape(-1, 1))
        W_lp = brute_assignment(C)
        xs, ys = np.sort(x).astype(np.float64), np.sort(y).astype(np.float64)
        W_sorted = float(np.mean((xs - ys) ** 2))              # P:110 NW solution, n=m uniform
        assert abs(W_lp - W_sorted) < 1e-12
        # DualSort fixed point certifies optimality: feasible and tight on the diagonal (A.1-A.2)
        f, _ = O.dualsort(xs, ys)
        Cs = (xs[:, None] - ys[None, :]) ** 2
        g = np.diag(Cs) - f
        assert np.all(f[:, None] + g[None, :] <= Cs + 1e-12)
        assert abs((f.mean() + g.mean()) - W_lp) < 1e-12
        # entropic brackets: W - eps(1+log nm) <= E* <= W - eps(1+log n) (DESIGN.md pin)
        for eps in (1.0, 0.1, 0.01):
            r = O.sinkhorn(x.reshape(-1, 1), y.reshape(-1, 1), eps, tol=1e-12, max_iter=200000)
            assert W_lp - eps * (1 + math.log(n * n)) - 1e-9 <= r.E <= W_lp - eps * (1 + math.log(n)) + 1e-9


def test_dualsort_golden_and_paper_mode(O):
    gd = GOLD["dualsort_swap"]
    f, s = O.dualsort(gd["xs"], gd["ys"])
    assert f.tolist() == gd["f"]
    rng = np.random.default_rng(11)
    xs, ys = np.sort(rng.random(50)), np.sort(rng.random(50))
    Cs = (xs[:, None] - ys[None, :]) ** 2
    f1, s1 = O.dualsort(xs, ys, sweeps=1)
    assert s1 == 1 and np.allclose(f1, np.min(Cs - np.diag(Cs)[None, :], axis=1), atol=0)
    f, s = O.dualsort(xs, ys)
    assert s <= 51
    # the fixed point is the largest f <= 0 satisfying feasibility (reading R-7):
    # perturbing any entry upward breaks feasibility or the f <= 0 cap.
    g = np.diag(Cs) - f
    slack = Cs - f[:, None] - g[None, :]
    assert slack.min() > -1e-12


def test_init_sort1d_equivariance(O):
    rng = np.random.default_rng(12)
    x = rng.random(64).astype(np.float32)
    y = (np.arange(64) / 63).astype(np.float32)
    f0 = O.init_sort1d(x, y)
    p = rng.permutation(64)
    assert np.allclose(O.init_sort1d(x[p], y)[np.argsort(p)], f0, atol=0)


def test_sort1d_init_helps_on_1d(O):
    # Sec. 3.1 claim on a small instance: the ε=0 dual is a much better start than 0
    rng = np.random.default_rng(13)
    x = rng.random(128).astype(np.float32).reshape(-1, 1)
    y = (np.arange(128) / 127).astype(np.float32).reshape(-1, 1)
    eps = 1e-3
    r0 = O.sinkhorn(x, y, eps)
    r1 = O.sinkhorn(x, y, eps, f0=O.init_sort1d(x, y))
    assert r1.converged and r1.iterations < r0.iterations / 2


# ------------------------------------------------------------------ Gaussian
def test_bures_and_monge_closed_forms(O):
    gb = GOLD["bures_4I_I"]
    assert abs(O.bures2(4 * np.eye(2), np.eye(2)) - gb["value"]) < 1e-12
    assert np.allclose(O.monge_A(np.eye(3), 4 * np.eye(3)), GOLD["monge_I_4I"]["A_diag"] * np.eye(3))
    rng = np.random.default_rng(14)
    G = rng.standard_normal((4, 4)); S = G @ G.T + 0.1 * np.eye(4)
    assert np.allclose(O.monge_A(S, S), np.eye(4), atol=1e-10)
    assert abs(O.bures2(S, S)) < 1e-10
    H = rng.standard_normal((4, 4)); T = H @ H.T + 0.2 * np.eye(4)
    assert abs(O.bures2(S, T) - O.bures2(T, S)) < 1e-10
    A = O.monge_A(S, T)
    assert np.allclose(A, A.T) and np.allclose(A @ S @ A, T, atol=1e-9)       # push-forward
    # W2^2 via the map, E||x - T(x)||^2 = tr((I-A) S (I-A)) + |dm|^2, equals Eq. (6)
    m1, m2 = rng.standard_normal(4), rng.standard_normal(4)
    I = np.eye(4)
    assert abs(np.trace((I - A) @ S @ (I - A)) + np.sum((m1 - m2) ** 2) - O.w2_gaussians(m1, S, m2, T)) < 1e-9


def _sigma_point_mean(q, m, S):
    """Exact E[q(y)] for quadratic q, y ~ N(m, S): q(m) + 1/2 sum_k [q(m+Le_k)+q(m-Le_k)-2q(m)]."""
    L = np.linalg.cholesky(S)
    q0 = q(m)
    return q0 + 0.5 * sum(q(m + L[:, k]) + q(m - L[:, k]) - 2 * q0 for k in range(len(m)))


def test_gaussian_potential_is_optimal_dual(O):
    """Gaussian-Potential appendix, cost ||x-y||^2: E_mu[f] + E_nu[f^c] = W2^2 (Eq. 6)
    and T = Id - 1/2 grad f.  This pins the sign of the linear term (reading R-4)."""
    rng = np.random.default_rng(15)
    d = 3
    G = rng.standard_normal((d, d)); S1 = G @ G.T + 0.3 * np.eye(d)
    H = rng.standard_normal((d, d)); S2 = H @ H.T + 0.3 * np.eye(d)
    m1, m2 = rng.standard_normal(d), rng.standard_normal(d)
    A = O.monge_A(S1, S2)
    f = lambda x: float(O.gaussian_potential(np.asarray(x)[None, :], m1, m2, A)[0])
    Ai = np.linalg.inv(A)

    def fc(y):  # c-transform, minimiser x* = m1 + A^{-1}(y - m2) (grad of |x-y|^2 - f vanishes)
        xs = m1 + Ai @ (y - m2)
        return float(np.sum((xs - y) ** 2)) - f(xs)

    # x* really is the minimiser (finite differences of |x-y|^2 - f(x))
    yv = rng.standard_normal(d)
    xs = m1 + Ai @ (yv - m2)
    obj = lambda x: float(np.sum((x - yv) ** 2)) - f(x)
    for k in range(d):
        e = np.zeros(d); e[k] = 1e-5
        assert abs((obj(xs + e) - obj(xs - e)) / 2e-5) < 1e-6
    dual = _sigma_point_mean(f, m1, S1) + _sigma_point_mean(fc, m2, S2)
    assert abs(dual - O.w2_gaussians(m1, S1, m2, S2)) < 1e-9
    # T(x) = A(x - m1) + m2 = x - 1/2 grad f(x)
    x0 = rng.standard_normal(d)
    grad = np.array([(f(x0 + h) - f(x0 - h)) / 2e-6 for h in np.eye(d) * 1e-6])
    assert np.allclose(x0 - 0.5 * grad, A @ (x0 - m1) + m2, atol=1e-6)
    # Eq. (5)'s printed linear term (m2 - A m1) with the 1/2-cost convention fails this test
    f5 = lambda x: 0.5 * x @ (np.eye(d) - A) @ x + (m2 - A @ m1) @ x
    grad5 = np.array([(f5(x0 + h) - f5(x0 - h)) / 2e-6 for h in np.eye(d) * 1e-6])
    assert not np.allclose(x0 - grad5, A @ (x0 - m1) + m2, atol=1e-3)


def test_gaussian_special_cases(O):
    rng = np.random.default_rng(16)
    x = rng.standard_normal((500, 2)).astype(np.float32)
    # equal moments -> A = I -> f constant (= -|m|^2)
    f0, side = O.init_gaussian(x, x)
    assert side == 0 and np.ptp(f0) < 1e-9
    # m_mu = 0, m_nu = t, S = I -> f = -2 t^T x
    t = np.array([0.7, -0.2])
    A = O.monge_A(np.eye(2), np.eye(2))
    f = O.gaussian_potential(x, np.zeros(2), t, A)
    assert np.allclose(f, -2 * x.astype(np.float64) @ t, atol=1e-12)
    # moments: independent numpy weighted covariance
    w = rng.uniform(0.5, 1.5, 500); w /= w.sum()
    m, S = O.moments(x, w, ridge_rel=0.0)
    assert np.allclose(m, np.average(x, axis=0, weights=w))
    assert np.allclose(S, np.cov(x.T.astype(np.float64), aweights=w, bias=True), atol=1e-12)
    # side selection: n > m -> potential on y
    _, side = O.init_gaussian(x, x[:100])
    assert side == 1


# ------------------------------------------------------------------ GMM
def _mix(rng, K, d):
    means = rng.normal(0, 2, (K, d))
    covs = []
    for _ in range(K):
        G = rng.standard_normal((d, d)) / np.sqrt(d)
        covs.append(G.T @ G + 0.05 * np.eye(d))
    w = rng.uniform(0.5, 1.5, K); w /= w.sum()
    return {"weights": w, "means": means, "covs": np.array(covs)}


def test_gmm_responsibilities_independent(O):
    from scipy.stats import multivariate_normal
    rng = np.random.default_rng(17)
    g = _mix(rng, 4, 3)
    x = rng.standard_normal((50, 3)) * 2
    lr = O.gmm_log_resp(x, g["weights"], g["means"], g["covs"])
    dens = np.stack([g["weights"][k] * multivariate_normal(g["means"][k], g["covs"][k]).pdf(x)
                     for k in range(4)], 1)
    assert np.allclose(np.exp(lr), dens / dens.sum(1, keepdims=True), atol=1e-12)
    assert np.allclose(np.exp(lr).sum(1), 1.0)


def test_gmm_cost_and_init_properties(O):
    rng = np.random.default_rng(18)
    gx, gy = _mix(rng, 3, 2), _mix(rng, 3, 2)
    C = O.gmm_cost(gx["means"], gx["covs"], gx["means"], gx["covs"])
    assert np.allclose(np.diag(C), 0, atol=1e-10)
    I = np.array([np.eye(2)] * 3)
    Ci = O.gmm_cost(gx["means"], I, gy["means"], I)
    assert np.allclose(Ci, ((gx["means"][:, None] - gy["means"][None]) ** 2).sum(-1), atol=1e-12)
    x = rng.standard_normal((40, 2)).astype(np.float32)
    y = rng.standard_normal((60, 2)).astype(np.float32)
    # K = 1 -> responsibilities are 1 -> constant potential
    g1 = {k: v[:1] for k, v in gx.items()}; g1["weights"] = np.ones(1)
    h1 = {k: v[:1] for k, v in gy.items()}; h1["weights"] = np.ones(1)
    f, side = O.init_gmm(x, y, g1, h1, 0.5)
    assert side == 0 and np.ptp(f) < 1e-12
    # relabelling invariance
    f, _ = O.init_gmm(x, y, gx, gy, 0.5)
    p = [2, 0, 1]
    gp = {k: v[p] for k, v in gx.items()}
    fp, _ = O.init_gmm(x, y, gp, gy, 0.5)
    assert np.allclose(f, fp, atol=1e-9)


def _tiny_cov_mixture(points, weights, var=1e-8):
    d = points.shape[1]
    return {"weights": np.asarray(weights, np.float64), "means": np.asarray(points, np.float64),
            "covs": np.array([var * np.eye(d)] * len(points))}


@pytest.mark.parametrize("n,m", [(6, 9), (9, 6)])
def test_gmm_init_point_limit_is_the_point_cloud_potential(O, n, m):
    """"in the limit where K -> n, n components with means (x_i)_i and zero covariance"
    the GMM initializer recovers the original potential f*.  Components at the points with
    covariance 1e-8 I (Bures cost 0, responsibilities one-hot) and the points' own weights: the
    centred f^(0) equals the converged point-cloud potential of the oracle's Sinkhorn (on the
    smaller side: f* for n <= m, g* otherwise).  Non-uniform weights and n != m, so a
    transposed or side-swapped K x K problem, a sign error or a wrong eps fails."""
    rng = np.random.default_rng(40 + n)
    x = rng.uniform(-1, 1, (n, 2)).astype(np.float32)
    y = (rng.uniform(-1, 1, (m, 2)) + 0.3).astype(np.float32)
    a = rng.uniform(0.5, 1.5, n); a /= a.sum()
    b = rng.uniform(0.5, 1.5, m); b /= b.sum()
    eps = 0.3
    f0, side = O.init_gmm(x, y, _tiny_cov_mixture(x, a), _tiny_cov_mixture(y, b), eps)
    ref = O.sinkhorn(x, y, eps, a=a, b=b, tol=1e-13, max_iter=200000)
    assert ref.converged
    want = ref.f if n <= m else ref.g
    assert side == (0 if n <= m else 1)
    c = (f0 - f0.mean()) - (want - want.mean())
    assert np.abs(c).max() <= 1e-6 * max(np.abs(want).max(), eps), np.abs(c).max()
    # the same with a wrong eps, or the transposed problem, is far off (the pin discriminates)
    f_bad, _ = O.init_gmm(x, y, _tiny_cov_mixture(x, a), _tiny_cov_mixture(y, b), 2 * eps)
    assert np.abs((f_bad - f_bad.mean()) - (want - want.mean())).max() > 1e-3


def test_gmm_init_separated_components_take_their_dual_value(O):
    """Well-separated components with tiny covariances: every point's
    responsibilities are one-hot at its own component, so f^(0)_i = f~_k(i), and f~ is the dual of
    the discrete problem between the component means with weights (alpha, beta) (Bures cost 0 for
    equal covariances, Eq. 6) - solved here as a point-cloud problem of the means."""
    rng = np.random.default_rng(44)
    mx = np.array([[0.0, 0.0], [6.0, 0.0], [0.0, 7.0]])
    my = np.array([[1.0, 1.0], [5.0, 2.0], [2.0, 6.0], [7.0, 7.0]])
    al = np.array([0.5, 0.3, 0.2]); be = np.array([0.1, 0.4, 0.3, 0.2])
    lab = rng.integers(0, 3, 40)
    x = (mx[lab] + 1e-4 * rng.standard_normal((40, 2))).astype(np.float32)
    y = rng.standard_normal((60, 2)).astype(np.float32)
    eps = 1.5
    gx, gy = _tiny_cov_mixture(mx, al, 1e-6), _tiny_cov_mixture(my, be, 1e-6)
    f0, side = O.init_gmm(x, y, gx, gy, eps)
    ref = O.sinkhorn(mx.astype(np.float32), my.astype(np.float32), eps, a=al, b=be, tol=1e-13, max_iter=200000)
    # the means are exact in fp32 here, so the point problem is the K x K problem
    diff = f0 - ref.f[lab]
    assert side == 0 and np.ptp(diff) <= 1e-7 * max(np.abs(ref.f).max(), eps), np.ptp(diff)


def test_gmm_dual_plain_and_anderson_land_on_the_same_solution(O):
    """The K x K problem's solution does not depend on the solver (R-29: the GPU's K11 solves it
    with Anderson): plain Sinkhorn (the oracle, O2) and Anderson (memory 5) to 1e-12 give the same
    gauge-fixed f~."""
    rng = np.random.default_rng(45)
    gx, gy = _mix(rng, 6, 3), _mix(rng, 5, 3)
    ft, r = O.gmm_dual(gx, gy, 0.4)
    assert r.converged and r.err < 1e-12
    C = O.gmm_cost(gx["means"], gx["covs"], gy["means"], gy["covs"])
    ra = O.sinkhorn_matrix(C, 0.4, a=gx["weights"], b=gy["weights"], tol=1e-12, max_iter=100000, anderson=5)
    a = np.asarray(gx["weights"], np.float64)
    fa = ra.f - (a * ra.f).sum() / a.sum()
    assert ra.converged and ra.iterations < r.iterations
    assert np.abs(fa - ft).max() <= 1e-7 * np.abs(ft).max()
    with pytest.raises(ValueError):
        O.sinkhorn_matrix(C, 0.4, a=gx["weights"], b=gy["weights"], anderson=17)


# ------------------------------------------------------------------ adaptive momentum (R-31)
def test_adaptive_momentum_reduces_to_the_pinned_solvers(O):
    """Adaptive momentum ("adapt=10"; reading R-31) is the plain solver
    until its first adaptation and the (pinned) relaxed solver between adaptations:
    (a) the first 2T + 1 sweeps equal plain Sinkhorn exactly;
    (b) the omega it switches to at sweep 2T + 2 is 2/(1 + sqrt(1 - rho)) with rho the per-sweep
        contraction of the explicit L1 errors of an independent plain run at sweeps T and 2T;
    (c) the next T sweeps equal the relaxed solver at that omega started from (f, g) of sweep
        2T + 1;  (d) it reaches the plain optimum, in fewer sweeps than plain Sinkhorn on C1."""
    p = gen.c1()
    T = 10
    plain = O.sinkhorn(p.x, p.y, p.eps, tol=0, max_iter=2 * T + 1)
    ad = O.sinkhorn_adaptive(p.x, p.y, p.eps, T, tol=0, max_iter=2 * T + 1)
    assert np.array_equal(ad.f, plain.f) and np.array_equal(ad.g, plain.g)
    assert np.all(ad.omega == 1.0)
    eT = O.marginal_error(p.x, p.y, *[O.sinkhorn(p.x, p.y, p.eps, tol=0, max_iter=T)[k] for k in ("f", "g")], p.eps)
    e2T = O.marginal_error(p.x, p.y, *[O.sinkhorn(p.x, p.y, p.eps, tol=0, max_iter=2 * T)[k] for k in ("f", "g")],
                           p.eps)
    rho = (e2T / eT) ** (1.0 / T)
    w_star = min(max(2.0 / (1.0 + math.sqrt(max(0.0, 1.0 - rho))), 1.0), 1.95)
    s = T - 1
    long = O.sinkhorn_adaptive(p.x, p.y, p.eps, T, tol=0, max_iter=2 * T + 1 + s)
    assert abs(long.omega[2 * T + 1] - w_star) < 1e-12 and 1.0 < w_star < 1.95
    assert np.all(long.omega[2 * T + 1:] == long.omega[2 * T + 1])
    rel = O.sinkhorn_adaptive(p.x, p.y, p.eps, 0, tol=0, max_iter=s, f0=ad.f, g0=ad.g, omega=long.omega[2 * T + 1])
    assert np.abs(rel.f - long.f).max() < 1e-12 and np.abs(rel.g - long.g).max() < 1e-12
    # g0 is read by the relaxed g-update only: at omega = 1 it changes nothing
    r1 = O.sinkhorn_adaptive(p.x, p.y, p.eps, 0, tol=0, max_iter=3, g0=np.full(p.m, 5.0))
    r2 = O.sinkhorn(p.x, p.y, p.eps, tol=0, max_iter=3)
    assert np.array_equal(r1.f, r2.f) and np.array_equal(r1.g, r2.g)
    # (d) the same optimum, fewer sweeps
    ref = O.sinkhorn(p.x, p.y, p.eps, tol=1e-10, max_iter=100000)
    adc = O.sinkhorn_adaptive(p.x, p.y, p.eps, T, tol=1e-10, max_iter=100000)
    assert adc.converged and adc.iterations < ref.iterations
    fa, ga = adc.f - adc.f.mean(), adc.g + adc.f.mean()
    fr, gr = ref.f - ref.f.mean(), ref.g + ref.f.mean()
    assert np.abs(fa - fr).max() < 1e-7 * max(np.abs(fr).max(), 1) and np.abs(ga - gr).max() < 1e-7 * max(np.abs(gr).max(), 1)
    at = O.sinkhorn_adaptive(p.x, p.y, p.eps, T)
    assert at.converged and at.iterations < O.sinkhorn(p.x, p.y, p.eps).iterations / 2
    assert abs(O.marginal_error(p.x, p.y, at.f, at.g, p.eps) - at.err) < 1e-12


# ------------------------------------------------------------------ Subsample
def test_subsample_full_equals_solution(O):
    rng = np.random.default_rng(19)
    n = 48
    x, y = rand_cloud(rng, n, 2), rand_cloud(rng, n, 2, 0.5)
    eps = 0.2
    idx = np.arange(n)
    f0, side, inner = O.init_subsample(x, y, idx, idx, eps, inner_tol=1e-11, inner_max_iter=100000)
    full = O.sinkhorn(x, y, eps, tol=1e-11, max_iter=100000)
    assert side == 0 and inner.converged
    assert np.allclose(O.center(f0), O.center(full.f), atol=1e-9)


def test_subsample_degenerate_and_shift(O):
    rng = np.random.default_rng(20)
    x, z = rand_cloud(rng, 30, 3), rand_cloud(rng, 1, 3)
    gb = np.array([0.3])
    f0 = O.subsample_extrapolate(x, z, gb, 0.05)
    c = ((x.astype(np.float64) - z.astype(np.float64)) ** 2).sum(1)
    assert np.allclose(f0, c - 0.3, atol=1e-12)
    z = rand_cloud(rng, 12, 3)
    gb = rng.standard_normal(12)
    assert np.allclose(O.subsample_extrapolate(x, z, gb + 0.9, 0.3),
                       O.subsample_extrapolate(x, z, gb, 0.3) - 0.9, atol=1e-12)


# ------------------------------------------------------------------ sharded decomposition (O9)
def test_shard_merge_equals_unsharded_g_update(O):
    rng = np.random.default_rng(21)
    x, y = rand_cloud(rng, 64, 3), rand_cloud(rng, 40, 3)
    f = rng.standard_normal(64)
    eps = 0.25
    b = np.full(40, 1 / 40)
    parts = [O.column_partials(x[s], y, f[s], eps) for s in (slice(0, 16), slice(16, 48), slice(48, 64))]
    assert np.allclose(O.merge_partials(parts, b, eps), O.g_update(x, y, f, eps), atol=1e-12)


# ------------------------------------------------- Alg. 1 relaxation (NEXT-1, omega != 1)
def test_relaxed_one_point_closed_form():
    """n = m = 1, a = b = 1, C = [[c]]: g_sk(f) = c - f and f_sk(g) = c - g (soft-min of one
    entry), so the relaxed sweep of Alg. 1 (R-1) is the linear recurrence
        g <- (1 - w) g + w (c - f),   f <- (1 - w) f + w (c - g)
    derived by hand; the oracle's generic LSE path must reproduce it sweep for sweep."""
    from oracle import oracle as O
    c, f0, eps = 2.5, 0.7, 0.3
    x = np.array([[0.0]])
    y = np.array([[np.sqrt(c)]])
    for w in (0.6, 1.0, 1.5, 1.9):
        f, g = f0, 0.0
        for L in range(1, 7):
            g = (1 - w) * g + w * (c - f)
            f = (1 - w) * f + w * (c - g)
            r = O.sinkhorn(x, y, eps, tol=0, max_iter=L, f0=np.array([f0]), omega=w)
            assert abs(r.f[0] - f) < 1e-12 and abs(r.g[0] - g) < 1e-12, (w, L)
            # Eq. (2) with one atom: E = f + g - eps exp((f + g - c)/eps)
            assert abs(r.E - (f + g - eps * np.exp((f + g - c) / eps))) < 1e-12


def test_relaxed_iterations_reach_the_same_optimum():
    """The relaxed map's fixed points are the Sinkhorn fixed points for any omega != 0:
    omega in {0.7, 1.5} converges to the omega = 1 optimum (centred potentials, E)."""
    from oracle import oracle as O
    p = gen.c1(n=40, seed=2, eps_factor=0.1)
    ref = O.sinkhorn(p.x, p.y, p.eps, tol=1e-11, max_iter=100000)
    assert ref.converged
    fr = ref.f - ref.f.mean()
    for w in (0.7, 1.5):
        r = O.sinkhorn(p.x, p.y, p.eps, tol=1e-11, max_iter=100000, omega=w)
        assert r.converged and r.err < 1e-11
        assert np.abs((r.f - r.f.mean()) - fr).max() < 1e-8 * max(1.0, np.abs(fr).max())
        assert abs(r.E - ref.E) < 1e-10 * max(1.0, abs(ref.E))


def test_relaxed_error_and_objective_are_explicit():
    """With omega != 1 the rows are not exact after an f-update: the oracle's err and E are
    the explicit plan sums (threshold appendix, Eq. 2), recomputed here from the returned pair."""
    from oracle import oracle as O
    p = gen.c1(n=40, seed=4)
    r = O.sinkhorn(p.x, p.y, p.eps, tol=0, max_iter=5, omega=1.6)
    x, y = p.x.astype(np.float64), p.y.astype(np.float64)
    C = ((x[:, None, :] - y[None, :, :]) ** 2).sum(-1)
    P = np.exp((r.f[:, None] + r.g[None, :] - C) / p.eps)
    n, m = C.shape
    err = np.abs(P.sum(1) - 1 / n).sum() + np.abs(P.sum(0) - 1 / m).sum()
    assert abs(r.err - err) < 1e-12 * max(1.0, err)
    E = r.f.mean() + r.g.mean() - p.eps * P.sum()
    assert abs(r.E - E) < 1e-12 * max(1.0, abs(E))
    assert np.abs(P.sum(1) - 1 / n).sum() > 1e-6   # the row term is really non-zero here


# ------------------------------------------------------ soft ranks / soft sort (NEXT-2)
def test_soft_rank_sort_eps_to_zero_gives_hard_ranks_and_sort():
    """as eps -> 0 the entropic plan tends to the sorted matching, so n P z -> the
    ranks of x (1-based) and n P^T x -> sorted x; checked against numpy's argsort / sort."""
    from oracle import oracle as O
    rng = np.random.default_rng(11)
    n = 6
    x = rng.random(n)
    y = np.linspace(0.0, 1.0, n)
    ranks = np.empty(n)
    ranks[np.argsort(x, kind="stable")] = np.arange(1, n + 1)
    errs = []
    f0 = O.init_sort1d(x, y)   # the sorted eps = 0 dual: the small-eps solves converge fast
    for eps in (1e-2, 1e-3, 2e-4):
        r = O.sinkhorn(x[:, None], y[:, None], eps, tol=1e-6, max_iter=2000000, f0=f0)
        assert r.converged
        rk, st = O.soft_rank_sort(x, y, r.f, r.g, eps)
        errs.append(max(np.abs(rk - ranks).max(), np.abs(st - np.sort(x)).max()))
    assert errs[-1] < 1e-3 and errs[0] > errs[-1]   # converges to the hard operators


def test_soft_rank_equals_literal_nPz_when_marginals_are_uniform_and_is_equivariant():
    """R-22: the conditional means equal the paper's literal n P z and n P^T x when P has
    the uniform marginals: after the oracle's last f-update the rows are exactly 1/n, so the rank
    must equal n P z to rounding; at convergence (tol 1e-10) the sort equals n P^T x.  And
    permuting x permutes the soft ranks and leaves the soft sort unchanged."""
    from oracle import oracle as O
    rng = np.random.default_rng(12)
    n = 9
    x, y = rng.random(n), np.linspace(0.0, 1.0, n)
    eps = 0.02
    r = O.sinkhorn(x[:, None], y[:, None], eps, tol=1e-10, max_iter=100000)
    rk, st = O.soft_rank_sort(x, y, r.f, r.g, eps)
    P = np.exp((r.f[:, None] + r.g[None, :] - (x[:, None] - y[None, :]) ** 2) / eps)
    z = np.arange(1, n + 1)
    assert np.abs(rk - n * P @ z).max() < 1e-9 * n
    assert np.abs(st - n * P.T @ x).max() < 1e-8
    perm = rng.permutation(n)
    rp = O.sinkhorn(x[perm, None], y[:, None], eps, tol=1e-10, max_iter=100000)
    rk2, st2 = O.soft_rank_sort(x[perm], y, rp.f, rp.g, eps)
    assert np.abs(rk2 - rk[perm]).max() < 1e-6 and np.abs(st2 - st).max() < 1e-6


# --------------------------------------------------------------- GMM fitting (NEXT-3)
def test_gmm_fit_matches_sklearn_em():
    """The oracle's EM is sklearn's GaussianMixture (full covariance, the paper's fitting tool,
    P:568) started from the same parameters: equal weights, means and covariances."""
    from oracle import oracle as O
    from sklearn.mixture import GaussianMixture
    rng = np.random.default_rng(21)
    x = np.concatenate([rng.standard_normal((300, 3)) * 0.5 + c for c in ([0, 0, 0], [3, 1, 0], [-2, 2, 1])])
    K, iters, reg = 3, 12, 1e-6
    idx = rng.choice(len(x), K, replace=False)
    w, m, S, ll = O.gmm_fit(x, K, idx, iters, reg)
    m0 = x.mean(0)
    cov0 = (x - m0).T @ (x - m0) / len(x) + reg * np.eye(3)
    gm = GaussianMixture(K, covariance_type="full", reg_covar=reg, max_iter=iters, tol=0.0, init_params="random",
                         weights_init=np.full(K, 1.0 / K), means_init=x[idx],
                         precisions_init=np.repeat(np.linalg.inv(cov0)[None], K, 0), random_state=0)
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        gm.fit(x)
    assert np.abs(w - gm.weights_).max() < 1e-10
    assert np.abs(m - gm.means_).max() < 1e-9
    assert np.abs(S - gm.covariances_).max() < 1e-9
    assert abs(ll - gm.score(x)) < 1e-9


def test_gmm_fit_em_monotone_and_single_component_closed_form():
    """EM never decreases the likelihood (textbook property); K = 1 gives the sample mean and
    biased covariance (+ reg) after one step, whatever the start."""
    from oracle import oracle as O
    rng = np.random.default_rng(22)
    x = rng.standard_normal((400, 4)) @ rng.standard_normal((4, 4)) + 1.5
    idx = rng.choice(400, 4, replace=False)
    lls = [O.gmm_fit(x, 4, idx, t)[3] for t in range(0, 8)]
    assert all(b >= a - 1e-12 for a, b in zip(lls, lls[1:]))
    w, m, S, _ = O.gmm_fit(x, 1, [7], 1, 1e-6)
    mu = x.mean(0)
    assert abs(w[0] - 1) < 1e-12 and np.abs(m[0] - mu).max() < 1e-12
    assert np.abs(S[0] - ((x - mu).T @ (x - mu) / 400 + 1e-6 * np.eye(4))).max() < 1e-12


def test_kmeans_matches_sklearn_lloyd():
    """R-28: the oracle's Lloyd iterations are sklearn's KMeans (algorithm="lloyd", the same
    initial centers, n_init=1, tol=0) for several iteration counts: equal centers and labels."""
    from oracle import oracle as O
    from sklearn.cluster import KMeans
    rng = np.random.default_rng(23)
    x = np.concatenate([rng.standard_normal((250, 4)) * 0.7 + c for c in rng.standard_normal((4, 4)) * 3])
    idx = rng.choice(len(x), 4, replace=False)
    for T in (1, 3, 20):
        c, lab = O.kmeans(x, idx, T)
        km = KMeans(4, init=x[idx], n_init=1, max_iter=T, tol=0.0, algorithm="lloyd").fit(x)
        assert np.abs(c - km.cluster_centers_).max() < 1e-12, T
        assert np.array_equal(lab, km.labels_), T


def test_gmm_fit_kmeans_start_matches_sklearn_em():
    """R-28: with kmeans_iters > 0 the fit starts from the one-hot M-step of the k-means labels
    (sklearn's init_params="kmeans"), written here independently (counts, cluster means, np.cov
    with bias), and the EM steps then equal sklearn's GaussianMixture from that start."""
    from oracle import oracle as O
    from sklearn.mixture import GaussianMixture
    rng = np.random.default_rng(24)
    x = np.concatenate([rng.standard_normal((300, 3)) * 0.6 + c for c in ([0, 0, 0], [3, 1, 0], [-2, 2, 1])])
    K, reg = 3, 1e-6
    idx = rng.choice(len(x), K, replace=False)
    _, lab = O.kmeans(x, idx, 5)
    w0 = np.array([(lab == k).sum() for k in range(K)]) / len(x)
    m0 = np.stack([x[lab == k].mean(0) for k in range(K)])
    S0 = np.stack([np.cov(x[lab == k].T, bias=True) + reg * np.eye(3) for k in range(K)])
    w, m, S, _ = O.gmm_fit(x, K, idx, 0, reg, kmeans_iters=5)
    assert np.abs(w - w0).max() < 1e-12 and np.abs(m - m0).max() < 1e-12 and np.abs(S - S0).max() < 1e-12
    w, m, S, ll = O.gmm_fit(x, K, idx, 7, reg, kmeans_iters=5)
    gm = GaussianMixture(K, covariance_type="full", reg_covar=reg, max_iter=7, tol=0.0, init_params="random",
                         weights_init=w0, means_init=m0, precisions_init=np.linalg.inv(S0), random_state=0)
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        gm.fit(x)
    assert np.abs(w - gm.weights_).max() < 1e-10
    assert np.abs(m - gm.means_).max() < 1e-9
    assert np.abs(S - gm.covariances_).max() < 1e-9
    assert abs(ll - gm.score(x)) < 1e-9


def test_gmm_fit_tol_stops_like_sklearn():
    """R-28: with tol > 0 the EM loop stops as sklearn's GaussianMixture(tol) does: the same
    iteration count and parameters from the same start."""
    from oracle import oracle as O
    from sklearn.mixture import GaussianMixture
    rng = np.random.default_rng(25)
    x = np.concatenate([rng.standard_normal((400, 3)) * 0.8 + c for c in ([0, 0, 0], [2.5, 1, 0], [-2, 2, 1])])
    K, reg = 3, 1e-6
    idx = rng.choice(len(x), K, replace=False)
    _, lab = O.kmeans(x, idx, 6)
    w0 = np.array([(lab == k).sum() for k in range(K)]) / len(x)
    m0 = np.stack([x[lab == k].mean(0) for k in range(K)])
    S0 = np.stack([np.cov(x[lab == k].T, bias=True) + reg * np.eye(3) for k in range(K)])
    import warnings
    for tol in (1e-2, 1e-3, 1e-5):
        w, m, S, ll, it = O.gmm_fit(x, K, idx, 100, reg, kmeans_iters=6, tol=tol, return_iters=True)
        gm = GaussianMixture(K, covariance_type="full", reg_covar=reg, max_iter=100, tol=tol,
                             weights_init=w0, means_init=m0, precisions_init=np.linalg.inv(S0))
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            gm.fit(x)
        assert it == gm.n_iter_, (tol, it, gm.n_iter_)
        assert np.abs(m - gm.means_).max() < 1e-9 and np.abs(S - gm.covariances_).max() < 1e-9
        assert np.abs(w - gm.weights_).max() < 1e-10


# --------------------------------------------------- implicit differentiation (NEXT-4)
def _solve_tight(O, x, y, eps, a=None, b=None, f0=None):
    r = O.sinkhorn(x, y, eps, a=a, b=b, tol=1e-13, max_iter=200000, f0=f0)
    assert r.converged
    return r


def test_vjp_matches_finite_differences_of_the_solve():
    """the implicit VJP equals central differences of the (tightly converged) oracle
    solve for a shift-invariant loss l = <zf, f*> + <zg, g*> (sum zf = sum zg), w.r.t. x, y and
    simplex-tangent perturbations of a."""
    from oracle import oracle as O
    rng = np.random.default_rng(31)
    n, m, d = 6, 5, 2
    x, y = rng.standard_normal((n, d)), rng.standard_normal((m, d)) + 0.3
    a = gen.random_weights(n, rng).astype(np.float64)
    eps = 0.4
    zf, zg = rng.standard_normal(n), rng.standard_normal(m)
    zg += (zf.sum() - zg.sum()) / m
    base = _solve_tight(O, x, y, eps, a=a)
    gx, gy, ga, _ = O.sinkhorn_vjp(x, y, base.f, base.g, eps, zf, zg)  # (the VJP itself takes a only via f, g)

    def loss(xx, yy, aa):
        r = _solve_tight(O, xx, yy, eps, a=aa, f0=base.f)
        return zf @ r.f + zg @ r.g
    h = 1e-5
    for i, k in [(0, 0), (3, 1), (5, 0)]:
        dx = np.zeros_like(x); dx[i, k] = h
        fd = (loss(x + dx, y, a) - loss(x - dx, y, a)) / (2 * h)
        assert abs(fd - gx[i, k]) < 1e-6 * max(1.0, abs(fd)), (i, k, fd, gx[i, k])
    for j, k in [(1, 0), (4, 1)]:
        dy = np.zeros_like(y); dy[j, k] = h
        fd = (loss(x, y + dy, a) - loss(x, y - dy, a)) / (2 * h)
        assert abs(fd - gy[j, k]) < 1e-6 * max(1.0, abs(fd)), (j, k, fd, gy[j, k])
    da = np.zeros(n); da[1], da[4] = h, -h    # tangent to the simplex
    fd = (loss(x, y, a + da) - loss(x, y, a - da)) / (2 * h)
    assert abs(fd - (ga[1] - ga[4])) < 1e-6 * max(1.0, abs(fd))


def test_vjp_envelope_closed_form():
    """z = (a, b): l = <a, f*> + <b, g*> = E* + eps, and by the envelope theorem
    dE*/dx_i = sum_j P_ij dC_ij/dx_i = 2 sum_j P_ij (x_i - y_j) (closed form, no linear solve)."""
    from oracle import oracle as O
    p = gen.c1(n=48, seed=5, eps_factor=0.05)
    r = _solve_tight(O, p.x, p.y, p.eps)
    n = len(r.f)
    gx, gy, _, _ = O.sinkhorn_vjp(p.x, p.y, r.f, r.g, p.eps, np.full(n, 1 / n), np.full(len(r.g), 1 / len(r.g)))
    x, y = p.x.astype(np.float64), p.y.astype(np.float64)
    C = ((x[:, None] - y[None]) ** 2).sum(-1)
    P = np.exp((r.f[:, None] + r.g[None] - C) / p.eps)
    env_x = 2 * (P.sum(1)[:, None] * x - P @ y)
    env_y = 2 * (P.sum(0)[:, None] * y - P.T @ x)
    assert np.abs(gx - env_x).max() < 1e-8 and np.abs(gy - env_y).max() < 1e-8


# ------------------------------------------------------------------ eps-decay (NEXT-1)
def test_eps_decay_is_a_chain_of_plain_sweeps():
    """R-25: with omega = 1 a sweep maps f to f (its g-update reads only f), so L sweeps with
    eps-decay equal T single plain sweeps at eps_l = eps 5 0.8^(l-1) chained through f0,
    followed by L - T plain sweeps at eps (the plain solver is pinned above)."""
    from oracle import oracle as O
    p = gen.c1(n=50, seed=6)
    L = 14
    r = O.sinkhorn(p.x, p.y, p.eps, tol=0, max_iter=L, eps_decay=(5.0, 0.8))
    f = None
    T = 0
    while p.eps * 5.0 * 0.8 ** T > p.eps:
        f = O.sinkhorn(p.x, p.y, p.eps * 5.0 * 0.8 ** T, tol=0, max_iter=1, f0=f).f
        T += 1
    assert T == 8
    q = O.sinkhorn(p.x, p.y, p.eps, tol=0, max_iter=L - T, f0=f)
    assert np.abs(r.f - q.f).max() < 1e-12 and np.abs(r.g - q.g).max() < 1e-12 and abs(r.E - q.E) < 1e-12


def test_eps_decay_same_optimum_and_off_switch():
    from oracle import oracle as O
    p = gen.c1(n=40, seed=7, eps_factor=0.1)
    ref = O.sinkhorn(p.x, p.y, p.eps, tol=1e-11, max_iter=100000)
    r = O.sinkhorn(p.x, p.y, p.eps, tol=1e-11, max_iter=100000, eps_decay=(5.0, 0.8))
    assert r.converged
    assert np.abs((r.f - r.f.mean()) - (ref.f - ref.f.mean())).max() < 1e-8
    off = O.sinkhorn(p.x, p.y, p.eps, tol=1e-3, eps_decay=(1.0, 0.8))   # init <= 1: no decay sweep
    plain = O.sinkhorn(p.x, p.y, p.eps, tol=1e-3)
    assert off.iterations == plain.iterations and np.array_equal(off.f, plain.f)


# -------------------------------------------- general 1D NW + Alg. 3/4 (NEXT-2, R-26)
def test_nw1d_reduces_to_dualsort_when_n_equals_m():
    """Uniform n = m: the NW plan is the sorted identity (n one-edge trees) and Alg. 3 in reading
    R-26 is DualSort's Jacobi iteration from f = 0 (Alg. 2, R-5/R-7, pinned above): the same
    fixed point."""
    from oracle import oracle as O
    rng = np.random.default_rng(41)
    for n in (1, 2, 7, 40):
        x, y = rng.random(n).astype(np.float32), rng.random(n).astype(np.float32)
        assert np.abs(O.init_nw1d(x, y) - O.init_sort1d(x, y)).max() < 1e-12


@pytest.mark.parametrize("n,m,weights", [(3, 5, False), (6, 4, True), (5, 5, True), (4, 6, False), (2, 6, True),
                                          (6, 6, False), (4, 2, False)])
def test_nw1d_dual_is_lp_optimal(n, m, weights):
    """The eps = 0 dual of the general 1D problem: feasible (f_i + g_j <= c_ij), tight on the NW
    support, and <f, a> + <g, b> equals the optimal value of the transport LP solved by brute
    force (scipy linprog) — strong duality."""
    from oracle import oracle as O
    from scipy.optimize import linprog
    rng = np.random.default_rng(n * 10 + m)
    x, y = rng.random(n).astype(np.float32), rng.random(m).astype(np.float32)
    a = gen.random_weights(n, rng) if weights else np.full(n, 1.0 / n, np.float32)
    b = gen.random_weights(m, rng) if weights else np.full(m, 1.0 / m, np.float32)
    px, py = np.argsort(x, kind="stable"), np.argsort(y, kind="stable")
    xs, ys = x[px].astype(np.float64), y[py].astype(np.float64)
    C = (xs[:, None] - ys[None, :]) ** 2
    edges, tree = O.nw_corner_support(a[px] if weights else np.ones(n), b[py] if weights else np.ones(m),
                                      uniform=not weights)
    f, g, _ = O.dual_from_primal(C, edges, tree)
    assert (f[:, None] + g[None, :] - C).max() <= 1e-12
    for (i, j) in edges:
        assert abs(f[i] + g[j] - C[i, j]) <= 1e-12
    A_eq = np.zeros((n + m, n * m))
    for i in range(n):
        A_eq[i, i * m:(i + 1) * m] = 1
    for j in range(m):
        A_eq[n + j, j::m] = 1
    aa, bb = a[px].astype(np.float64), b[py].astype(np.float64)
    bb = bb * aa.sum() / bb.sum()
    lp = linprog(C.ravel(), A_eq=A_eq, b_eq=np.concatenate([aa, bb]), bounds=(0, None), method="highs")
    # g on every sink (the c-transform also covers sinks a tree never reached: none for NW)
    assert abs(f @ aa + g @ bb - lp.fun) < 1e-9


# ------------------------------------------------- Anderson acceleration (NEXT-1, R-27)
def test_anderson_memory_one_is_plain_sinkhorn():
    """mem = 1 keeps no second residual, so f^{l+1} = T(f^l): sweep L returns (f^{L-1},
    g_sk(f^{L-1})), i.e. the plain solver's f after L - 1 sweeps and its g after L."""
    from oracle import oracle as O
    p = gen.c1(n=60, seed=8)
    f0 = np.linspace(-0.1, 0.1, 60)
    for L in (1, 2, 7):
        r = O.sinkhorn_anderson(p.x, p.y, p.eps, mem=1, tol=0, max_iter=L, f0=f0)
        q = O.sinkhorn(p.x, p.y, p.eps, tol=0, max_iter=L, f0=f0)
        fq = f0 if L == 1 else O.sinkhorn(p.x, p.y, p.eps, tol=0, max_iter=L - 1, f0=f0).f
        assert np.abs(r.g - q.g).max() < 1e-12 and np.abs(r.f - fq).max() < 1e-12 and r.iterations == L


def test_anderson_mixing_step_is_the_constrained_least_squares_combination():
    """One mixing step checked against an independent solution of min |sum_u alpha_u r_u|^2 +
    lam |alpha|^2 s.t. sum alpha = 1 (alpha_0 = 1 - sum gamma, unconstrained lstsq in gamma on
    the stacked system [R; sqrt(lam) I]; the oracle solves the normal equations), with the map
    T(f) = f_sk(g_sk(f)) taken from single plain sweeps (R-27)."""
    from oracle import oracle as O
    p = gen.c1(n=50, seed=9)
    T = lambda f: O.sinkhorn(p.x, p.y, p.eps, tol=0, max_iter=1, f0=f)
    f0 = np.zeros(50)
    for mem, L in ((3, 4), (5, 4), (2, 5)):
        fs, Fs = [f0], []
        for l in range(L - 1):            # sweeps 1..L-1 each mix; sweep L returns (f^{L-1}, g~)
            Fs.append(T(fs[-1]).f)
            Rk = [Fs[u] - fs[u] for u in range(len(Fs))][-mem:]
            Fk = Fs[-mem:]
            if len(Rk) < 2:
                fs.append(Fk[-1])
                continue
            # the Tikhonov term lam |alpha|^2 (lam = 1e-8 tr(R^T R)/cnt) as extra rows sqrt(lam) I
            k = len(Rk)
            lam = 1e-8 * sum(float(r @ r) for r in Rk) / k
            Ra = np.concatenate([np.stack(Rk, 1), np.sqrt(lam) * np.eye(k)], 0)
            R0, D = Ra[:, 0], Ra[:, 1:] - Ra[:, :1]
            gam = np.linalg.lstsq(D, -R0, rcond=None)[0]
            alpha = np.concatenate([[1 - gam.sum()], gam])
            fs.append(sum(al * F for al, F in zip(alpha, Fk)))
        r = O.sinkhorn_anderson(p.x, p.y, p.eps, mem=mem, tol=0, max_iter=L, f0=f0)
        scale = np.abs(fs[-1]).max()
        assert np.abs(r.f - fs[-1]).max() < 1e-9 * scale, (mem, L)
        assert np.abs(r.g - T(fs[-1]).g).max() < 1e-9 * scale


def test_anderson_reaches_the_sinkhorn_optimum_with_explicit_error():
    """Anderson's fixed points are T's: the converged pair is the plain optimum (centred), its
    err is the explicit plan error (columns exact), and on C1 it needs fewer sweeps."""
    from oracle import oracle as O
    p = gen.c1(n=40, seed=10, eps_factor=0.1)
    ref = O.sinkhorn(p.x, p.y, p.eps, tol=1e-11, max_iter=100000)
    r = O.sinkhorn_anderson(p.x, p.y, p.eps, mem=5, tol=1e-11, max_iter=100000)
    assert r.converged and r.err < 1e-11
    fr = ref.f - ref.f.mean()
    assert np.abs((r.f - r.f.mean()) - fr).max() < 1e-8 * max(1.0, np.abs(fr).max())
    assert abs(r.E - ref.E) < 1e-10 * max(1.0, abs(ref.E))
    s = O.sinkhorn_anderson(p.x, p.y, p.eps, mem=4, tol=0, max_iter=6)
    x, y = p.x.astype(np.float64), p.y.astype(np.float64)
    C = ((x[:, None, :] - y[None, :, :]) ** 2).sum(-1)
    P = np.exp((s.f[:, None] + s.g[None, :] - C) / p.eps)
    n, m = C.shape
    assert np.abs(P.sum(0) - 1 / m).max() < 1e-13   # g = g_sk(f): exact columns
    err = np.abs(P.sum(1) - 1 / n).sum()
    assert abs(s.err - err) < 1e-12 * max(1.0, err) and err > 1e-6
    q = gen.c1()
    assert O.sinkhorn_anderson(q.x, q.y, q.eps, mem=5).iterations < O.sinkhorn(q.x, q.y, q.eps).iterations / 3
