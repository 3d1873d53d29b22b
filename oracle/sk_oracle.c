/*
 * sk_oracle.c — fp64 CPU ORACLE for the Sinkhorn hot path of
 * Thornton & Cuturi, "Rethinking Initialization of the Sinkhorn Algorithm"
 * (arXiv 2206.07630; cited as PAPER.md line numbers "P:n").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with the CUDA path.
 *
 * Everything is plain fp64, written in the paper's order and notation:
 *   - cost c(x_i, y_j) = sum_k (x_ik - y_jk)^2, by direct differences (P:165,
 *     "c(x,y)=||x-y||_2^2"); never the expanded |x|^2+|y|^2-2<x,y> form;
 *   - soft-min  min_eps(S)_i = -eps log sum_j exp(-S_ij/eps), evaluated
 *     with a max shift and a serial, fixed-order sum;
 *   - Sinkhorn (Alg. 1, omega = 1) with the sign reading R-1 and the
 *     g-then-f order of reading R-2:
 *         g_j <- eps log b_j - eps LSE_i((f_i - C_ij)/eps)
 *         f_i <- eps log a_i - eps LSE_j((g_j - C_ij)/eps);
 *   - the stopping rule of the threshold appendix: the explicit L1
 *     marginal error of p_ij = exp((f_i + g_j - C_ij)/eps);
 *   - the dual objective Eq. (2) as the explicit triple sum;
 *   - a stable merge sort (ties by index) for the sorting permutation;
 *   - DualSort (Alg. 2) as Jacobi min-plus sweeps
 *     f_i <- min_j (c_ij - c_jj + f_j) (reading R-5), from f = 0;
 *   - the Subsample extrapolation Eq. (8).
 * OpenMP parallelises only the outer loop over independent rows/columns; every
 * inner reduction is serial in index order.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* Below this many cost entries a loop runs on one thread (OpenMP start-up
 * dominates); the arithmetic and its order are identical either way. */
#define PAR_MIN 16384

/* ------------------------------------------------------------------ cost -- */
/* A problem is either two point clouds (x: n x d, y: m x d, row-major) whose
 * cost is evaluated by direct differences, or an explicit n x m matrix C. */
typedef struct {
    int64_t n, m;
    int d;
    const double *x, *y; /* point clouds, or NULL */
    const double *C;     /* explicit cost, or NULL */
} ora_prob;

static double cost_ij(const ora_prob *p, int64_t i, int64_t j) {
    if (p->C) return p->C[i * p->m + j];
    const double *xi = p->x + i * p->d, *yj = p->y + j * p->d;
    double s = 0.0;
    for (int k = 0; k < p->d; ++k) {
        double t = xi[k] - yj[k];
        s += t * t;
    }
    return s;
}

int ora_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void ora_set_num_threads(int t) {
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
#else
    (void)t;
#endif
}

void ora_cost_matrix(int64_t n, int64_t m, int d, const double *x, const double *y, double *C) {
    ora_prob p = {n, m, d, x, y, NULL};
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < m; ++j) C[i * m + j] = cost_ij(&p, i, j);
}

/* ------------------------------------------------------------- soft-min -- */
/* min_eps over one row of S: -eps log sum_j exp(-S_j/eps), max-shifted. */
double ora_softmin(int64_t m, const double *S, double eps) {
    double mx = -INFINITY;
    for (int64_t j = 0; j < m; ++j) mx = fmax(mx, -S[j] / eps);
    double s = 0.0;
    for (int64_t j = 0; j < m; ++j) s += exp(-S[j] / eps - mx);
    return -eps * (mx + log(s));
}

/* f-update of Alg. 1 line 4 (reading R-1), for rows rows[0..cnt) (all if rows==NULL):
 *   f_i = eps log a_i - eps LSE_j((g_j - C_ij)/eps)  ==  eps log a_i + min_eps(C_i. - g)_i */
static void f_update(const ora_prob *p, const double *a, const double *g, double eps,
                     double *f, const int64_t *rows, int64_t cnt) {
    int64_t N = rows ? cnt : p->n;
#pragma omp parallel if (N * p->m > PAR_MIN)
    {
        double *S = (double *)malloc(sizeof(double) * (size_t)p->m);
#pragma omp for schedule(static)
        for (int64_t r = 0; r < N; ++r) {
            int64_t i = rows ? rows[r] : r;
            for (int64_t j = 0; j < p->m; ++j) S[j] = cost_ij(p, i, j) - g[j];
            double v = log(a[i]) * eps + ora_softmin(p->m, S, eps);
            if (rows) f[r] = v; else f[i] = v;
        }
        free(S);
    }
}

/* g-update of Alg. 1 line 5: g_j = eps log b_j - eps LSE_i((f_i - C_ij)/eps). */
static void g_update(const ora_prob *p, const double *b, const double *f, double eps,
                     double *g, const int64_t *cols, int64_t cnt) {
    int64_t M = cols ? cnt : p->m;
#pragma omp parallel if (M * p->n > PAR_MIN)
    {
        double *S = (double *)malloc(sizeof(double) * (size_t)p->n);
#pragma omp for schedule(static)
        for (int64_t c = 0; c < M; ++c) {
            int64_t j = cols ? cols[c] : c;
            for (int64_t i = 0; i < p->n; ++i) S[i] = cost_ij(p, i, j) - f[i];
            double v = log(b[j]) * eps + ora_softmin(p->n, S, eps);
            if (cols) g[c] = v; else g[j] = v;
        }
        free(S);
    }
}

/* ----------------------------------------------- error and dual objective -- */
/* Threshold appendix: p_ij = exp((f_i + g_j - c_ij)/eps),
 * err = sum_i |sum_j p_ij - a_i| + sum_j |sum_i p_ij - b_j|. */
static double marginal_error(const ora_prob *p, const double *a, const double *b,
                             const double *f, const double *g, double eps) {
    double *row = (double *)malloc(sizeof(double) * (size_t)p->n);
    double *col = (double *)malloc(sizeof(double) * (size_t)p->m);
#pragma omp parallel for schedule(static) if (p->n * p->m > PAR_MIN)
    for (int64_t i = 0; i < p->n; ++i) {
        double s = 0.0;
        for (int64_t j = 0; j < p->m; ++j) s += exp((f[i] + g[j] - cost_ij(p, i, j)) / eps);
        row[i] = s;
    }
#pragma omp parallel for schedule(static) if (p->n * p->m > PAR_MIN)
    for (int64_t j = 0; j < p->m; ++j) {
        double s = 0.0;
        for (int64_t i = 0; i < p->n; ++i) s += exp((f[i] + g[j] - cost_ij(p, i, j)) / eps);
        col[j] = s;
    }
    double err = 0.0;
    for (int64_t i = 0; i < p->n; ++i) err += fabs(row[i] - a[i]);
    for (int64_t j = 0; j < p->m; ++j) err += fabs(col[j] - b[j]);
    free(row);
    free(col);
    return err;
}

/* Eq. (2): E(f,g) = <f,a> + <g,b> - eps sum_ij exp(f_i/eps) K_ij exp(g_j/eps),
 * K = exp(-C/eps); the bilinear term is summed as sum_ij exp((f_i+g_j-C_ij)/eps). */
static double dual_objective(const ora_prob *p, const double *a, const double *b,
                             const double *f, const double *g, double eps) {
    double *row = (double *)malloc(sizeof(double) * (size_t)p->n);
#pragma omp parallel for schedule(static) if (p->n * p->m > PAR_MIN)
    for (int64_t i = 0; i < p->n; ++i) {
        double s = 0.0;
        for (int64_t j = 0; j < p->m; ++j) s += exp((f[i] + g[j] - cost_ij(p, i, j)) / eps);
        row[i] = s;
    }
    double fa = 0.0, gb = 0.0, mass = 0.0;
    for (int64_t i = 0; i < p->n; ++i) { fa += f[i] * a[i]; mass += row[i]; }
    for (int64_t j = 0; j < p->m; ++j) gb += g[j] * b[j];
    free(row);
    return fa + gb - eps * mass;
}

/* --------------------------------------------------------------- Sinkhorn -- */
/* Alg. 1 with relaxation omega, line by line in the R-1 reading:
 *   g <- g + omega (eps log b + min_eps(C^T - g (+) f)) = (1 - omega) g + omega g_sk(f)
 *   f <- f + omega (eps log a + min_eps(C - f (+) g))   = (1 - omega) f + omega f_sk(g)
 * (g_sk, f_sk: the omega = 1 updates above; omega > 1 is the over-relaxed "momentum" of
 * P:73).  omega == 1 is the plain algorithm. */
static double omega_g = 1.0;   /* the current call's omega (set by the public entry) */
/* eps-decay ("gradually reducing the regularization term from 5 eps to eps by a factor of
 * 0.8"; reading R-25): sweep l = 1, 2, ... uses eps_l = max(eps, eps * decay_init * decay_rate^(l-1))
 * for both of its updates; the T sweeps with eps_l > eps are not checked, the stop rule runs on
 * the sweeps l > T with (l - T) % check_every == 0.  decay_init = 0: off. */
static double decay_init_g = 0.0, decay_rate_g = 1.0;
/* Adaptive momentum ("adaptive momentum (adapt=10, meaning adaptation is recomputed after 10
 * iterations)"; reading R-31 after SPEC S:178): with window T = adapt_g > 0 the
 * solve starts plain (omega = 1); after sweep l = kT (k >= 2) the per-sweep contraction of the
 * explicit L1 error over the last window, rho = (err_l / err_{l-T})^(1/T), gives
 * omega = 2 / (1 + sqrt(max(0, 1 - rho))) clipped to [1, 1.95], used from sweep l + 2 on (the
 * fused error of sweep l is known during sweep l + 1).  A non-finite ratio keeps omega.
 * g0 (nullable) starts g (the relaxed g-update reads it); omega_out (nullable, max_iter entries)
 * receives the omega of every sweep. */
static int adapt_g = 0;
static const double *g0_g = NULL;
static double *omega_out_g = NULL;

static double adaptive_omega(double ratio, int T, double cur) {
    if (!isfinite(ratio) || ratio < 0.0) return cur;
    const double rho = pow(ratio, 1.0 / (double)T);
    double w = 2.0 / (1.0 + sqrt(fmax(0.0, 1.0 - rho)));
    if (!(w >= 1.0)) w = 1.0;
    if (w > 1.95) w = 1.95;
    return w;
}

static void relax(int64_t k, double *v, const double *vsk, double omega) {
    if (omega == 1.0) { for (int64_t i = 0; i < k; ++i) v[i] = vsk[i]; return; }
    for (int64_t i = 0; i < k; ++i) v[i] = (1.0 - omega) * v[i] + omega * vsk[i];
}

/* Alg. 1, g-then-f (reading R-2): start f = f0 (0 if NULL), g = 0.
 * For l = 1..max_iter: g-update, f-update; every check_every sweeps compute the
 * explicit error (threshold appendix) and stop when err < tol.  tol <= 0 runs
 * exactly max_iter sweeps ("lockstep").  On return: f, g = (f^(L), g^(L)),
 * *iters = L, *err = err_L (always evaluated at the returned iterate), *E = Eq. (2).
 * trace (nullable, max_iter entries) receives E after every sweep. */
static int sinkhorn(const ora_prob *p, const double *a, const double *b, double eps,
                    double tol, int max_iter, int check_every, const double *f0,
                    double *f, double *g, int *iters, double *err, double *E, double *trace) {
    for (int64_t i = 0; i < p->n; ++i) f[i] = f0 ? f0[i] : 0.0;
    for (int64_t j = 0; j < p->m; ++j) g[j] = g0_g ? g0_g[j] : 0.0;
    const int adapt = adapt_g;
    double omega = adapt ? 1.0 : omega_g, omega_sched = omega, err_win = 0.0;
    int sched_at = -1;
    double *gs = (double *)malloc(sizeof(double) * (size_t)p->m);
    double *fs = (double *)malloc(sizeof(double) * (size_t)p->n);
    int l = 0, converged = 0, T = 0;
    double e = INFINITY;
    while (l < max_iter) {
        ++l;
        if (l == sched_at) omega = omega_sched;
        if (omega_out_g) omega_out_g[l - 1] = omega;
        double el = eps;
        if (decay_init_g > 0.0) {
            const double v = eps * decay_init_g * pow(decay_rate_g, (double)(l - 1));
            if (v > eps) { el = v; T = l; }
        }
        g_update(p, b, f, el, gs, NULL, 0);
        relax(p->m, g, gs, omega);
        f_update(p, a, g, el, fs, NULL, 0);
        relax(p->n, f, fs, omega);
        if (trace) trace[l - 1] = dual_objective(p, a, b, f, g, eps);
        int have_e = 0;
        if (tol > 0.0 && l > T && (l - T) % check_every == 0) {
            e = marginal_error(p, a, b, f, g, eps);
            have_e = 1;
            if (e < tol) { converged = 1; break; }
        }
        if (adapt && l % adapt == 0) {   /* the end of a window: err_l against err_{l-T} */
            const double en = have_e ? e : marginal_error(p, a, b, f, g, eps);
            if (l >= 2 * adapt) { omega_sched = adaptive_omega(en / err_win, adapt, omega); sched_at = l + 2; }
            err_win = en;
        }
    }
    if (!converged) e = marginal_error(p, a, b, f, g, eps);
    free(gs);
    free(fs);
    *iters = l;
    *err = e;
    *E = dual_objective(p, a, b, f, g, eps);
    return converged;
}

/* Anderson acceleration (NEXT-1; "Anderson acceleration (And = 5)"; reading
 * R-27): type-II Anderson with memory mem on the sweep map T(f) = f_sk(g_sk(f)).  Sweep l:
 *   g~ = g_sk(f), f~ = T(f) = f_sk(g~);  the iterate's pair (f, g~) has exact columns, so
 *   err_l = the explicit L1 error of (f, g~) (its row term); stop if err_l < tol (checked when
 *   l % k == 0 and at l = max_iter);
 *   r = f~ - f; keep the last mem (f~, r); with >= 2 kept:
 *   alpha = argmin |R alpha|^2 + lam |alpha|^2 s.t. sum alpha = 1 (lam = 1e-8 tr(R^T R)/cnt, 1 if 0),
 *   i.e. alpha = x / sum x with (R^T R + lam I) x = 1;  f <- sum_i alpha_i f~_i (else f <- f~).
 * Returns (f, g~) of the last evaluated sweep. */
static int sinkhorn_anderson(const ora_prob *p, const double *a, const double *b, double eps, double tol,
                             int max_iter, int check_every, const double *f0, int mem, double *f, double *g,
                             int *iters, double *err, double *E) {
    const int64_t n = p->n, m = p->m;
    for (int64_t i = 0; i < n; ++i) f[i] = f0 ? f0[i] : 0.0;
    double *ft = (double *)malloc(sizeof(double) * (size_t)n);
    double *F = (double *)malloc(sizeof(double) * (size_t)n * mem);
    double *R = (double *)malloc(sizeof(double) * (size_t)n * mem);
    double G[16 * 16], x[16];
    int l = 0, converged = 0, cnt = 0, head = 0;
    double e = INFINITY;
    while (l < max_iter) {
        ++l;
        g_update(p, b, f, eps, g, NULL, 0);
        f_update(p, a, g, eps, ft, NULL, 0);
        if (tol > 0.0 && (l % check_every == 0 || l == max_iter)) {
            e = marginal_error(p, a, b, f, g, eps);
            if (e < tol) { converged = 1; break; }
        }
        if (l == max_iter) break;
        for (int64_t i = 0; i < n; ++i) { F[(int64_t)head * n + i] = ft[i]; R[(int64_t)head * n + i] = ft[i] - f[i]; }
        head = (head + 1) % mem;
        if (cnt < mem) ++cnt;
        if (cnt < 2) { for (int64_t i = 0; i < n; ++i) f[i] = ft[i]; continue; }
        double tr = 0.0;
        for (int u = 0; u < cnt; ++u)
            for (int v = 0; v < cnt; ++v) {
                double s = 0.0;
                for (int64_t i = 0; i < n; ++i) s += R[(int64_t)u * n + i] * R[(int64_t)v * n + i];
                G[u * cnt + v] = s;
                if (u == v) tr += s;
            }
        const double lam = tr > 0.0 ? 1e-8 * tr / cnt : 1.0;   /* (all residuals 0: equal weights) */
        for (int u = 0; u < cnt; ++u) { G[u * cnt + u] += lam; x[u] = 1.0; }
        for (int c = 0; c < cnt; ++c)        /* Gaussian elimination (SPD: no pivoting) */
            for (int r = c + 1; r < cnt; ++r) {
                const double q = G[r * cnt + c] / G[c * cnt + c];
                for (int k = c; k < cnt; ++k) G[r * cnt + k] -= q * G[c * cnt + k];
                x[r] -= q * x[c];
            }
        for (int r = cnt - 1; r >= 0; --r) {
            double s = x[r];
            for (int k = r + 1; k < cnt; ++k) s -= G[r * cnt + k] * x[k];
            x[r] = s / G[r * cnt + r];
        }
        double sx = 0.0;
        for (int u = 0; u < cnt; ++u) sx += x[u];
        /* degenerate least squares (R-30; SPEC "fall back to the plain update for that
         * step"): a non-finite or zero sum, or a non-finite weight -> f <- f~ this sweep */
        int degen = !isfinite(sx) || sx == 0.0;
        for (int u = 0; u < cnt; ++u) degen |= !isfinite(x[u] / sx);
        if (degen) { for (int64_t i = 0; i < n; ++i) f[i] = ft[i]; continue; }
        for (int64_t i = 0; i < n; ++i) {
            double v = 0.0;
            for (int u = 0; u < cnt; ++u) v += (x[u] / sx) * F[(int64_t)u * n + i];
            f[i] = v;
        }
    }
    if (!converged) e = marginal_error(p, a, b, f, g, eps);
    free(ft); free(F); free(R);
    *iters = l;
    *err = e;
    *E = dual_objective(p, a, b, f, g, eps);
    return converged;
}

int ora_sinkhorn_points_anderson(int64_t n, int64_t m, int d, const double *x, const double *y, const double *a,
                                 const double *b, double eps, int mem, double tol, int max_iter, int check_every,
                                 const double *f0, double *f, double *g, int *iters, double *err, double *E) {
    ora_prob p = {n, m, d, x, y, NULL};
    if (mem < 1 || mem > 16) return -1;
    return sinkhorn_anderson(&p, a, b, eps, tol, max_iter, check_every, f0, mem, f, g, iters, err, E);
}

/* Public entry points: point clouds (cost by direct differences) ... */
int ora_sinkhorn_points(int64_t n, int64_t m, int d, const double *x, const double *y,
                        const double *a, const double *b, double eps, double tol, int max_iter,
                        int check_every, const double *f0, double *f, double *g, int *iters,
                        double *err, double *E, double *trace) {
    ora_prob p = {n, m, d, x, y, NULL};
    return sinkhorn(&p, a, b, eps, tol, max_iter, check_every, f0, f, g, iters, err, E, trace);
}

/* Relaxed variant (omega > 0; Alg. 1's omega). */
int ora_sinkhorn_points_omega(int64_t n, int64_t m, int d, const double *x, const double *y,
                              const double *a, const double *b, double eps, double omega, double tol,
                              int max_iter, int check_every, const double *f0, double *f, double *g,
                              int *iters, double *err, double *E, double *trace) {
    ora_prob p = {n, m, d, x, y, NULL};
    omega_g = omega;
    int r = sinkhorn(&p, a, b, eps, tol, max_iter, check_every, f0, f, g, iters, err, E, trace);
    omega_g = 1.0;
    return r;
}

/* ... with adaptive momentum (R-31) and an optional starting g. */
int ora_sinkhorn_points_adaptive(int64_t n, int64_t m, int d, const double *x, const double *y,
                                 const double *a, const double *b, double eps, double omega, int adapt_iters,
                                 double tol, int max_iter, int check_every, const double *f0, const double *g0,
                                 double *f, double *g, int *iters, double *err, double *E, double *omega_out) {
    if (adapt_iters < 0) return -1;
    ora_prob p = {n, m, d, x, y, NULL};
    omega_g = omega;
    adapt_g = adapt_iters;
    g0_g = g0;
    omega_out_g = omega_out;
    int r = sinkhorn(&p, a, b, eps, tol, max_iter, check_every, f0, f, g, iters, err, E, NULL);
    omega_g = 1.0;
    adapt_g = 0;
    g0_g = NULL;
    omega_out_g = NULL;
    return r;
}

/* ... with eps-decay (R-25). */
int ora_sinkhorn_points_decay(int64_t n, int64_t m, int d, const double *x, const double *y,
                              const double *a, const double *b, double eps, double omega, double decay_init,
                              double decay_rate, double tol, int max_iter, int check_every, const double *f0,
                              double *f, double *g, int *iters, double *err, double *E, double *trace) {
    ora_prob p = {n, m, d, x, y, NULL};
    omega_g = omega;
    decay_init_g = decay_init;
    decay_rate_g = decay_rate;
    int r = sinkhorn(&p, a, b, eps, tol, max_iter, check_every, f0, f, g, iters, err, E, trace);
    omega_g = 1.0;
    decay_init_g = 0.0;
    decay_rate_g = 1.0;
    return r;
}

/* ... or an explicit cost matrix (GMM's K x K Bures cost). */
int ora_sinkhorn_matrix(int64_t n, int64_t m, const double *C, const double *a, const double *b,
                        double eps, double tol, int max_iter, int check_every, const double *f0,
                        double *f, double *g, int *iters, double *err, double *E, double *trace) {
    ora_prob p = {n, m, 0, NULL, NULL, C};
    return sinkhorn(&p, a, b, eps, tol, max_iter, check_every, f0, f, g, iters, err, E, trace);
}

int ora_sinkhorn_matrix_anderson(int64_t n, int64_t m, const double *C, const double *a, const double *b,
                                 double eps, int mem, double tol, int max_iter, int check_every, const double *f0,
                                 double *f, double *g, int *iters, double *err, double *E) {
    ora_prob p = {n, m, 0, NULL, NULL, C};
    if (mem < 1 || mem > 16) return -1;
    return sinkhorn_anderson(&p, a, b, eps, tol, max_iter, check_every, f0, mem, f, g, iters, err, E);
}

void ora_f_update_points(int64_t n, int64_t m, int d, const double *x, const double *y,
                         const double *a, const double *g, double eps, double *f,
                         const int64_t *rows, int64_t cnt) {
    ora_prob p = {n, m, d, x, y, NULL};
    f_update(&p, a, g, eps, f, rows, cnt);
}

void ora_g_update_points(int64_t n, int64_t m, int d, const double *x, const double *y,
                         const double *b, const double *f, double eps, double *g,
                         const int64_t *cols, int64_t cnt) {
    ora_prob p = {n, m, d, x, y, NULL};
    g_update(&p, b, f, eps, g, cols, cnt);
}

double ora_marginal_error_points(int64_t n, int64_t m, int d, const double *x, const double *y,
                                 const double *a, const double *b, const double *f,
                                 const double *g, double eps) {
    ora_prob p = {n, m, d, x, y, NULL};
    return marginal_error(&p, a, b, f, g, eps);
}

double ora_dual_objective_points(int64_t n, int64_t m, int d, const double *x, const double *y,
                                 const double *a, const double *b, const double *f,
                                 const double *g, double eps) {
    ora_prob p = {n, m, d, x, y, NULL};
    return dual_objective(&p, a, b, f, g, eps);
}

double ora_marginal_error_matrix(int64_t n, int64_t m, const double *C, const double *a,
                                 const double *b, const double *f, const double *g, double eps) {
    ora_prob p = {n, m, 0, NULL, NULL, C};
    return marginal_error(&p, a, b, f, g, eps);
}

double ora_dual_objective_matrix(int64_t n, int64_t m, const double *C, const double *a,
                                 const double *b, const double *f, const double *g, double eps) {
    ora_prob p = {n, m, 0, NULL, NULL, C};
    return dual_objective(&p, a, b, f, g, eps);
}

/* Row sums / column sums of p_ij (sampled), for marginal property checks. */
void ora_plan_row_sums(int64_t n, int64_t m, int d, const double *x, const double *y,
                       const double *f, const double *g, double eps, const int64_t *rows,
                       int64_t cnt, double *out) {
    ora_prob p = {n, m, d, x, y, NULL};
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < cnt; ++r) {
        int64_t i = rows[r];
        double s = 0.0;
        for (int64_t j = 0; j < m; ++j) s += exp((f[i] + g[j] - cost_ij(&p, i, j)) / eps);
        out[r] = s;
    }
}

void ora_plan_col_sums(int64_t n, int64_t m, int d, const double *x, const double *y,
                       const double *f, const double *g, double eps, const int64_t *cols,
                       int64_t cnt, double *out) {
    ora_prob p = {n, m, d, x, y, NULL};
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < cnt; ++c) {
        int64_t j = cols[c];
        double s = 0.0;
        for (int64_t i = 0; i < n; ++i) s += exp((f[i] + g[j] - cost_ij(&p, i, j)) / eps);
        out[c] = s;
    }
}

/* ------------------------------------------------------ Eq. (8) subsample -- */
/* f0_i = -eps log (1/ms) sum_j exp((gb_j - c(x_i, z_j))/eps),
 * evaluated with a max shift; z: ms x d subsample of y, gb: its inner potential. */
void ora_subsample_extrapolate(int64_t n, int64_t ms, int d, const double *x, const double *z,
                               const double *gb, double eps, double *f0, const int64_t *rows,
                               int64_t cnt) {
    ora_prob p = {n, ms, d, x, z, NULL};
    int64_t N = rows ? cnt : n;
#pragma omp parallel
    {
        double *v = (double *)malloc(sizeof(double) * (size_t)ms);
#pragma omp for schedule(static)
        for (int64_t r = 0; r < N; ++r) {
            int64_t i = rows ? rows[r] : r;
            double mx = -INFINITY;
            for (int64_t j = 0; j < ms; ++j) {
                v[j] = (gb[j] - cost_ij(&p, i, j)) / eps;
                mx = fmax(mx, v[j]);
            }
            double s = 0.0;
            for (int64_t j = 0; j < ms; ++j) s += exp(v[j] - mx);
            /* -eps log((1/ms) * exp(mx) * s) */
            f0[r] = -eps * (log(s) + mx - log((double)ms));
        }
        free(v);
    }
}

/* ---------------------------------------------------------------- sorting -- */
/* Stable ascending merge sort of indices by value (ties keep index order);
 * -0.0 compares equal to +0.0 (reading R-16).  Returns -1 on NaN. */
static int less_key(float a, float b) { return a < b; } /* -0.0 < +0.0 is false */

static void merge_sort(int32_t *idx, int32_t *tmp, const float *v, int64_t lo, int64_t hi) {
    if (hi - lo < 2) return;
    int64_t mid = lo + (hi - lo) / 2;
    merge_sort(idx, tmp, v, lo, mid);
    merge_sort(idx, tmp, v, mid, hi);
    int64_t i = lo, j = mid, k = lo;
    while (i < mid && j < hi) {
        /* take from the right run only if strictly smaller: stability */
        if (less_key(v[idx[j]], v[idx[i]])) tmp[k++] = idx[j++];
        else tmp[k++] = idx[i++];
    }
    while (i < mid) tmp[k++] = idx[i++];
    while (j < hi) tmp[k++] = idx[j++];
    memcpy(idx + lo, tmp + lo, sizeof(int32_t) * (size_t)(hi - lo));
}

/* perm[k] = index of the k-th smallest entry (sigma of P:110); rank[perm[k]] = k. */
int ora_sort_rank(int64_t B, int64_t n, const float *x, int32_t *perm, int32_t *rank) {
    for (int64_t t = 0; t < B * n; ++t)
        if (isnan(x[t])) return -1;
#pragma omp parallel
    {
        int32_t *tmp = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
#pragma omp for schedule(static)
        for (int64_t b = 0; b < B; ++b) {
            int32_t *pb = perm + b * n;
            for (int64_t k = 0; k < n; ++k) pb[k] = (int32_t)k;
            merge_sort(pb, tmp, x + b * n, 0, n);
            if (rank)
                for (int64_t k = 0; k < n; ++k) rank[b * n + pb[k]] = (int32_t)k;
        }
        free(tmp);
    }
    return 0;
}

/* --------------------------------------------------------------- DualSort -- */
/* Alg. 2 (appendix), vectorised (Jacobi) form, reading R-5:
 *   f_i <- min_j (c_ij - c_jj + f_j),   c_ij = (xs_i - ys_j)^2 on sorted supports,
 * from f = 0.  sweeps > 0: exactly that many sweeps (paper mode, "3 iterations",
 * P:245).  sweeps == 0: repeat until no entry changes (fixed point; reached in at
 * most n sweeps since there are no negative cycles, Lemma 1 / P:625-633).
 * Returns the number of sweeps performed. */
int ora_dualsort(int64_t n, const double *xs, const double *ys, int sweeps, double *f) {
    double *fn = (double *)malloc(sizeof(double) * (size_t)n);
    double *cjj = (double *)malloc(sizeof(double) * (size_t)n);
    for (int64_t j = 0; j < n; ++j) { f[j] = 0.0; cjj[j] = (xs[j] - ys[j]) * (xs[j] - ys[j]); }
    int s = 0;
    for (;;) {
        if (sweeps > 0 && s >= sweeps) break;
        if (sweeps == 0 && s > n + 1) break; /* cannot happen without negative cycles */
        int changed = 0;
#pragma omp parallel for schedule(static) reduction(| : changed)
        for (int64_t i = 0; i < n; ++i) {
            double best = INFINITY;
            for (int64_t j = 0; j < n; ++j) {
                double c = (xs[i] - ys[j]) * (xs[i] - ys[j]);
                double v = c - cjj[j] + f[j];
                if (v < best) best = v;
            }
            fn[i] = best;
            changed |= (best != f[i]);
        }
        memcpy(f, fn, sizeof(double) * (size_t)n);
        ++s;
        if (sweeps == 0 && !changed) break;
    }
    free(fn);
    free(cjj);
    return s;
}
