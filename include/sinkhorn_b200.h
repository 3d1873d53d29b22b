/*
 * sinkhorn_b200.h — C ABI of the B200-native (sm_100a) hot path of
 *   J. Thornton, M. Cuturi, "Rethinking Initialization of the Sinkhorn Algorithm"
 *   (arXiv 2206.07630).  "P:n" cites PAPER.md line n; "R-k" cites reading k of
 *   DESIGN.md (where the paper is silent, garbled or inconsistent).
 *
 * Problem: discrete measures mu = sum_i a_i delta_{x_i} (n points),
 * nu = sum_j b_j delta_{y_j} (m points) in R^d, squared-L2 cost
 * C_ij = ||x_i - y_j||^2, regularisation eps > 0.  The library computes
 * the dual potentials (f, g) maximising Eq. (2) with the log-domain
 * Sinkhorn iteration of Alg. 1 (omega = 1; sign reading R-1, g-then-f
 * order R-2):
 *     g_j <- eps log b_j - eps LSE_i((f_i - C_ij)/eps)
 *     f_i <- eps log a_i - eps LSE_j((g_j - C_ij)/eps)
 * stopping when the L1 marginal error of p_ij = exp((f_i+g_j-C_ij)/eps)
 * (threshold appendix) drops below tol, checked every check_every
 * sweeps; plus the paper's initializers f^(0) (Sec. 3).
 *
 * CONVENTIONS (every entry point)
 *  - Arrays are row-major fp32 (points: [n][d]) or int32 (indices).  Unless an
 *    entry says otherwise, an array pointer may be DEVICE memory (e.g. a torch
 *    CUDA tensor's data_ptr) or HOST memory (pinned or pageable); host arrays are
 *    staged through the context workspace with copies on the context stream.
 *  - The caller owns every array.  The library owns only the opaque context:
 *    its stream binding, lazily grown device workspace and optional NCCL
 *    communicator.  It never frees or retains caller memory.
 *  - All work is ordered on the context's CUDA stream.  Entries return after
 *    their work is enqueued, except where "blocks" is stated (the solvers block
 *    until their host report is filled).
 *  - Errors: a status code; sk_last_error() gives a message for the last
 *    failing call on that context.  SK_EINVAL for bad sizes/arguments or
 *    non-finite / non-positive inputs where positivity is required (zero weights
 *    are rejected: eps log a_i diverges).  Non-convergence is NOT an error
 *    (SK_OK with converged = 0).  SK_ENONFINITE when a potential becomes
 *    non-finite: f and g then hold the last finite iterate.
 *  - Determinism: identical inputs, configuration and world size give
 *    bit-identical outputs (fixed reduction orders, no float atomics).  The
 *    sharded solver is bit-identical across world sizes 1, 2, 4, 8.
 *  - Iteration semantics: iterations = number of full (g, f) sweeps L at return;
 *    (f, g) = (f^(L), g^(L)); marginal_error = err_L; dual_objective = E(f^(L), g^(L)).
 *    Initializer-internal iterations are reported separately, never added.
 */
#ifndef SINKHORN_B200_H
#define SINKHORN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sk_ctx sk_ctx;

typedef enum {
    SK_OK = 0,
    SK_EINVAL = 1,        /* invalid argument (sizes, eps, tol, weights, NaN/Inf inputs) */
    SK_ECUDA = 2,         /* CUDA runtime / launch error */
    SK_ENONFINITE = 3,    /* a potential became non-finite; last finite iterate returned */
    SK_ENCCL = 4,         /* NCCL missing or failed */
    SK_ENOMEM = 5,        /* device workspace allocation failed */
    SK_EUNSUPPORTED = 6   /* valid request outside this build's kernels (stated per entry) */
} sk_status;

typedef enum {
    SK_COST_AUTO = 0,     /* stored if 4*n*m bytes fit the workspace budget and n*m is large, else online */
    SK_COST_ONLINE = 1,   /* C_ij recomputed from the point clouds in every pass (never materialised) */
    SK_COST_STORED = 2    /* C materialised once in HBM (fp32, 4nm bytes), streamed every sweep */
} sk_cost_mode;

/* Host-side report of one solve (one entry per problem of a batch). */
typedef struct {
    int32_t iterations;     /* full sweeps L */
    int32_t converged;      /* 1 if err_L < tol at a check */
    float marginal_error;   /* err_L (threshold appendix) */
    double dual_objective;  /* E(f^L, g^L), Eq. (2) */
    double init_ms;         /* initializer time inside this call (0 if none) */
    double build_ms;        /* stored-cost build time (0 if online) */
    double solve_ms;        /* Sinkhorn iterations, device time on the context stream */
} sk_report;

/* Cumulative per-context counters (for the bench's roofline / launch count). */
typedef struct {
    int64_t kernel_launches;   /* every kernel this library launched on the context */
    int64_t lse_launches;      /* launches of the dominant LSE-pass / on-chip solver kernels */
    double lse_ms;             /* device time of those launches (CUDA events on the context stream;
                                  only accumulated while timing is enabled) */
    double lse_ex2;            /* algorithmic exp2 evaluations of those launches (2 per cost entry
                                  per sweep, counted from the iteration counts) */
    double lse_bytes;          /* algorithmic HBM bytes of those launches (stored mode: 4 per entry) */
    /* Per-launch timing of the dominant kernel alone (CUDA events recorded around each launch
       on the context stream while timing is enabled; launches that returned at entry because
       the solve had already stopped are excluded): */
    int64_t dom_launches;      /* launches of the dominant kernel that did work */
    double dom_ms;             /* sum of their durations */
    double dom_entries;        /* cost entries they processed (n*m per pass; the fused stored sweep
                                  processes 2 passes per launch) */
    double dom_bytes;          /* algorithmic HBM bytes they read (stored mode: 4 per entry read) */
} sk_counters;

/* ---------------------------------------------------------------- context -- */
/* Create a context bound to CUDA device `device` and stream `cuda_stream`
 * (a cudaStream_t; NULL = the legacy default stream).  *ctx receives the handle. */
sk_status sk_create(sk_ctx **ctx, int device, void *cuda_stream);
/* Rebind the context stream (e.g. to torch's current stream). */
sk_status sk_set_stream(sk_ctx *ctx, void *cuda_stream);
void sk_destroy(sk_ctx *ctx);
const char *sk_last_error(const sk_ctx *ctx);
const char *sk_status_string(int status);
int32_t sk_version(void);
/* Alg. 1's relaxation omega (read as in DESIGN.md R-1) for the following solves on
 * this context: every update becomes h <- (1 - omega) h_old + omega h_sinkhorn (omega > 1:
 * the over-relaxed "momentum" of P:73; omega = 1: plain Sinkhorn, the default).
 * With omega != 1 the row marginals are not exact after an f-update, so err_l adds the row
 * term sum_i a_i |expm1((f_i - fsk_i)/eps)| and E uses sum_ij P_ij (both exact, O(n)).
 * omega must lie in (0, 2) (SK_EINVAL otherwise); the sharded entries sum the row terms over
 * the ranks (one ncclAllReduce of 2 doubles per sweep). */
sk_status sk_set_relaxation(sk_ctx *ctx, float omega);
/* eps-decay ("gradually reducing the regularization term from 5 eps to eps by a factor
 * of 0.8"; R-25) for the following solves on this context: sweep l = 1, 2, ... uses
 * eps_l = max(eps, eps * init * rate^(l-1)) for both of its updates; the T sweeps with
 * eps_l > eps are not checked (the stop rule runs on sweeps l > T with (l - T) % check_every
 * == 0) and count in rep.iterations.  init <= 1 turns it off (the default); otherwise rate
 * must lie in (0, 1) (SK_EINVAL).  On the multi-kernel paths it needs omega = 1
 * (SK_EUNSUPPORTED otherwise) and max_iter > T; the sharded entries chain the T decay sweeps
 * the same way (each rank's rows through its own f). */
sk_status sk_set_eps_decay(sk_ctx *ctx, float init, float rate);
/* Anderson acceleration ("Anderson acceleration (And = 5)"; R-27) for
 * the following solves on this context: type-II Anderson with memory mem on the sweep map
 * T(f) = f_sk(g_sk(f)).  Sweep l evaluates g~ = g_sk(f^l) and T(f^l); err_l is the L1 error of
 * the pair (f^l, g~) (its columns are exact: err_l = sum_i a_i |expm1((f^l_i - T(f^l)_i)/eps)|),
 * checked when l % check_every == 0 and at l = max_iter; then f^{l+1} = sum_u alpha_u T(f_u)
 * over the last mem sweeps, alpha = argmin |R alpha|^2 + lam |alpha|^2 subject to
 * sum alpha = 1 (R = residuals T(f_u) - f_u, lam = 1e-8 tr(R^T R) / count, or 1 when all
 * residuals are 0).  The result is
 * (f^l, g~) of the last sweep and rep.iterations the sweeps evaluated.  mem in {0, 1}: off (the
 * default); mem in [2, 8]: on; otherwise SK_EINVAL.  Runs on every path (the on-chip solver
 * K13; the online FFMA / tensor-core / stored multi-kernel solvers via K19, the stored one
 * with separate row and column passes; the sharded entries sum the Gram dots and the error
 * over the ranks: one ncclAllReduce of 9 doubles per sweep); omega != 1 and eps-decay return
 * SK_EUNSUPPORTED. */
sk_status sk_set_anderson(sk_ctx *ctx, int32_t mem);
/* Adaptive momentum ("adaptive momentum", "adapt=10, meaning adaptation is
 * recomputed after 10 iterations"; R-31 after SPEC S:178) for the following
 * solves on this context, window T = adapt_iters: the solve starts plain (omega = 1); whenever a
 * window ends at sweep l = kT with k >= 2, the per-sweep contraction of the L1 marginal error
 * over the window, rho = (err_l / err_{l-T})^(1/T), sets omega = 2 / (1 + sqrt(max(0, 1 - rho)))
 * clipped to [1, 1.95], which Alg. 1's relaxed updates (as sk_set_relaxation) use from sweep
 * l + 2 on (the fused error of sweep l is known during sweep l + 1); a non-finite ratio keeps
 * omega.  err_l is evaluated at every window end whatever check_every is.  adapt_iters = 0: off
 * (the default); < 0: SK_EINVAL.  Runs on the on-chip solver (per problem) and the multi-kernel
 * solvers (omega lives on the device: no host round trip), sharded included (the row terms summed
 * over the ranks as for a fixed omega; the stored path runs its separate row / column passes);
 * a fixed omega != 1, Anderson and eps-decay return SK_EUNSUPPORTED with it. */
sk_status sk_set_adaptive_momentum(sk_ctx *ctx, int32_t adapt_iters);
/* The solver options currently set on this context (each output nullable, host): omega
 * (sk_set_relaxation), the eps-decay (init, rate) (init 0 = off), the Anderson memory (0 = off)
 * and the adaptive-momentum window (0 = off).  Lets a caller change an option for one solve and
 * restore the previous setting. */
sk_status sk_get_solver_options(const sk_ctx *ctx, float *omega, float *decay_init, float *decay_rate,
                                int32_t *anderson, int32_t *adapt_iters);
/* Diagnostics / tuning of kernel variants (DESIGN.md section 6 measures each): key = value for the
 * following calls on this context.  None changes what is computed beyond fp32 rounding; each
 * selects a kernel variant or a balance of the exponential between MUFU and the FMA pipe:
 *   "tc" 0|1 (1): tcgen05 cross term (K3) for d in [tc_min_d, 256], and for every d on large
 *       problems (max(n, m) > 16384) while "tc_small_d" is 1; 0 = FFMA kernel K2 everywhere;
 *   "tc_min_d" 1..65 (17), "tc_small_d" 0|1 (1): see "tc";
 *   "fused" 0|1 (1): stored mode's fused single-read sweep K5; 0 = separate row/column passes;
 *   "seeded" 0|1 (1): max-free (seeded) LSE passes from the second sweep on ("seed_from" >= 1 (1):
 *       the first seeded sweep, 0-based);
 *   "tc_margin" [0, 1000] (4): K3 seeded shift above the previous LSE, log2 units;
 *   "lse_margin" [0, 1000] (4): K2 seeded shift above the previous LSE, log2 units (a margin
 *       beyond ~100 forces every seeded point through its exact fallback / the column redo);
 *   "lse_emu8" 0..2 (1): K2 seeded (d <= 4) exponential pairs of 8 on the FMA pipe;
 *   "tc_emu" 0..6 (2): K3 exponential pairs of 8 on the FMA pipe;
 *   "tc_epi" 16|162 (16): K3 epilogue organisation (16 warps on every tile, or two tile groups of 8);
 *   "tc_pipe" 0|1 (0): K3 seeded epilogue with software-pipelined TMEM loads (tile groups only);
 *   "batched_shape" 0|1 (1): K13 512 threads x 2 points (1) or 1024 x 1 (0) for 512 < P <= 1024;
 *   "batched_cl" 0..2 (0): K13 one CTA (1) or a CTA pair (2) per problem (0: pair only for B = 1);
 *   "batched_park" >= 0 (12): K13 batches with more problems than resident CTAs run at most this
 *       many sweeps per turn, then park (state to the workspace) and re-queue with their predicted
 *       remaining sweeps as priority (bit-identical results; 0: one turn per problem, FIFO);
 *   "grid_solver" 0|1 (1): the subsample initializer's inner solve (plain Sinkhorn, d <= 4, both
 *       subsamples in every SM's shared memory, ns * ms > 2^18) in one grid-persistent launch
 *       (K20); 0 = the general solver (K13 / multi-kernel).
 * SK_EINVAL for an unknown key or a value out of range. */
sk_status sk_set_tuning(sk_ctx *ctx, const char *key, double value);
/* Enable (1) / disable (0) CUDA-event timing of the dominant kernels into sk_counters. */
sk_status sk_set_timing(sk_ctx *ctx, int32_t enable);
sk_status sk_get_counters(const sk_ctx *ctx, sk_counters *out /* host */);
sk_status sk_reset_counters(sk_ctx *ctx);

/* --------------------------------------------------------- multi-GPU (NCCL) -- */
/* Row sharding of x across `world` ranks (one process per GPU).  Rank 0 calls
 * sk_nccl_unique_id, the caller broadcasts the 128 bytes (e.g. with
 * torch.distributed), then every rank calls sk_comm_init.  NCCL is loaded at
 * run time (libnccl.so.2); SK_ENCCL if unavailable. */
sk_status sk_nccl_unique_id(sk_ctx *ctx, void *out_128B /* host */);
sk_status sk_comm_init(sk_ctx *ctx, const void *id_128B /* host */, int32_t rank, int32_t world);
/* Test hook: with enable = 1 a communicator of world size 1 (sk_comm_init(ctx, id, 0, 1)) takes
 * the NCCL branch of sinkhorn_solve_sharded (ncclAllGather of the block partials, the
 * ncclAllReduce sites of omega != 1 and Anderson) instead of the local shortcut, so the NCCL
 * data plane runs on a one-GPU box; results are bit-identical to world 1 without it. */
sk_status sk_set_force_nccl(sk_ctx *ctx, int32_t enable);
/* Row block owned by `rank` in the fixed global partition used by
 * sinkhorn_solve_sharded: rows [*row0, *row0 + *n_local) of n_total.  The
 * partition is a function of n_total only (SK_SHARD_BLOCKS blocks), which is what
 * makes the result independent of the world size. */
#define SK_SHARD_BLOCKS 8
sk_status sk_shard_rows(int64_t n_total, int32_t rank, int32_t world, int64_t *row0, int64_t *n_local);

/* ----------------------------------------------------------- initializers -- */
/* Batched stable sort / rank of B rows of n fp32 keys (the sorting permutations
 * sigma of P:110): perm[b][k] = index of the k-th smallest key of row b, ties by
 * index (stable), -0.0 == +0.0 (R-16); rank[b][perm[b][k]] = k.  perm or rank may
 * be NULL.  Bit-exact.  SK_EINVAL on NaN keys.  n <= 2^24 per row (n <= 8192: one CTA per row
 * in shared memory; longer rows: the bitonic network over a global key array, 8192-key segments
 * in shared memory). */
sk_status sinkhorn_sort1d_batched(sk_ctx *ctx, int64_t B, int64_t n, const float *x,
                                  int32_t *perm, int32_t *rank);

/* Implicit differentiation: the vector-Jacobian product of the
 * optimal potentials (f*, g*) = F(x, y, a, b) with a cotangent z = (zf, zg), for the cost
 * |x - y|^2.  With P_ij = exp((f_i + g_j - C_ij)/eps), r = P 1, c = P^T 1 and
 * M = [[diag(r), P], [P^T, diag(c)]] (= -eps J_H,(f,g), H = the gradient of Eq. (2))
 * gives J_F^T z = eps J_H,.^T w with w = M^+ z: w by conjugate gradients preconditioned with
 * diag(r, c), z first projected on e^perp, e = (1_n, -1_m) (the shift of (f, g): only
 * shift-invariant losses, sum zf = sum zg, are meaningful; the e component is dropped), until
 * |residual| <= cg_tol |z| (checked every 8 iterations, at most cg_max_iter); then
 *   grad_x_i = 2 sum_j P_ij (w_f,i + w_g,j)(x_i - y_j),  grad_y_j = 2 sum_i P_ij (w_f,i + w_g,j)(y_j - x_i),
 *   grad_a = eps w_f,  grad_b = eps w_g.
 * (f, g) must be (close to) optimal — normally sinkhorn_solve's output.  x: n x d, y: m x d,
 * f: n, g: m, zf: n, zg: m; outputs (each nullable): grad_x n x d, grad_y m x d, grad_a n,
 * grad_b m.  cg_iters / cg_relres (host, nullable): iterations and the final relative
 * residual.  d in [1, 256] (d > 64: 32-point CTAs with the coordinates in shared memory).
 * SK_EINVAL on bad sizes (d > 256), eps or cg_tol <= 0, non-finite inputs.  Blocks. */
sk_status sinkhorn_vjp(sk_ctx *ctx, int64_t n, int64_t m, int32_t d, const float *x, const float *y,
                       float eps, const float *f, const float *g, const float *zf, const float *zg,
                       float cg_tol, int32_t cg_max_iter, float *grad_x, float *grad_y, float *grad_a,
                       float *grad_b, int32_t *cg_iters, double *cg_relres);

/* GMM fitting for the GMM initializer (Sec. 3.3, "we fit first two K-component GMMs";
 * the paper fits on the CPU with sklearn): `iters` EM steps for a
 * full-covariance K-component mixture of x (n x d, row-major).  Start (R-23/R-28):
 * kmeans_iters = 0: weights 1/K, means x[init_idx[k]], covariances = biased covariance of x +
 * reg_covar I; kmeans_iters > 0 (sklearn's init_params="kmeans"): kmeans_iters Lloyd steps
 * from centers x[init_idx[k]] (nearest center in fp64, ties to the lowest k, an empty cluster
 * keeps its center), a final assignment, and the M-step of those one-hot responsibilities.  Each
 * M-step adds reg_covar I (as sklearn's reg_covar).  tol > 0 stops EM as sklearn's
 * GaussianMixture(tol) does: after the M-step of an iteration whose E-step log-likelihood moved by
 * less than tol (tol = 0: exactly `iters` steps).  fp64 state and sufficient statistics,
 * deterministic.  Outputs (caller-owned, device or host): weights K, means K x d, covs
 * K x d x d (fp32, the layout sinkhorn_init_gmm takes); loglik (host, nullable) = mean
 * log-likelihood of the returned parameters; n_iter (host, nullable) = EM steps run.
 * d in [1, 256]: d <= 32 runs the fused E-step (statistics in registers), d > 32 the tiled one
 * (responsibilities in workspace, the x x^T statistics by 64 x 64 tiles).
 * SK_EINVAL: bad sizes, d > 256, K > n, iters < 0, kmeans_iters < 0, tol < 0,
 * reg_covar < 0, non-finite x, init_idx not K distinct indices in [0, n); SK_EUNSUPPORTED:
 * K > 64; SK_ENONFINITE: a covariance lost positive definiteness.  Blocks. */
sk_status sinkhorn_fit_gmm(sk_ctx *ctx, int64_t n, int32_t d, const float *x, int32_t K,
                           const int32_t *init_idx, int32_t kmeans_iters, int32_t iters, float tol,
                           float reg_covar, float *weights, float *means, float *covs, double *loglik,
                           int32_t *n_iter);

/* Soft ranks and soft sort (Sec. 3.1) of B 1D problems with
 * cost (x - y)^2, from potentials (f, g) (normally the output of sinkhorn_solve): with the
 * plan P_ij = exp((f_i + g_j - (x_i - y_j)^2)/eps) of Eq. (2),
 *     rank_i = sum_j P_ij z_j / sum_j P_ij,      sort_j = sum_i P_ij x_i / sum_i P_ij
 * (R-22: conditional means under the plan, which equal the paper's n P z and
 * n P^T x whenever P has the uniform marginals).  x: B x n; y: m values (y_shared = 1) or
 * B x m; f: B x n, g: B x m; z: m (nullable: z_j = j + 1, 1-based ranks); rank: B x n,
 * sort: B x m (either nullable).  One K15 pass (two sweeps of the other side per output, max
 * first, so no overflow for any finite (f, g); problems whose 2n + 3m floats exceed 200 KiB read
 * the other side from global memory).  SK_EINVAL on bad sizes, eps <= 0 or non-finite inputs;
 * SK_EUNSUPPORTED for n or m > 2^24 or B > 65535.
 * Asynchronous except for the input check. */
sk_status sinkhorn_soft_rank_sort(sk_ctx *ctx, int64_t B, int64_t n, int64_t m, const float *x,
                                  const float *y, int32_t y_shared, float eps, const float *f,
                                  const float *g, const float *z, float *rank, float *sort);

/* f^(0) = 0: writes B*n zeros to pot. */
sk_status sinkhorn_init_zero(sk_ctx *ctx, int64_t B, int64_t n, float *pot);

/* 1D initializer (Sec. 3.1; DualSort appendix) for d = 1,
 * n == m, uniform weights, cost (x - y)^2: sort x (sigma) and y (rho); the
 * sorted identity matching is optimal; f^(0)_{sigma(k)} = f~_k where f~ is
 * the eps = 0 dual of the sorted problem produced by Alg. 2 (R-5):
 *   dualsort_iters == 0: the fixed point of Alg. 2 from f = 0 (R-6, R-7),
 *     computed in O(n) by prefix/suffix scans;
 *   dualsort_iters == L > 0: exactly L vectorised (Jacobi) sweeps of Alg. 2,
 *     O(L n^2) (the paper's "3 iterations").
 * x: B x n; y: m values (y_shared = 1) or B x m.  pot: B x n (x side).  perm /
 * rank (nullable): the sort of x as in sinkhorn_sort1d_batched.  n <= 2^24 (the closed form;
 * n > 4096 keeps its scans in workspace), paper mode n <= 4096.
 * SK_EUNSUPPORTED if n != m (sinkhorn_init_nw1d takes any n, m) or beyond those sizes. */
sk_status sinkhorn_init_sort1d(sk_ctx *ctx, int64_t B, int64_t n, int64_t m, const float *x,
                               const float *y, int32_t y_shared, int32_t dualsort_iters,
                               float *pot, int32_t *perm, int32_t *rank);

/* General 1D initializer (Sec. 3.1 for any n, m and weights; Alg. 3/4,
 * P:429-455) for d = 1 and cost (x - y)^2: sort x (sigma) and y (rho); the
 * north-west corner plan of (a_sigma, b_rho) — a staircase whose cumulative-mass ties split it
 * into trees (exact ties: integers for uniform weights, fp64 cumulative sums of the fp32
 * weights otherwise); its eps = 0 dual by Alg. 3 in reading R-26 (every tree's root bounded by
 * the feasibility of all its sources, all trees from f = 0, Jacobi rounds, UpdateTree after
 * each) until f is unchanged or max_rounds rounds (0 = n + m + 2); f^(0)_{sigma(k)} = f~_k.
 * With n = m and uniform weights this is DualSort's fixed point (sinkhorn_init_sort1d is the
 * O(n) route for that case).  x: B x n; y: m (y_shared) or B x m; a: B x n, b like y
 * (nullable = uniform, positive); pot: B x n (x side); rounds: B (nullable).  n, m <= 2^20:
 * one CTA per problem, O(n m) per round (many-tree problems — uniform weights with n, m sharing
 * a large divisor — take many rounds); the arrays in shared memory up to ~4096 points, in a
 * global slot beyond.  SK_EINVAL: bad sizes, NaN, non-positive weights; SK_EUNSUPPORTED: too
 * large.  Blocks. */
sk_status sinkhorn_init_nw1d(sk_ctx *ctx, int64_t B, int64_t n, int64_t m, const float *x,
                             const float *y, int32_t y_shared, const float *a, const float *b,
                             int32_t max_rounds, float *pot, int32_t *rounds);

/* Gaussian initializer (Sec. 3.2): weighted means and biased
 * covariances (+ ridge_rel * tr/d * I, R-11) computed on device with fp64
 * accumulation; matrix square roots by fp64 coupled Newton-Schulz (R-12);
 * A = S_mu^{-1/2} (S_mu^{1/2} S_nu S_mu^{1/2})^{1/2} S_mu^{-1/2};
 * potential f*(x) = ||x||^2 - (x - m_mu)^T A (x - m_mu) - 2 m_nu^T x
 * (Gaussian-Potential appendix, R-4), evaluated on the smaller side
 * (n <= m: x, *side = 0; else y with roles swapped, *side = 1, R-15).
 * a, b nullable (uniform).  pot: n (side 0) or m (side 1).  d in [1, 256] (SK_EINVAL beyond);
 * d > 64 runs the square roots over the whole grid (one cooperative launch, matrices in L2). */
sk_status sinkhorn_init_gaussian(sk_ctx *ctx, int64_t n, int64_t m, int32_t d, const float *x,
                                 const float *a, const float *y, const float *b, float ridge_rel,
                                 float *pot, int32_t *side /* host */);

/* GMM initializer (Sec. 3.3): given mixtures rho (Kx components:
 * weights wx[Kx], means mux[Kx][d], covariances covx[Kx][d][d]) fitted to mu and
 * tau (Ky, wy, muy, covy) fitted to nu: C~_kl = ||m_k - m'_l||^2 + B^2(S_k, S'_l)
 * (Eq. 6) with fp64 Newton-Schulz square roots; the Kx x Ky entropic
 * problem at the same eps (R-13) is solved in fp64 with Anderson acceleration (memory 5,
 * DESIGN.md R-29; err = the row term of (f^l, g_sk(f^l))) to inner_tol (max inner_max_iter
 * sweeps; the binding's default 1e-9: ~100 sweeps at C3) -> f~; f^(0)(x) = sum_k f~_k p_k(x),
 * p_k the posterior responsibilities (Eq. 7), on the smaller side (*side as above).
 * Mixture parameters are inputs (sinkhorn_fit_gmm fits them).  K <= 64; d in [1, 256]
 * (SK_EINVAL beyond); d > 64 keeps each CTA's d x d matrices in global memory (L2). */
sk_status sinkhorn_init_gmm(sk_ctx *ctx, int64_t n, int64_t m, int32_t d, const float *x,
                            const float *y, int32_t Kx, const float *wx, const float *mux,
                            const float *covx, int32_t Ky, const float *wy, const float *muy,
                            const float *covy, float eps, float inner_tol, int32_t inner_max_iter,
                            float *pot, int32_t *side /* host */);

/* Subsample initializer (Sec. 3.4): w = x[idx_x] (ns points),
 * z = y[idx_y] (ms points), uniform weights; inner Sinkhorn at the same eps to
 * inner_tol (max inner_max_iter) -> g~ (one grid-persistent launch, K20, when it applies: see
 * sk_set_tuning "grid_solver"); then Eq. (8)
 *   f^(0)_i = -eps log (1/ms) sum_j exp((g~_j - c(x_i, z_j))/eps)
 * in one online LSE pass over all of x.  Indices must be distinct and in range.
 * *side as above (n > m: roles swapped).  inner (nullable, host): report of the
 * inner solve.  pot: n (side 0) or m (side 1).  d in [1, 256] (SK_EINVAL beyond). */
sk_status sinkhorn_init_subsample(sk_ctx *ctx, int64_t n, int64_t m, int32_t d, const float *x,
                                  const float *y, int64_t ns, const int32_t *idx_x, int64_t ms,
                                  const int32_t *idx_y, float eps, float inner_tol,
                                  int32_t inner_max_iter, float *pot, int32_t *side /* host */,
                                  sk_report *inner /* host, nullable */);

/* ----------------------------------------------------------------- solver -- */
/* Solve B independent problems (B >= 1) of equal sizes.
 *   x: B x n x d;  y: B x m x d, or m x d shared by all problems (y_shared = 1);
 *   a: B x n or NULL (uniform 1/n);  b: B x m (or m if y_shared) or NULL (uniform);
 *   eps > 0, tol > 0, max_iter >= 1, check_every >= 1;
 *   f_init: B x n or NULL, g_init: B x m or NULL — at most one non-NULL.
 *     With f_init (or neither) each sweep is g-update then f-update (R-2).  With
 *     g_init the transposed problem is solved (x<->y, a<->b, f<->g).
 *   f: B x n, g: B x m outputs;  rep: B host reports.
 * Kernels: problems with d <= 4 that fit one CTA's shared memory (n, m up to ~4096) run the
 * on-chip solver K13 (one CTA or CTA pair per problem, the whole iteration loop on chip,
 * per-problem convergence); larger problems run the multi-kernel path: online LSE passes with
 * the cost recomputed per pass (the tcgen05 cross term K3 for d in (16, 256] — d > 64 in K
 * chunks of 64 — and, on problems with max(n, m) > 16384, for every d; the FFMA cross term K2
 * otherwise and when the scaled coordinates leave the fp16 range; for d > 64 K2 keeps the output
 * point's coordinates in shared memory) or, with SK_COST_STORED
 * (or AUTO for 8 <= d < 32 when the 4nm bytes fit the device's free memory; AUTO falls back
 * to the online cost otherwise), the stored-cost sweep (K4 build, K5 fused
 * single-read sweep).  Blocks until the reports are filled.
 * SK_EINVAL for d < 1 or d > 256 (and the conventions above); SK_EUNSUPPORTED for
 * n, m >= 2^31. */
sk_status sinkhorn_solve(sk_ctx *ctx, int64_t B, int64_t n, int64_t m, int32_t d, const float *x,
                         const float *y, int32_t y_shared, const float *a, const float *b, float eps,
                         float tol, int32_t max_iter, int32_t check_every, sk_cost_mode mode,
                         const float *f_init, const float *g_init, float *f, float *g,
                         sk_report *rep /* host, B entries */);

/* Row-sharded solve of ONE problem across the communicator's ranks (8(e) of the
 * design): this rank owns rows [row0, row0 + n_local) as given by sk_shard_rows.
 * x_local, a_local (nullable), f_init_local (nullable), f_local: this rank's
 * rows; y, b (nullable), g: replicated (m).  Every sweep: local row pass (f),
 * local column partials (max, sum-exp), merged per fixed row block on the rank (8 B per column
 * per block), ncclAllGather of the block partials (SK_SHARD_BLOCKS / world blocks per rank),
 * identical block-order merge on every rank (g, error, stop flag).  From the second sweep the
 * column pass is seeded (max-free); if any column's seeded sum leaves [2^-100, 2^100] the
 * merge flags it and the column pass is redone exactly (one more allgather, enqueued every
 * sweep, a no-op otherwise).  The unsharded solver runs the same merge tree, so the results are
 * bit-identical to sinkhorn_solve's for plain Sinkhorn (omega = 1, no Anderson, online cost).
 * Requires sk_comm_init (world 1 works without it).  d as sinkhorn_solve.  Blocks. */
sk_status sinkhorn_solve_sharded(sk_ctx *ctx, int64_t n_total, int64_t row0, int64_t n_local,
                                 int64_t m, int32_t d, const float *x_local, const float *y,
                                 const float *a_local, const float *b, float eps, float tol,
                                 int32_t max_iter, int32_t check_every, sk_cost_mode mode,
                                 const float *f_init_local, float *f_local, float *g,
                                 sk_report *rep /* host */);

/* Test / diagnostic entry: the sharded algorithm of sinkhorn_solve_sharded for
 * `world` virtual ranks inside one process on one GPU.  Every sweep each virtual
 * rank computes the column partials of its sk_shard_rows row block into its own
 * slots (what ncclAllGather delivers on a real box), then the same rank-order merge
 * runs once.  Same partition, kernels and merge order, hence bit-identical to a
 * world-GPU run and to world = 1; it exercises the partial/merge math without
 * NCCL.  x, a, f_init, f: all n rows (global order).  Blocks. */
sk_status sinkhorn_solve_sharded_emulated(sk_ctx *ctx, int32_t world, int64_t n, int64_t m, int32_t d,
                                          const float *x, const float *y, const float *a,
                                          const float *b, float eps, float tol, int32_t max_iter,
                                          int32_t check_every, sk_cost_mode mode, const float *f_init,
                                          float *f, float *g, sk_report *rep /* host */);

/* Diagnostic: out[i][j] = <x_i, y_j> for 128 x d and 128 x d fp32 inputs (row-major;
 * out 128 x 128), computed by the tensor-core path of the LSE pass (K3: 3-product fp16
 * hi/lo split of power-of-two scaled operands, tcgen05.mma kind::f16, fp32 accumulators read
 * back from TMEM and unscaled exactly).  d in [1, 256].  For
 * testing the operand layout and the error compensation.  Blocks. */
sk_status sk_selftest_tc_dot(sk_ctx *ctx, int32_t d, const float *x, const float *y, float *out);

/* K14 microbenchmarks (roofline denominators measured on this device, CUDA events on the
 * context stream): kind 0 = MUFU.EX2 throughput (ex2/s); 1 = FP32 FMA throughput (FMA
 * lane-operations/s, packed FFMA2); 2 = streaming HBM read bandwidth (bytes/s, 4 GiB,
 * 128-bit non-allocating loads); 3 = tcgen05 kind::f16 MMA throughput (flop/s, the K3
 * kernel with its epilogue skipped); 4 = the same without reloading the B operand ring
 * (pure MMA issue rate); 5..8 = raw tcgen05.mma rate of one shape in flop per SM clock
 * (M = 128; 5: f16 N = 128, 6: f16 N = 256, 7: tf32 N = 128, 8: tf32 N = 256); 9, 10 = kinds
 * 3, 4 in flop per SM clock (cycles of the first CTA); 11 = the K3 kernel with its MMAs
 * skipped (epilogue-only rate); 12 = MMAs skipped and the epilogue only releasing the
 * buffers (operand stream and synchronisation rate); 13 = the epilogue's arithmetic without
 * MMAs or TMEM loads; 14 = the whole seeded K3 kernel (MMAs + TMEM loads + epilogue); 9..14 in
 * equivalent flop per SM clock; 100 + (shape | mode << 2) = the raw
 * probe with diagnostic mode bits (sk_tc.cu k_mb_mma).  *value (host)
 * receives the rate.  Blocks. */
sk_status sk_microbench(sk_ctx *ctx, int32_t kind, double *value);

#ifdef __cplusplus
}
#endif
#endif /* SINKHORN_B200_H */
