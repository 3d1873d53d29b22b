// sk_internal.h — host-side declarations shared by the .cu translation units.
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

namespace sk {

// ------------------------------------------------------------ K13 on-chip
struct BatchLaunch {
    int B, n, m, d;
    int *queue;       // device int (dynamic problem queue)
    const float *x; long long x_stride;
    const float *y; long long y_stride;
    const float *a; long long a_stride;
    const float *b; long long b_stride;
    const float *finit;
    float *f, *g;
    float eps, tol;
    int max_iter, check_every;
    int *iters, *conv, *nonfinite;
    float *err;
    double *E;
    float omega = 1.f;   // Alg. 1's relaxation
    float decay_init = 0.f, decay_rate = 1.f;   // eps-decay (R-25; decay_init <= 0: off)
    int anderson = 0;    // Anderson memory (R-27; < 2: off)
    int shape = 1;       // sk_set_tuning "batched_shape" (512 x 2 points for 512 < P <= 1024)
    int cl = 0;          // sk_set_tuning "batched_cl": 0 auto, 1 one CTA, 2 CTA pair per problem
    int adapt = 0;       // adaptive momentum window T (R-31; 0: off)
    // park / resume scheduling of batches (sweeps per turn; 0: off) and its workspace:
    // pq park_queue_ints(B) ints, pseed [B][n + m] float, phdr [B][8] double, done [1] int
    int park = 0;
    int *pq = nullptr;
    float *pseed = nullptr;
    double *phdr = nullptr;
    int *done = nullptr;
};
// Adaptive momentum (R-31): from the error ratio err_l / err_{l-T} of one window,
// rho = ratio^(1/T) and omega = 2 / (1 + sqrt(max(0, 1 - rho))) clipped to [1, 1.95]; a
// non-finite or negative ratio keeps the current omega.
__host__ __device__ inline float adaptive_omega(double ratio, int T, float cur) {
    if (!(ratio >= 0.0) || ratio > 1e300) return cur;
    const double rho = pow(ratio, 1.0 / (double)T);
    double w = 2.0 / (1.0 + sqrt(fmax(0.0, 1.0 - rho)));
    if (!(w >= 1.0)) w = 1.0;
    if (w > 1.95) w = 1.95;
    return (float)w;
}
bool batched_supported(int d, int n, int m, int mem = 0);
size_t park_queue_ints(int B);
// K18 general 1D initializer (NW corner + Alg. 3/4, R-26) on sorted supports
size_t nw1d_smem_bytes(int n, int m);
cudaError_t launch_nw1d(const float *xs, const int *xperm, const float *ys, const int *yperm, int y_shared,
                        const float *a, const float *b, int B, int n, int m, int max_rounds, float *pot, int *rounds,
                        cudaStream_t st, char *gscr = nullptr);
size_t nw1d_slot_bytes(int n, int m);   // per-problem global slot beyond shared memory
// K16 GMM fitting by EM (NEXT-3); state and partial workspace sizes in doubles
size_t em_state_doubles(int K, int d);
size_t em_partial_doubles(int K, int d);
size_t em_work_doubles(int K, int d);   // partials + the reduced statistics (launch_gmm_fit's part)
size_t em_wide_doubles(long long n, int K, int d);   // d > 32: responsibilities [n][K] + Cholesky scratch
cudaError_t launch_gmm_fit(const float *x, long long n, int d, int K, const int *idx, const double *cov0,
                           int kmeans_iters, int iters, double tol, double reg,
                           double *state /* 2 x em_state_doubles */, double *part,
                           int *flags /* [3]: non-PD, converged, EM steps */, float *w, float *mu, float *cov,
                           double *ll_out, int *h_conv /* pinned host int, nullable: convergence polls */,
                           cudaStream_t st, double *wide = nullptr /* d > 32: em_wide_doubles */);
// K17 implicit differentiation (NEXT-4)
size_t vjp_work_doubles(long long n, long long m, int d);
cudaError_t launch_vjp(long long n, long long m, int d, const float *x, const float *y, float eps, const float *f,
                       const float *g, const float *zf, const float *zg, double tol, int max_iter, double *work,
                       float *gx, float *gy, float *ga, float *gb, int *iters, double *relres, cudaStream_t st);
// K15 soft ranks / soft sort of B 1D problems from their potentials (NEXT-2)
size_t soft_rank_sort_smem(int n, int m);
cudaError_t launch_soft_rank_sort(long long B, int n, int m, const float *x, const float *y, long long ys,
                                  const float *f, const float *g, const float *z, float eps, float *rank,
                                  float *sort, cudaStream_t st);
size_t batched_smem_bytes(int D, int n, int m, int mem = 0);
cudaError_t launch_batched(const BatchLaunch &L, cudaStream_t st);

// ------------------------------------------------ K20: grid-persistent medium solver
// One problem (online cost, d <= 4, both clouds in every CTA's shared memory), plain Sinkhorn
// (omega = 1), solved in one cooperative launch (sk_grid.cu).  Used for the subsample
// initializer's inner solve.
struct GridResult {
    double E;
    int iterations, converged, nonfinite;
    float err;
};
struct GridLaunch {
    int n, m, d;
    const float *x, *y, *a, *b, *finit;   // device; a, b, finit nullable
    float eps, tol;
    int max_iter, check_every;
    float *f, *g;                         // device outputs
    void *work;                           // grid_solver_workspace_bytes(n, m, #SMs)
    GridResult *res_host;                 // pinned host result (copied on the stream), nullable
};
bool grid_solver_supported(int d, int n, int m);
size_t grid_solver_smem(int d, int n, int m);
size_t grid_solver_workspace_bytes(int n, int m, int nsm);
cudaError_t launch_grid_solver(const GridLaunch &L, cudaStream_t st);

// ------------------------------------------------- multi-kernel online path
// Device status of one solve (all fields written only by kernels' last blocks).
struct DevStatus {
    int iter;        // completed sweeps l: (f^l, g^l) live in buffers [l & 1]
    int stop;        // kernels return immediately once set
    int converged;
    int nonfinite;
    int final_iter;
    float err;       // last computed err_l
    unsigned ticket_col, ticket_row, ticket_rep;
    int max_iter, check_every;
    float tol;
    double E;        // dual objective of the returned iterate
    double fa_local; // sharded: this rank's <f,a> - eps sum(a) partial
    int colfail;     // stored fused sweep: some column sum left the scaled range -> exact column pass
    double row_err;  // relaxed (omega != 1): sum_i a_i |expm1((f_i - fsk_i)/eps)| of the last row merge
    double mass_dev; //                        sum_ij P_ij - sum_i a_i = sum_i a_i expm1((f_i - fsk_i)/eps)
    int g_off;       // Anderson (R-27): the returned g is g_sk(f^L), in buffer [(L + 1) & 1]
    float omega;     // the relaxation of the current sweep (adaptive momentum, R-31, changes it)
    float omega_next;//   set by the column merge at the end of a window, applied by the row merge
    float err_win;   //   err at the end of the previous window
};

// Packed tile layout of one side: tiles of tq points; tile t at t*(D+1)*tq floats:
// [D][tq] coordinates then [tq] w = (h - |p|^2) log2(e)/eps; padding w = -inf.
int lse_dpad(int d);          // instantiated D >= d (0 if unsupported)
int lse_tq(int D);            // points per tile for D
__host__ __device__ inline long long lse_tiles(long long P, int tq) { return (P + tq - 1) / tq; }

struct Side {
    int P, d, D, tq;
    float *pack;      // tiles * (D+1) * tq
    float *c;         // [P] eps log w_p + |p|^2 (finalize constant)
    float *nk;        // [P] |p|^2 log2(e)/eps
    float *pot[2];    // double-buffered potential
    float *lse;       // [P] last merged LSE (log2 units): the seed of the next pass (nullable)
    const float *raw = nullptr;  // PACK_TC: the caller's P x d fp32 coordinates (exact fallback of a seeded pass)
    unsigned char *tcimg = nullptr;  // PACK_TC: the side's K3 images (K6 rewrites w and the shift)
    float tc_c = 16.f;               //          c of the extra columns
    int tc_rb = 128;                 //          image row bytes (32: the compact d <= 16 layout)
};

// Pack points (P x d, fp32 row-major), optional weights and initial potential.
// If wts == nullptr the log-weight is the constant logw_const.  mode: PACK_ONLINE (coords
// in the tiles, |p|^2 folded), PACK_STORED (D = 0, no |p|^2: the cost is stored), PACK_TC
// (D = 0, |p|^2 folded, coordinates live in the tensor-core images).
enum PackMode { PACK_ONLINE = 0, PACK_STORED = 1, PACK_TC = 2 };
cudaError_t pack_side(const Side &S, const float *pts, const float *wts, float logw_const,
                      const float *pot0, float eps, cudaStream_t st, int mode = -1);

// ------------------------------------------------------- K3 tensor-core pass
// Per side one image allocation (layout in sk_common.cuh): fp16 hi/lo of alpha x (K-major
// SW128, K padded to 64, tiles of 128 points padded to 256) plus the extra-column images EA/EB
// (w and the row shift folded into the MMA) and the exact shifts.  The x side is scaled by 2^s,
// the y side by (2 log2(e)/eps) 2^-s (s from both sides' max |coordinate|, amax2 = [x, y] as
// device uint float bits), so the accumulator is the log2-domain exponent minus the row shift.
struct TcPass {
    const void *Aimg, *Bimg;    // images of the output side (A, P points) and the reduced side (B)
    int P;  long long Q;
    int ksteps;                 // ceil(d / 16): K = 16 MMA steps
    int nblk, blk_tiles, split_q;   // Q split structure in tiles of 256 points
    float2 *part;
    float eps;
    const int *stop;
    float *debug_acc = nullptr;
    int mma_only = 0;
    long long *cyc = nullptr;   // K14: SM cycles of CTA 0
    int seeded = 0;             // the output side's shifts were folded by K6 (max-free pass)
    const int *only_if = nullptr;   // run only if *only_if != 0 (the exact redo of a seeded column pass)
    int emu = 2;                // exponential pairs (of every 8) on the FMA pipe (sk_set_tuning "tc_emu")
    int epi = 16;               // epilogue organisation (sk_set_tuning "tc_epi": 16 or 162)
    int pipe = 0;               // seeded epilogue with software-pipelined TMEM loads (sk_set_tuning "tc_pipe")
    int rb = 128;               // image row bytes of both sides (32: compact K = 16 images, ksteps == 1)
};
size_t tc_image_bytes(long long P, int rb = 128);
// image row bytes for d: 32 (compact K = 16, d <= 16), 128 (K = 64), 128 KC (KC chunks of K = 64,
// d in (64, 256])
inline int tc_row_bytes(int d) {
    const int ks = (d + 15) / 16;
    return ks == 1 ? 32 : 128 * ((ks + 3) / 4);
}
cudaError_t launch_absmax(const float *pts, long long cnt, unsigned *out, cudaStream_t st);  // out zeroed first
cudaError_t launch_pack_tc(const float *pts, long long P, int d, const unsigned *amax2, int role, float eps,
                           void *img, cudaStream_t st, int rb = 128);   // role 0: x side, 1: y side
cudaError_t launch_pack_tc_ext(long long P, const float *w, void *img, cudaStream_t st,
                               int rb = 128);  // w: plain [P] (nullable = 0)
bool tc_fold_ok(float amax_x, float amax_y, float eps);   // both scaled sides within fp16 range
float tc_fold_c();                                         // c of the extra columns
cudaError_t launch_lse_tc(const TcPass &L, cudaStream_t st);
int tc_points_per_tile();  // K3 tile: 256 output points per CTA pair, 256 reduction points per B tile

// One LSE pass: outputs P side points, reduces over Q side.  Splits:
// nblk blocks of blk_tiles Q tiles each (the last may be shorter; blk_tiles = 0
// means one block of all tiles), each cut into split_q sub-splits.  Writes
// part[s * P + p] = (M, S) for s in [0, nblk*split_q).
struct LsePass {
    const Side *Pside, *Qside;
    int nblk, blk_tiles, split_q;
    float2 *part;
    float eps;
    const int *stop;  // device flag (nullable)
    int seeded = 0;   // fixed shift = Pside->lse[p] + margin (no running max); see k_merge
    const int *only_if = nullptr;   // run only if *only_if != 0 (the exact redo of a seeded column pass)
    int emu8 = 1;     // seeded D <= 4: exponential pairs (of 8) on the FMA pipe (sk_set_tuning "lse_emu8")
    float margin = 4.f;   // seeded: log2 units above the previous LSE (sk_set_tuning "lse_margin")
    int R = 0;            // output points per thread: 0 = the default for D, 1 = one (D <= 4: small problems)
    float2 *xchg = nullptr;   // non-null: fused K6a - the block partials [nblk][P] (this slice's
    int *cnt = nullptr;       //   slots) and the arrival counters [nblk][P tiles] (zero between launches)
};
// K6a: per fixed row block, the stable merge of its split_q sub-split partials in fixed order:
// part [nblk * split_q][P] -> out [nblk][P], one (M, S) per point per block (the exchange payload
// of the column pass; the same merge tree for every partition of the rows).
cudaError_t launch_premerge(const float2 *part, int nblk, int split_q, long long P, float2 *out, const int *stop,
                            const int *only_if, cudaStream_t st);
cudaError_t launch_lse(const LsePass &L, cudaStream_t st);
int lse_occupancy_ctas(int D, int R = 0);  // resident CTAs per SM of the LSE kernel for D (R = 0: default)

enum MergeMode { MERGE_COL = 0, MERGE_ROW = 1, MERGE_OUT = 2 };
struct MergePass {
    MergeMode mode;
    const Side *S;    // output side (its c, nk, pack.w and pot buffers)
    const float2 *part;
    int nsplit;
    float eps;
    const float *wts;         // b (COL) weights for the error, nullable = uniform
    DevStatus *st;
    double *blk_err;          // per-block scratch
    int *blk_bad;
    float *out;               // MERGE_OUT destination
    float out_const;          // MERGE_OUT: added constant (eps log ms for Eq. 8)
    int sharded;              // non-finite f is detected by the next (replicated) column merge
    int no_iter_inc;          // MERGE_ROW of a non-final slice (emulated ranks): keep the counter
    int precomputed = 0;      // MERGE_ROW: potential and w already written (fused stored sweep)
    const Side *Q = nullptr;  // seeded passes: the reduced side, for the exact fallback
    int scaled = 0;           // MERGE_COL of the fused stored sweep: partials are (-g kappa, A_j)
    const float *Cst = nullptr;   // scaled: the full stored C (n_rows x m) for the in-merge exact fallback
    const float *xw = nullptr;    //         and the X side w = f kappa (n_rows)
    long long n_rows = 0;
    const int *only_if = nullptr;  // run only if *only_if != 0 (the exact column fallback)
    int tc_fold = 0;          // K3 side: also fold lse + margin as the next pass's row shift
    float tc_margin = 4.f;    //          log2 units above the LSE (SK_TC_SEED_MARGIN: test knob)
    float omega = 1.f;        // Alg. 1's relaxation: h <- (1 - omega) h_old + omega h_sinkhorn
    int accum = 0;            // relaxed ROW of a later slice: add its row terms (row_err, mass_dev)
    int anderson = 0;         // Anderson (R-27): COL takes no decision; ROW writes its slice's
    double *and_err = nullptr;//   row term of err_l for (f^l, g~) to *and_err (K19 decides)
    int adapt = 0;            // adaptive momentum window T (R-31): omega from st->omega, and the
                              //   column merge estimates the next omega at the end of a window
    long long n_uniform = 0;  // uniform weights (wts == nullptr): 1 / n_uniform (0: the side's own P);
                              //   a row slice of a sharded solve weighs its rows by 1 / n_total
    int range_redo = 0;       // COL after a seeded pass: a sum outside [2^-100, 2^100] sets
                              //   st->colfail (no decision) and the column pass is redone exactly
};
cudaError_t launch_merge(const MergePass &M, cudaStream_t st);
// K19 Anderson (sk_anderson.cu): state = anderson_state_bytes() (zeroed before the solve); per
// slice F/R = 2 x mem x n floats, blk = anderson_blk_doubles(), vec = anderson_vec_doubles()
// (vec[0..8): Gram dots, vec[8]: the row term of err_l written by the row merge).
size_t anderson_state_bytes();
size_t anderson_blk_doubles();
size_t anderson_vec_doubles();
cudaError_t launch_anderson_dots(const Side &X, const DevStatus *st, const void *state, int mem, float *F,
                                 float *R, double *blk, double *vec, cudaStream_t s);
cudaError_t launch_anderson_decide(DevStatus *st, void *state, int mem, const double *vec, int ns, cudaStream_t s);
cudaError_t launch_anderson_mix(const Side &X, const DevStatus *st, const void *state, const float *F, float eps,
                                cudaStream_t s);
constexpr int kMergeMaxBlocks = 1184;   // blk_err holds 2 x kMergeMaxBlocks doubles
int merge_blocks(int P);

// E = <f,a> + <g,b> - eps sum(a) of the iterate status->final_iter.
cudaError_t launch_report(const Side &X, const Side &Y, const float *a, const float *b, float eps,
                          DevStatus *st, int local_only, long long n_uniform, cudaStream_t s);

cudaError_t launch_status_init(DevStatus *st, int max_iter, int check_every, float tol,
                               cudaStream_t s, int g_off = 0, float omega0 = 1.f);
cudaError_t launch_report_blocks(const Side &X, const float *a, float eps, DevStatus *st, long long n_uniform,
                                 long long row0, long long bs, double *out, cudaStream_t s);

// ------------------------------------------------------------ misc kernels
cudaError_t launch_fill(float *p, long long n, float v, cudaStream_t st);
struct CheckList {   // up to 8 arrays checked by one launch (n > 0 entries only)
    const float *p[8];
    long long n[8];
    int positive[8];
    int cnt;
    long long total;
};
cudaError_t launch_check_multi(const CheckList &L, int *flag, cudaStream_t st);
cudaError_t launch_check_finite(const float *p, long long n, int *flag, cudaStream_t st);
cudaError_t launch_check_positive(const float *p, long long n, int *flag, cudaStream_t st);
cudaError_t launch_gather_rows(const float *src, const int *idx, long long cnt, int d, float *dst,
                               cudaStream_t st);
cudaError_t launch_check_indices(const int *idx, long long cnt, long long n, int *flag, int *scratch,
                                 cudaStream_t st);

// ----------------------------------------------------------------- sort1d
// rows of n > 8192 keys need gkeys (sort_rows_scratch_keys(B, n) u64); the closed-form dual for
// n > 4096 needs gscr (4 B n doubles)
size_t sort_rows_scratch_keys(int B, int n);
cudaError_t launch_sort_rows(const float *x, int B, int n, long long stride, int *perm, int *rank,
                             float *sorted, int *nanflag, cudaStream_t st, unsigned long long *gkeys = nullptr);
cudaError_t launch_sort1d_dual(const float *xs_sorted, const int *perm, const float *ys_sorted,
                               int y_shared, int B, int n, int iters, float *pot, cudaStream_t st,
                               double *gscr = nullptr);

// --------------------------------------------------------------- Gaussian
cudaError_t launch_moments(const float *x, const float *w, long long n, int d, double *mean,
                           double *cov, double *scratch, long long scratch_doubles, cudaStream_t st);
cudaError_t launch_gauss_A(const double *mean_mu, double *cov_mu, const double *mean_nu,
                           double *cov_nu, int d, float ridge_rel, double *A, int *ns_fail,
                           cudaStream_t st, double *work = nullptr);   // work: d > 64 (gauss_wide_work_doubles)
size_t gauss_wide_work_doubles(int d);
long long moments_blocks(int d);   // row blocks of the moment partials (scratch: moments_blocks(d) * d^2)
cudaError_t launch_gauss_potential(const float *x, long long n, int d, const double *m_mu,
                                   const double *m_nu, const double *A, float *pot, cudaStream_t st);

// -------------------------------------------------------------------- GMM
cudaError_t launch_gmm_init(const float *x, long long n, int d, int Kx, const float *wx,
                            const float *mux, const float *covx, int Ky, const float *wy,
                            const float *muy, const float *covy, float eps, float inner_tol,
                            int inner_max_iter, float *pot, double *work, int *flags,
                            cudaStream_t st);
size_t gmm_work_doubles(int d, int Kx, int Ky);

// ------------------------------------------------------------- stored mode
cudaError_t launch_build_cost(const float *x, const float *y, long long n, long long m, int d,
                              float *C, cudaStream_t st);
struct StoredPass {
    const float *C; long long n, m;   // row-major n x m fp32
    float eps;
    const float *wq;      // reduction-side w = h log2(e)/eps (the other side's D=0 pack)
    float2 *part;         // rows: [n] (one split); cols: [nblk * split_q][m]
    long long blk_rows;   // cols: rows per fixed block (0 = one block of all rows)
    int nblk, split_q;    // cols: blocks and sub-splits per block
    const int *stop;
    const int *only_if = nullptr;   // cols: run only if *only_if != 0
};
cudaError_t launch_stored_rows(const StoredPass &S, cudaStream_t st);
// Fused single-read sweep (H4s): f^{l+1} rows (written with their w) and the column partials
// of g^{l+2} from one read of each row block of C.
struct FusedLaunch {
    const float *C; long long n, m;
    float eps;
    const float *gw, *xc;
    float *xpot[2];
    float *xw;
    float *xlse;      // per-row LSE (log2 units) of the previous sweep: the row shift seed (-inf = none)
    float2 *part;
    long long blk_rows;
    int nblk, split_q;
    DevStatus *st;
    int sharded = 0;      // row bookkeeping as MERGE_ROW: non-finite rows are caught by the column merge
    int no_iter_inc = 0;  // non-final slice of the emulated ranks: keep the sweep counter
};
bool stored_fused_supported(long long m);
cudaError_t launch_stored_fused(const FusedLaunch &L, cudaStream_t st);
cudaError_t launch_stored_cols(const StoredPass &S, cudaStream_t st);

// ------------------------------------------------------------ K14 microbenchmarks
cudaError_t microbench_alu(int kind, cudaStream_t st, cudaEvent_t e0, cudaEvent_t e1, float *sink, double *ops);
cudaError_t microbench_mma(int kind, void *scratch, cudaStream_t st, double *flop_per_clk);
cudaError_t microbench_hbm(const float *buf, long long bytes, cudaStream_t st, cudaEvent_t e0, cudaEvent_t e1,
                           float *sink);

}  // namespace sk
