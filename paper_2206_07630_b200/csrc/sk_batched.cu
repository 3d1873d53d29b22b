// sk_batched.cu — K13: the on-chip Sinkhorn solver for batches of small problems.
//
// One CTA solves one problem end to end ("compounded when running
// many thousands of OT problems"): x, y, both potentials and the packed
// reduction operands live in shared memory; every sweep is
//     column pass  g_j <- eps log b_j - eps LSE_i((f_i - C_ij)/eps)   (Alg. 1 l.5, R-1)
//     [error check err_l = sum_j b_j |expm1((g_j^l - g_j^{l+1})/eps)| (H5,
//      threshold appendix) every check_every sweeps]
//     row pass     f_i <- eps log a_i - eps LSE_j((g_j - C_ij)/eps)   (Alg. 1 l.4)
// with C_ij = ||x_i||^2 + ||y_j||^2 - 2<x_i, y_j> evaluated on the fly (FFMA2),
// and per-problem convergence (each CTA leaves its loop independently).
// Deterministic: every output is produced by one thread in a fixed order and the
// block reductions have a fixed shape.
#include "sk_internal.h"
#include "sk_lse_tile.cuh"

#include <algorithm>
#include <cstdlib>

namespace sk {


struct BatchArgs {
    int B;
    int *queue;                     // dynamic problem queue (zeroed before launch)
    const float *x; long long xs;   // per-problem strides in floats (0 = shared)
    const float *y; long long ys;
    const float *a; long long as;   // nullable (uniform)
    const float *b; long long bs;
    const float *finit; long long fs;  // nullable
    float *f; float *g;             // B x n, B x m
    int n, m;
    float eps, tol;
    int max_iter, check_every;
    int *iters, *conv, *nonfinite;
    float *err;
    double *E;
    float omega;                    // Alg. 1's relaxation (1 = plain Sinkhorn)
    float decay_init, decay_rate;   // eps-decay (decay_init <= 0: off)
    int anderson;                   // Anderson memory (R-27; < 2: off)
    int adapt;                      // adaptive momentum window T (R-31; 0: off)
    // park / resume scheduling (CL = 1 batches larger than the resident CTAs; park = 0: off): a
    // problem runs at most `park` sweeps per turn, then its state is saved and it is re-queued
    // with the predicted number of remaining sweeps as its priority
    int park;
    unsigned long long *pq;         // [kParkBuckets] bucket stacks: (ABA tag << 32) | (top problem + 1),
                                    // then int next[B]: the problem below each parked one (+ 1; 0 = none)
    float *pseed;                   // [B][n + m] the per-point LSE seeds (mxs, mys)
    double *phdr;                   // [B][8] sweep count, relaxed / adaptive state
    int *done;                      // problems finished
};
// priority buckets of parked problems: predicted remaining sweeps, clamped to [0, 63]
constexpr int kParkBuckets = 64;

__host__ __device__ inline int round_up(int v, int a) { return (v + a - 1) / a * a; }

constexpr int kRedW = 4;              // values per pass reduction (error, flag, relaxed row terms)
constexpr int kRedDoubles = 2 * 32 * kRedW + 2 * 2 * 16;   // double-buffered partials, pair exchange
constexpr int kAndMax = 8;            // largest Anderson memory
constexpr int kAndDoubles = kAndMax * kAndMax + 2 * 32 * (kAndMax + 2);   // Gram matrix, partials

size_t batched_smem_bytes(int D, int n, int m, int mem) {
    const int Np = round_up(n, kChunk), Mp = round_up(m, kChunk);
    size_t floats = (size_t)(D + 1) * (Np + Mp)   // packed coords + w, both sides
                    + 2 * (size_t)(n + m)         // finalize constant c and ||.||^2 kappa
                    + 2 * (size_t)(n + m)         // double-buffered f and g
                    + (size_t)(n + m) + 2;        // last running max per point (seed), alignment
    size_t bytes = floats * sizeof(float) + kRedDoubles * sizeof(double);
    if (mem >= 2) bytes += kAndDoubles * sizeof(double) + 2 * (size_t)mem * n * sizeof(float);   // + T(f), residuals
    return bytes;
}

// Fixed-order block sums of v[0..k) (k <= ST); all threads get the results in v.  The
// partials alternate between two scratch halves (par), so one barrier per reduction suffices:
// reduction r + 2 rewrites a half only after every thread has passed reduction r + 1's
// barrier, i.e. finished reading reduction r.  The barrier also orders the pass's shared-memory
// writes before the next pass's reads.
template <int NT, int ST>
__device__ __forceinline__ void block_red(double *v, int k, double *scratch /* 2 x 32 x ST */, int &par) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    double *sc = scratch + par * 32 * ST;
    par ^= 1;
    double t[ST];
#pragma unroll
    for (int u = 0; u < ST; ++u) t[u] = u < k ? v[u] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)   // (level by level: the k shuffles of a level overlap)
#pragma unroll
        for (int u = 0; u < ST; ++u)
            if (u < k) t[u] += __shfl_xor_sync(0xffffffffu, t[u], o);
    if (l == 0) {
#pragma unroll
        for (int u = 0; u < ST; ++u)
            if (u < k) sc[w * ST + u] = t[u];
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < ST; ++u) {
        if (u >= k) continue;
        double a = 0.0;
#pragma unroll
        for (int i = 0; i < NT / 32; ++i) a += sc[i * ST + u];
        v[u] = a;
    }
}

constexpr float kSeedMargin = 4.f;   // log2 units added to the previous sweep's max

// One LSE pass over all P points owned by this CTA (R per thread per round).
// First sweep: exact online max per chunk (lse_chunk).  Later sweeps: the shift is
// fixed at the point's previous LSE + kSeedMargin (lse_chunk_seeded: no max, no
// rescale); if the sum leaves [2^-100, 2^100] the point is recomputed exactly.
// out(p, M, S) is called for every valid p by the thread that owns it.
template <int D, int R, int NT, int EMU, typename Out>
__device__ __forceinline__ void onchip_pass(const float *__restrict__ pc, int pstride, int p0, int P,
                                            const float *__restrict__ qc, const float *__restrict__ qw,
                                            int Qp, float tk, float *pm, bool seeded, Out out) {
    // outputs p in [p0, P)
    for (int pb = p0; pb < P; pb += R * NT) {
        float2 pd[R][D];
        float M[R];
        float2 S[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int p = pb + r * NT + threadIdx.x;
#pragma unroll
            for (int k = 0; k < D; ++k) {
                const float v = p < P ? pc[k * pstride + p] * tk : 0.f;
                pd[r][k] = make_float2(v, v);
            }
            M[r] = seeded && p < P ? pm[p] + kSeedMargin : -INFINITY;
            S[r] = make_float2(0.f, 0.f);
        }
        if (seeded) {
            for (int q = 0; q < Qp; q += kChunk) lse_chunk_seeded<D, R, EMU>(qc, Qp, qw, q, pd, M, S);
        } else {
            for (int q = 0; q < Qp; q += kChunk) lse_chunk<D, R, EMU>(qc, Qp, qw, q, pd, M, S);
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int p = pb + r * NT + threadIdx.x;
            if (p >= P) continue;
            float Sv = S[r].x + S[r].y;
            if (!(Sv >= 0x1p-100f && Sv <= 0x1p100f)) {  // seed far off the true max: exact recompute
                float2 Sr[1] = {make_float2(0.f, 0.f)};
                float Mr[1] = {-INFINITY};
                float2 pr[1][D];
#pragma unroll
                for (int k = 0; k < D; ++k) pr[0][k] = pd[r][k];
                for (int q = 0; q < Qp; q += kChunk) lse_chunk<D, 1, 0>(qc, Qp, qw, q, pr, Mr, Sr);
                M[r] = Mr[0];
                Sv = Sr[0].x + Sr[0].y;
            }
            pm[p] = M[r] + log2f(Sv);  // this sweep's LSE: the next sweep's seed
            out(p, M[r], Sv);
        }
    }
}

// ---------------------------------------------------------- CTA-pair (cluster) helpers
__device__ __forceinline__ uint32_t cl_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cl_map(const void *p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void cl_st(uint32_t addr, float v) {
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ void cl_st(uint32_t addr, double v) {
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ void cl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Solve problem `prob` with the whole CTA (CL = 1) or a CTA pair (CL = 2: each CTA computes the
// outputs of one half of every pass and stores them into both CTAs' shared memory (DSMEM);
// reductions combine the two halves' block partials in a fixed order, so both CTAs take the
// same decisions).  The per-point arithmetic is the same for CL = 1 and 2 (same potentials).
template <int D, int R, int NT, int EMU, int CL>
__device__ __forceinline__ int solve_one(const BatchArgs &A, int prob, bool resume, float *sm, uint32_t rank) {
    const int n = A.n, m = A.m;
    const int Np = round_up(n, kChunk), Mp = round_up(m, kChunk);
    const float eps_t = A.eps;          // the target eps
    float eps = eps_t;                  // this sweep's eps (eps-decay, R-25)
    float kap = kLog2e / eps;           // log2(e)/eps
    float tk = 2.f * kap;               // scale of the cross term
    float epsln2 = eps * kLn2;

    float *xq = sm;                     // [D][Np]
    float *wx = xq + D * Np;            // [Np]   (f_i - |x_i|^2) kappa
    float *yq = wx + Np;                // [D][Mp]
    float *wy = yq + D * Mp;            // [Mp]   (g_j - |y_j|^2) kappa
    float *cx = wy + Mp;                // [n]    eps log a_i + |x_i|^2
    float *nxk = cx + n;                // [n]    |x_i|^2 kappa
    float *cy = nxk + n;                // [m]
    float *nyk = cy + m;                // [m]
    float *fb = nyk + m;                // [2][n]
    float *gb = fb + 2 * n;             // [2][m]
    float *mxs = gb + 2 * m;            // [n]    last running max (x side, row pass)
    float *mys = mxs + n;               // [m]    (y side, column pass)
    double *red = reinterpret_cast<double *>(mys + m + ((n + m) & 1));  // scratch
    double *xr = red + 2 * 32 * kRedW;  // [2 halves][2 ranks][16] exchanged block partials (CL = 2)
    int rpar = 0, xpar = 0;             // the halves the next reductions use
    // Anderson (R-27): Gram matrix of the residuals, mixing weights, partials; T(f) and residuals
    const int am = A.anderson >= 2 ? A.anderson : 0;
    double *Gm = red + kRedDoubles;     // [kAndMax][kAndMax]
    double *vred = Gm + kAndMax * kAndMax;   // [2][32][kAndMax + 2]
    float *Fh = reinterpret_cast<float *>(vred + 2 * 32 * (kAndMax + 2));   // [am][n]
    float *Rh = Fh + (size_t)am * n;                                    // [am][n]
    // this CTA's output ranges (CL = 2: halves, aligned to R * NT rounds)
    const int hn = CL > 1 ? (n + 1) / 2 : n, hm = CL > 1 ? (m + 1) / 2 : m;
    const int i0 = CL > 1 ? (int)rank * hn : 0, i1 = CL > 1 ? min(n, i0 + hn) : n;
    const int j0 = CL > 1 ? (int)rank * hm : 0, j1 = CL > 1 ? min(m, j0 + hm) : m;
    const uint32_t peer_base = CL > 1 ? cl_map(sm, rank ^ 1u) : 0u;
    auto rput = [&](float *loc, float v) {   // the same slot in the peer CTA
        if constexpr (CL > 1) cl_st(peer_base + (smem_u32(loc) - smem_u32(sm)), v);
    };
    // sum of this CTA's block partial v[k] with the peer's (fixed order: rank 0 + rank 1).  One
    // cluster barrier: it also publishes the pass's DSMEM stores, and the two halves of xr
    // alternate (as in block_red), so a half is rewritten only after both CTAs have read it.
    auto xsum = [&](double *v, int cnt) {
        if constexpr (CL > 1) {
            double *xh = xr + xpar * 32;
            xpar ^= 1;
            if (threadIdx.x == 0)
                for (int k = 0; k < cnt; ++k) {
                    xh[rank * 16 + k] = v[k];
                    cl_st(peer_base + (smem_u32(&xh[rank * 16 + k]) - smem_u32(sm)), v[k]);
                }
            cl_sync();
            for (int k = 0; k < cnt; ++k) v[k] = xh[k] + xh[16 + k];
        }
    };

    const float *x = A.x + prob * A.xs;
    const float *y = A.y + prob * A.ys;
    const float *a = A.a ? A.a + prob * A.as : nullptr;
    const float *b = A.b ? A.b + prob * A.bs : nullptr;
    const float loga_u = (float)(-log((double)n)), logb_u = (float)(-log((double)m));

    // ---- load + precompute (K1)
    for (int i = threadIdx.x; i < Np; i += NT) {
        if (i < n) {
            float s = 0.f;
#pragma unroll
            for (int k = 0; k < D; ++k) {
                const float v = x[(size_t)i * D + k];
                xq[k * Np + i] = v;
                s = fmaf(v, v, s);
            }
            const float la = a ? logf(a[i]) : loga_u;
            cx[i] = fmaf(eps, la, s);
            nxk[i] = s * kap;
            // (resume: the parked f^l and seeds, written by another CTA: L2 loads)
            const float f0 = resume ? __ldcg(A.f + (size_t)prob * n + i)
                                    : (A.finit ? A.finit[(size_t)prob * A.fs + i] : 0.f);
            fb[i] = f0;
            wx[i] = fmaf(f0, kap, -nxk[i]);
            mxs[i] = resume ? __ldcg(A.pseed + (size_t)prob * (n + m) + i) : -INFINITY;
        } else {
#pragma unroll
            for (int k = 0; k < D; ++k) xq[k * Np + i] = 0.f;
            wx[i] = -INFINITY;
        }
    }
    for (int j = threadIdx.x; j < Mp; j += NT) {
        if (j < m) {
            float s = 0.f;
#pragma unroll
            for (int k = 0; k < D; ++k) {
                const float v = y[(size_t)j * D + k];
                yq[k * Mp + j] = v;
                s = fmaf(v, v, s);
            }
            const float lb = b ? logf(b[j]) : logb_u;
            cy[j] = fmaf(eps, lb, s);
            nyk[j] = s * kap;
            gb[j] = resume ? __ldcg(A.g + (size_t)prob * m + j) : 0.f;  // g^(0) = 0 (only f^(0) is needed)
            mys[j] = resume ? __ldcg(A.pseed + (size_t)prob * (n + m) + n + j) : -INFINITY;
        } else {
#pragma unroll
            for (int k = 0; k < D; ++k) yq[k * Mp + j] = 0.f;
            wy[j] = -INFINITY;
        }
    }
    __syncthreads();

    int l = 0, cur = 0, conv = 0, nonfin = 0;
    const double *hdr = A.phdr + (size_t)prob * 8;
    if (resume) l = (int)__ldcg(hdr);
    int a_cnt = 0, a_head = 0;   // Anderson history: filled slots, next slot
    bool out_gtilde = false;     // Anderson: the result is (f^l, g_sk(f^l)) (the g buffer not flipped)
    float err = INFINITY;
    // adaptive momentum (R-31): plain until the second window's error, then omega from each
    // window's contraction, applied two sweeps after the window's last sweep
    float om = A.adapt > 0 ? 1.f : A.omega, om_next = om, err_win = 0.f;
    const bool relaxed = A.adapt > 0 || om != 1.f;
    double row_err = 0.0, mass_dev = 0.0;   // relaxed: row term of err_l and sum P - sum a
    if (resume) {
        row_err = __ldcg(hdr + 1); mass_dev = __ldcg(hdr + 2); err = (float)__ldcg(hdr + 3);
        om = (float)__ldcg(hdr + 4); om_next = (float)__ldcg(hdr + 5); err_win = (float)__ldcg(hdr + 6);
    }
    // park after `park` sweeps of this turn; the errors of its last two sweeps predict the rest
    const int l_park = A.park > 0 ? l + A.park : 0x7fffffff;
    float pe1 = INFINITY, pe2 = INFINITY;
    // eps-decay (R-25): sweep l + 1 uses max(eps, eps init rate^l); the T decay sweeps
    // are not checked; the constants that carry eps are refreshed when it changes
    auto eps_of = [&](int s) {
        if (A.decay_init <= 0.f) return eps_t;
        const float v = eps_t * A.decay_init * powf(A.decay_rate, (float)s);
        return v > eps_t ? v : eps_t;
    };
    int T = 0;
    while (T < A.max_iter && eps_of(T) > eps_t) ++T;
    auto refresh = [&](float e) {
        eps = e; kap = kLog2e / e; tk = 2.f * kap; epsln2 = e * kLn2;
        const float *fc = fb + cur * n;
        for (int i = threadIdx.x; i < n; i += NT) {
            float s2 = 0.f;
#pragma unroll
            for (int k = 0; k < D; ++k) s2 = fmaf(xq[k * Np + i], xq[k * Np + i], s2);
            cx[i] = fmaf(e, a ? logf(a[i]) : loga_u, s2);
            nxk[i] = s2 * kap;
            wx[i] = fmaf(fc[i], kap, -nxk[i]);
        }
        for (int j = threadIdx.x; j < m; j += NT) {
            float s2 = 0.f;
#pragma unroll
            for (int k = 0; k < D; ++k) s2 = fmaf(yq[k * Mp + j], yq[k * Mp + j], s2);
            cy[j] = fmaf(e, b ? logf(b[j]) : logb_u, s2);
            nyk[j] = s2 * kap;
        }
        __syncthreads();
    };
    bool fresh = true;   // the LSE seeds (previous sweep's LSE) belong to this sweep's eps
    for (;;) {
        if (l >= l_park) {
            // park: (f^l, g^l), the seeds and the sweep state -> global; the priority is the
            // predicted remaining sweep count log(err_{l-1} / tol) / log(1 / rho),
            // rho = err_{l-1} / err_{l-2} (a problem without both errors goes first)
            const float *fo = fb + cur * n, *go = gb + cur * m;
            for (int i = threadIdx.x; i < n; i += NT) {
                A.f[(size_t)prob * n + i] = fo[i];
                A.pseed[(size_t)prob * (n + m) + i] = mxs[i];
            }
            for (int j = threadIdx.x; j < m; j += NT) {
                A.g[(size_t)prob * m + j] = go[j];
                A.pseed[(size_t)prob * (n + m) + n + j] = mys[j];
            }
            float key = 1e30f;
            if (threadIdx.x == 0) {
                double *h = A.phdr + (size_t)prob * 8;
                h[0] = (double)l; h[1] = row_err; h[2] = mass_dev; h[3] = (double)err;
                h[4] = (double)om; h[5] = (double)om_next; h[6] = (double)err_win;
                if (pe1 < INFINITY && pe2 < INFINITY && pe2 > 0.f) {
                    const float rho = fminf(fmaxf(pe2 / pe1, 1e-6f), 0.999999f);
                    key = fmaxf(logf(fmaxf(pe2, 1e-30f) / A.tol), 0.f) / -logf(rho);
                    if (!(key >= 0.f)) key = 1e30f;
                }
            }
            __threadfence();
            __syncthreads();
            if (threadIdx.x == 0) {   // push onto its priority bucket (lock-free stack, ABA-tagged)
                const int bk = key >= (float)(kParkBuckets - 1) ? kParkBuckets - 1 : (int)key;
                volatile int *nxt = reinterpret_cast<volatile int *>(A.pq + kParkBuckets);
                for (;;) {
                    const unsigned long long old = *(volatile unsigned long long *)(A.pq + bk);
                    nxt[prob] = (int)(old & 0xffffffffull);
                    __threadfence();
                    const unsigned long long nw = (((old >> 32) + 1ull) << 32) | (unsigned long long)(prob + 1);
                    if (atomicCAS(A.pq + bk, old, nw) == old) break;
                }
            }
            __syncthreads();   // smem is reused by the next problem
            return 1;
        }
        {
            const float el = eps_of(l);
            fresh = el == eps;
            if (!fresh) refresh(el);
        }
        const bool seeded = l >= 1 && fresh;
        // ---- column pass: g^{l+1} (P = y, Q = x)
        const bool check = !am && l > T && ((l - T) % A.check_every == 0 || l == A.max_iter);
        const bool chk_ad = A.adapt > 0 && l >= 1 && l % A.adapt == 0;   // err_l ends a window
        const bool chk_pk = l >= 1 && (l == l_park - 2 || l == l_park - 1);   // the park's predictor
        double e_loc = 0.0;
        int bad = 0;
        float *gold = gb + cur * m, *gnew = gb + (cur ^ 1) * m;
        onchip_pass<D, R, NT, EMU>(yq, Mp, j0, j1, xq, wx, Np, tk, mys, seeded, [&](int j, float Mv, float Sv) {
            const float gsk = cy[j] - epsln2 * (Mv + log2f(Sv));
            // Alg. 1 with relaxation (R-1): g <- (1 - omega) g + omega g_sk
            const float gn = relaxed ? fmaf(om, gsk - gold[j], gold[j]) : gsk;
            const float wv = fmaf(gn, kap, -nyk[j]);
            gnew[j] = gn;
            wy[j] = wv;
            rput(&gnew[j], gn);
            rput(&wy[j], wv);
            bad |= !isfinite(gn);
            if (check || chk_ad || chk_pk) {
                const double bj = b ? (double)b[j] : 1.0 / m;
                e_loc += bj * fabs((double)expm1f((gold[j] - gsk) / eps));
            }
        });
        double cv[2] = {e_loc, (double)bad};
        block_red<NT, kRedW>(cv, 2, red, rpar);
        xsum(cv, 2);   // (CL = 2: also publishes the peer's half of g and w)
        if (cv[1] != 0.0) { nonfin = 1; break; }
        if (check || chk_ad || chk_pk) {
            const float en = (float)(cv[0] + row_err);   // (row_err = 0 unless relaxed)
            if (chk_pk) { if (l == l_park - 2) pe1 = en; else pe2 = en; }
            if (check) {
                err = en;
                if (err < A.tol) { conv = 1; break; }
            }
            if (chk_ad) {
                if (l >= 2 * A.adapt) om_next = adaptive_omega((double)en / (double)err_win, A.adapt, om);
                err_win = en;
            }
        }
        if (!am && l >= A.max_iter) break;   // (also when max_iter <= T: no sweep is checked)
        // ---- row pass: f^{l+1} (P = x, Q = y); wy is visible after the reductions' barriers
        float *fnew = fb + (cur ^ 1) * n;
        const float *fold = fb + cur * n;
        bad = 0;
        if (am) {
            // Anderson (R-27): sweep l + 1 of the map T(f) = f_sk(g_sk(f)).  The
            // pair (f^l, g~) has exact columns: err = sum_i a_i |expm1((f_i - T(f)_i)/eps)|.
            const bool check_a = (l + 1) % A.check_every == 0 || l + 1 == A.max_iter;
            const int cn = a_cnt < am ? a_cnt + 1 : am;   // slots after this push
            onchip_pass<D, R, NT, EMU>(xq, Np, i0, i1, yq, wy, Mp, tk, mxs, seeded, [&](int i, float Mv, float Sv) {
                const float fsk = cx[i] - epsln2 * (Mv + log2f(Sv));
                bad |= !isfinite(fsk);
                Fh[(size_t)a_head * n + i] = fsk;   // (the residual and the dots after the pass:
            });                                     //  no extra registers live in it)
            double dv[kAndMax], e_row = 0.0;
#pragma unroll
            for (int u = 0; u < kAndMax; ++u) dv[u] = 0.0;
            for (int i = i0 + threadIdx.x; i < i1; i += NT) {   // (the points this thread wrote)
                const float fsk = Fh[(size_t)a_head * n + i];
                const float r = fsk - fold[i];
                if (check_a) e_row += (a ? (double)a[i] : 1.0 / n) * fabs((double)expm1f(-r / eps));
#pragma unroll
                for (int u = 0; u < kAndMax; ++u)
                    if (u < cn) dv[u] += (double)r * (double)(u == a_head ? r : Rh[(size_t)u * n + i]);
                Rh[(size_t)a_head * n + i] = r;
            }
            double vv[kAndMax + 2];   // slots 0..7: the dots (0 beyond cn), 8: the error, 9: the flag
#pragma unroll
            for (int u = 0; u < kAndMax; ++u) vv[u] = dv[u];
            vv[kAndMax] = e_row;
            vv[kAndMax + 1] = (double)bad;
            block_red<NT, kAndMax + 2>(vv, kAndMax + 2, vred, rpar);
            xsum(vv, kAndMax + 2);
            if (vv[kAndMax + 1] != 0.0) { nonfin = 1; break; }
            if (check_a) {
                err = (float)vv[kAndMax];
                if (err < A.tol) { conv = 1; out_gtilde = true; break; }
            }
            if (l + 1 >= A.max_iter) { out_gtilde = true; break; }
            // alpha from (G + lam I) x = 1, alpha = x / sum x: every warp solves the cn x cn
            // system redundantly in registers (lane r holds row r; Gauss-Jordan, pivots in
            // order, the same bits in every warp), so no barrier publishes alpha
            const int lane = threadIdx.x & 31;
            double dl = 0.0;          // this lane's new Gram entry <r_new, r_lane>
#pragma unroll
            for (int u = 0; u < kAndMax; ++u)
                if (u == lane) dl = vv[u];
            double row[kAndMax];
#pragma unroll
            for (int u = 0; u < kAndMax; ++u) {
                double gv;
                if (lane == a_head) gv = vv[u];
                else if (u == a_head) gv = dl;
                else gv = lane < kAndMax ? Gm[lane * kAndMax + u] : 0.0;
                row[u] = (lane < cn && u < cn) ? gv : (u == lane ? 1.0 : 0.0);
            }
            double diag = 0.0;
#pragma unroll
            for (int u = 0; u < kAndMax; ++u)
                if (u == lane) diag = row[u];
            double tr = lane < cn ? diag : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, o);
            const double lam = tr > 0.0 ? 1e-8 * tr / cn : 1.0;   // (all residuals 0: equal weights)
#pragma unroll
            for (int u = 0; u < kAndMax; ++u)
                if (u == lane && lane < cn) row[u] += lam;
            double rhs = lane < cn ? 1.0 : 0.0;
            for (int c = 0; c < cn; ++c) {
                double piv[kAndMax], myc = 0.0;
#pragma unroll
                for (int u = 0; u < kAndMax; ++u) {
                    piv[u] = __shfl_sync(0xffffffffu, row[u], c);
                    if (u == c) myc = row[u];
                }
                const double prhs = __shfl_sync(0xffffffffu, rhs, c);
                const double pcc = __shfl_sync(0xffffffffu, myc, c);
                if (lane != c) {
                    const double q = myc / pcc;
#pragma unroll
                    for (int u = 0; u < kAndMax; ++u) row[u] = fma(-q, piv[u], row[u]);
                    rhs = fma(-q, prhs, rhs);
                }
            }
#pragma unroll
            for (int u = 0; u < kAndMax; ++u)
                if (u == lane) diag = row[u];
            const double xl = lane < cn ? rhs / diag : 0.0;
            double sx = xl;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sx += __shfl_xor_sync(0xffffffffu, sx, o);
            // degenerate least squares (R-30): fall back to the plain update T(f^l) for this sweep
            double al_l = xl / sx;
            if (!isfinite(sx) || sx == 0.0 || __any_sync(0xffffffffu, lane < cn && !isfinite(al_l)))
                al_l = lane == a_head ? 1.0 : 0.0;
            double au[kAndMax];
#pragma unroll
            for (int u = 0; u < kAndMax; ++u) au[u] = __shfl_sync(0xffffffffu, al_l, u);
            if (threadIdx.x < 32 && lane < cn) {   // the Gram row/column of the new slot, for later sweeps
                Gm[a_head * kAndMax + lane] = dl;
                Gm[lane * kAndMax + a_head] = dl;
            }
            a_head = (a_head + 1) % am;
            a_cnt = cn;
            for (int i = i0 + threadIdx.x; i < i1; i += NT) {   // f^{l+1} = sum_u alpha_u T(f_u)
                double v = 0.0;                                  // (Fh[.][i] written by this thread)
#pragma unroll
                for (int u = 0; u < kAndMax; ++u)
                    if (u < cn) v = fma(au[u], (double)Fh[(size_t)u * n + i], v);
                const float fn = (float)v;
                const float wv = fmaf(fn, kap, -nxk[i]);
                fnew[i] = fn;
                wx[i] = wv;
                rput(&fnew[i], fn);
                rput(&wx[i], wv);
            }
            if constexpr (CL > 1) cl_sync(); else __syncthreads();
            cur ^= 1;
            ++l;
            continue;
        }
        double r_loc = 0.0, m_loc = 0.0;
        onchip_pass<D, R, NT, EMU>(xq, Np, i0, i1, yq, wy, Mp, tk, mxs, seeded, [&](int i, float Mv, float Sv) {
            const float fsk = cx[i] - epsln2 * (Mv + log2f(Sv));
            const float fn = relaxed ? fmaf(om, fsk - fold[i], fold[i]) : fsk;
            const float wv = fmaf(fn, kap, -nxk[i]);
            fnew[i] = fn;
            wx[i] = wv;
            rput(&fnew[i], fn);
            rput(&wx[i], wv);
            bad |= !isfinite(fn);
            if (relaxed) {   // sum_j P_ij = a_i exp((f_i - fsk_i)/eps)
                const double ai = a ? (double)a[i] : 1.0 / n;
                const double dv = (double)expm1f((fn - fsk) / eps);
                r_loc += ai * fabs(dv);
                m_loc += ai * dv;
            }
        });
        double rv[3] = {(double)bad, r_loc, m_loc};
        block_red<NT, kRedW>(rv, relaxed ? 3 : 1, red, rpar);
        xsum(rv, relaxed ? 3 : 1);
        if (rv[0] != 0.0) { nonfin = 1; break; }
        if (relaxed) { row_err = rv[1]; mass_dev = rv[2]; }
        om = om_next;   // (adaptive: the estimate from err_{l-1}'s window, from sweep l + 2 on)
        cur ^= 1;
        ++l;
    }

    // ---- epilogue: (f^l, g^l), E = <f,a> + <g,b> - eps sum(a) (Eq. 2 after an f-update), report
    const float *fo = fb + cur * n, *go = gb + (out_gtilde ? cur ^ 1 : cur) * m;
    double s = 0.0;
    for (int i = i0 + threadIdx.x; i < i1; i += NT) {
        A.f[(size_t)prob * n + i] = fo[i];
        const double ai = a ? (double)a[i] : 1.0 / n;
        s += (double)fo[i] * ai - (double)eps * ai;
    }
    for (int j = j0 + threadIdx.x; j < j1; j += NT) {
        A.g[(size_t)prob * m + j] = go[j];
        s += (double)go[j] * (b ? (double)b[j] : 1.0 / m);
    }
    double ev[1] = {s};
    block_red<NT, kRedW>(ev, 1, red, rpar);
    xsum(ev, 1);
    const double E = ev[0] - (double)eps * mass_dev;   // relaxed: sum P != sum a
    if (threadIdx.x == 0 && rank == 0) {
        A.iters[prob] = am ? l + 1 : l;   // (Anderson: sweeps evaluated, as the oracle counts)
        A.conv[prob] = conv;
        A.nonfinite[prob] = nonfin;
        A.err[prob] = err;
        A.E[prob] = E;
        if (A.done) atomicAdd(A.done, 1);
    }
    __syncthreads();  // smem is reused by the next problem
    return 0;
}

// Persistent CTAs (one or two per SM) pull problems from a global queue: iteration
// counts differ per problem, so dynamic assignment balances the SMs.  NT <= 512: two
// CTAs per SM (64 registers; C2 13.4 ms vs 14.0 ms at one CTA per SM with 124 registers).
template <int D, int R, int NT, int EMU, int CL>
__global__ void __launch_bounds__(NT, NT <= 512 ? 2 : 1) k_batched(BatchArgs A) {
    extern __shared__ __align__(16) float sm[];
    __shared__ int s_prob, s_res;
    const uint32_t rank = CL > 1 ? cl_rank() : 0u;
    for (;;) {
        if constexpr (CL == 1) {
            if (threadIdx.x < 32) {   // warp 0: the next problem - fresh ones first, then parked ones
                const int lane = threadIdx.x;
                int pr = 0, res = 0;
                if (lane == 0) pr = atomicAdd(A.queue, 1);
                pr = __shfl_sync(0xffffffffu, pr, 0);
                if (pr >= A.B) {
                    pr = A.B;
                    while (A.park > 0) {
                        // the highest non-empty priority bucket (most remaining sweeps): pop its
                        // top by compare-and-swap - O(1) per claim, no scan of the problems
                        volatile unsigned long long *hd = A.pq;
                        const unsigned long long a0 = hd[lane], a1 = hd[lane + 32];
                        const unsigned lo = __ballot_sync(0xffffffffu, (a0 & 0xffffffffull) != 0ull);
                        const unsigned hi = __ballot_sync(0xffffffffu, (a1 & 0xffffffffull) != 0ull);
                        if (lo | hi) {
                            const int bk = hi ? 32 + 31 - __clz(hi) : 31 - __clz(lo);
                            int got = 0;
                            if (lane == 0) {
                                const unsigned long long old = hd[bk];
                                const int top = (int)(old & 0xffffffffull);
                                if (top != 0) {
                                    const int below = reinterpret_cast<volatile int *>(A.pq + kParkBuckets)[top - 1];
                                    const unsigned long long nw = (((old >> 32) + 1ull) << 32) | (unsigned)below;
                                    if (atomicCAS(A.pq + bk, old, nw) == old) got = top;
                                }
                            }
                            got = __shfl_sync(0xffffffffu, got, 0);
                            if (got) { pr = got - 1; res = 1; break; }
                            continue;   // lost the race: look again
                        }
                        // nothing parked: done when every problem has finished, else wait for a park
                        if (*(volatile const int *)A.done >= A.B) break;
                        __nanosleep(1000);
                    }
                }
                if (lane == 0) { s_prob = pr; s_res = res; }
                __threadfence();   // (the claimed problem's parked state is read after this)
            }
        } else if (threadIdx.x == 0 && rank == 0) {
            const int pr = atomicAdd(A.queue, 1);
            s_prob = pr;
            s_res = 0;
            if constexpr (CL > 1) {   // the pair's problem id into the peer's s_prob
                const uint32_t pa = cl_map(&s_prob, 1u);
                asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(pa), "r"(pr) : "memory");
            }
        }
        if constexpr (CL > 1) cl_sync(); else __syncthreads();
        const int prob = s_prob;
        const bool resume = CL == 1 && s_res != 0;
        if constexpr (CL > 1) cl_sync(); else __syncthreads();
        if (prob >= A.B) break;
        solve_one<D, R, NT, EMU, CL>(A, prob, resume, sm, rank);
    }
}

// EMU: exponential pairs (of 4 per chunk) evaluated on the FMA pipe instead of MUFU: 1 (25 %)
// measured best on C2 (0 and 2 were tuning variants, dropped to bound compile time).
template <int D, int R, int NT, int EMU, int CL>
static cudaError_t launch_batched_c(const BatchArgs &A, int B, cudaStream_t st) {
    const size_t smem = batched_smem_bytes(D, A.n, A.m, A.anderson);
    cudaError_t e = cudaFuncSetAttribute(k_batched<D, R, NT, EMU, CL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    int occ = 0, dev = 0, nsm = 148;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_batched<D, R, NT, EMU, CL>, NT, smem);
    if (e != cudaSuccess) return e;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    BatchArgs Ap = A;
    if (CL == 1) {
        const int grid = std::max(1, std::min(B, nsm * std::max(occ, 1)));
        if (!(A.park > 0 && B > grid && A.pq)) Ap.park = 0;   // park only when problems queue up
        k_batched<D, R, NT, EMU, 1><<<grid, NT, smem, st>>>(Ap);
        return cudaGetLastError();
    }
    Ap.park = 0;   // (CTA pairs: one turn per problem)
    const int pairs = std::max(1, std::min(B, nsm * std::max(occ, 1) / 2));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * pairs);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_batched<D, R, NT, EMU, CL>, Ap);
}

// CTA pairs (CL = 2: two halves of every pass, DSMEM exchange) halve a problem's latency; on
// a batch (C2) that should shorten the idle tail of the dynamic queue (21 % of SM time with
// uneven iteration counts) but measures on par with one CTA per problem (14.0 vs 13.8 ms: the
// cluster barriers and the R = 1 shape cost what the tail saves), so batches use one CTA.
template <int D, int R, int NT, int CL>
static cudaError_t launch_batched_e(const BatchArgs &A, int B, cudaStream_t st) {
    return launch_batched_c<D, R, NT, 1, CL>(A, B, st);
}

// One wide CTA per problem: NT threads x R output points per thread per round.
// shape 1 (sk_set_tuning "batched_shape", default) selects 512 threads x 2 points for
// 512 < P <= 1024, shape 0 1024 x 1.  With a CTA pair (CL = 2) each CTA's shape covers its half
// of the points (no idle lanes).
template <int D>
static cudaError_t launch_batched_d(const BatchArgs &A, int B, int shape, int clk, cudaStream_t st) {
    // CTA pair: opt-in for batches (sk_set_tuning "batched_cl" = 2), the default for one
    // latency-bound problem (C1: 0.267 vs 0.295 ms for 34 sweeps); 1 forces one CTA
    const int P = A.n > A.m ? A.n : A.m;
    const bool pair = clk == 2 || (clk == 0 && B == 1);
    if (pair && P > 128 && P <= 2048) {
        if (P <= 256) return launch_batched_e<D, 1, 128, 2>(A, B, st);
        if (P <= 512) return launch_batched_e<D, 1, 256, 2>(A, B, st);
        if (P <= 1024) return launch_batched_e<D, 1, 512, 2>(A, B, st);
        return launch_batched_e<D, 1, 1024, 2>(A, B, st);
    }
    if (P <= 256) return launch_batched_e<D, 1, 256, 1>(A, B, st);
    if (P <= 512) return launch_batched_e<D, 1, 512, 1>(A, B, st);
    if (P <= 1024) return shape == 1 ? launch_batched_e<D, 2, 512, 1>(A, B, st) : launch_batched_e<D, 1, 1024, 1>(A, B, st);
    return launch_batched_e<D, 2, 1024, 1>(A, B, st);  // more rounds of 2048 points for larger P
}

size_t park_queue_ints(int B) { return 2 * (size_t)kParkBuckets + (size_t)B; }

bool batched_supported(int d, int n, int m, int mem) {
    return d >= 1 && d <= 4 && mem <= kAndMax && batched_smem_bytes(d, n, m, mem) <= 200 * 1024;
}

cudaError_t launch_batched(const BatchLaunch &L, cudaStream_t st) {
    BatchArgs A;
    A.B = L.B;
    A.queue = L.queue;
    cudaError_t e = cudaMemsetAsync(L.queue, 0, sizeof(int), st);
    if (e != cudaSuccess) return e;
    A.x = L.x; A.xs = L.x_stride; A.y = L.y; A.ys = L.y_stride;
    A.a = L.a; A.as = L.a_stride; A.b = L.b; A.bs = L.b_stride;
    A.finit = L.finit; A.fs = L.n;
    A.f = L.f; A.g = L.g;
    A.n = L.n; A.m = L.m; A.eps = L.eps; A.tol = L.tol;
    A.max_iter = L.max_iter; A.check_every = L.check_every;
    A.iters = L.iters; A.conv = L.conv; A.nonfinite = L.nonfinite; A.err = L.err; A.E = L.E;
    A.omega = L.omega;
    A.decay_init = L.decay_init; A.decay_rate = L.decay_rate;
    A.anderson = L.anderson;
    A.adapt = L.adapt;
    A.park = (L.anderson >= 2 || L.decay_init > 0.f) ? 0 : L.park;
    A.pq = reinterpret_cast<unsigned long long *>(L.pq); A.pseed = L.pseed; A.phdr = L.phdr; A.done = L.done;
    if (A.park > 0) {
        if (!A.pq || !A.done || !A.pseed || !A.phdr) return cudaErrorInvalidValue;
        e = cudaMemsetAsync(A.pq, 0, sizeof(int) * 2 * kParkBuckets, st);   // empty stacks
        if (e == cudaSuccess) e = cudaMemsetAsync(A.done, 0, sizeof(int), st);
        if (e != cudaSuccess) return e;
    } else if (A.done) {
        e = cudaMemsetAsync(A.done, 0, sizeof(int), st);
        if (e != cudaSuccess) return e;
    }
    switch (L.d) {
        case 1: return launch_batched_d<1>(A, L.B, L.shape, L.cl, st);
        case 2: return launch_batched_d<2>(A, L.B, L.shape, L.cl, st);
        case 3: return launch_batched_d<3>(A, L.B, L.shape, L.cl, st);
        case 4: return launch_batched_d<4>(A, L.B, L.shape, L.cl, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace sk
