// sk_stored.cu — stored-cost mode (BJ.ns "a stored-cost mode for problems whose C
// fits in HBM, streaming C with 128-bit vectorised coalesced loads").
//
//  K4 k_build_cost : C_ij = sum_k (x_ik - y_jk)^2 in fp32 (direct differences),
//                    written once (4nm bytes; BJ.cfg3: 16384^2 = 1 GiB).
//  K5r k_rows      : f-pass, one warp per row, float4 streaming loads along the
//                    row: (max, sum 2^(t - max)) of t_ij = g_j log2(e)/eps - C_ij log2(e)/eps.
//  K5c k_cols      : g-pass, each thread owns 4 adjacent columns (one float4 per
//                    row, so a warp reads 512 contiguous bytes per row), CTAs split
//                    the rows; partials (max, sum) per column and split.
// Both feed the same merge kernel (K6) as the online path (the stored side has
// D = 0 and no |p|^2 folding).  Each pass reads C once: 4nm bytes per launch.
#include <algorithm>

#include "sk_internal.h"
#include "sk_common.cuh"

namespace sk {

// ------------------------------------------------------------------- K4
// Block = 256 columns x 32 rows; x rows staged transposed in shared memory ([k][32 rows]) so a
// thread reads 4 rows' coordinate k with one broadcast LDS.128; (x_ik - y_jk)^2 accumulated
// over k in order with packed FFMA2 (each lane is the scalar fmaf chain, bit for bit).
template <int DP>
__global__ void __launch_bounds__(256) k_build_cost(const float *__restrict__ x, const float *__restrict__ y,
                                                    long long n, long long m, int d, float *C) {
    __shared__ __align__(16) float sx[DP][32];
    const long long i0 = (long long)blockIdx.y * 32;
    const long long j = (long long)blockIdx.x * 256 + threadIdx.x;
    for (int t = threadIdx.x; t < 32 * DP; t += 256) {
        const int r = t / DP, k = t % DP;
        const long long i = i0 + r;
        sx[k][r] = (i < n && k < d) ? x[i * d + k] : 0.f;
    }
    __syncthreads();
    if (j >= m) return;
    float yj[DP];
#pragma unroll
    for (int k = 0; k < DP; ++k) yj[k] = k < d ? y[j * d + k] : 0.f;
    const int rows = (int)min(32LL, n - i0);
#pragma unroll
    for (int r = 0; r < 32; r += 4) {
        float2 a01 = make_float2(0.f, 0.f), a23 = a01;
#pragma unroll
        for (int k = 0; k < DP; ++k) {
            const float4 xv = *reinterpret_cast<const float4 *>(&sx[k][r]);
            const float2 yy = make_float2(yj[k], yj[k]);
            const float2 t01 = sub2(make_float2(xv.x, xv.y), yy), t23 = sub2(make_float2(xv.z, xv.w), yy);
            a01 = fma2(t01, t01, a01);
            a23 = fma2(t23, t23, a23);
        }
        float *out = C + (i0 + r) * m + j;
        if (r + 0 < rows) out[0] = a01.x;
        if (r + 1 < rows) out[m] = a01.y;
        if (r + 2 < rows) out[2 * m] = a23.x;
        if (r + 3 < rows) out[3 * m] = a23.y;
    }
}

// d in (64, 256]: the same per-lane fmaf chains (k in order), y taken 32 coordinates at a time
// into registers and the 32 rows' sums kept across the chunks
template <int DP>
__global__ void __launch_bounds__(256) k_build_cost_wide(const float *__restrict__ x, const float *__restrict__ y,
                                                         long long n, long long m, int d, float *C) {
    __shared__ __align__(16) float sx[DP][32];
    const long long i0 = (long long)blockIdx.y * 32;
    const long long j = (long long)blockIdx.x * 256 + threadIdx.x;
    for (int t = threadIdx.x; t < 32 * DP; t += 256) {
        const int r = t / DP, k = t % DP;
        const long long i = i0 + r;
        sx[k][r] = (i < n && k < d) ? x[i * d + k] : 0.f;
    }
    __syncthreads();
    if (j >= m) return;
    float2 acc[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) acc[r] = make_float2(0.f, 0.f);
    for (int kc = 0; kc < DP; kc += 32) {
        float yj[32];
#pragma unroll
        for (int kk = 0; kk < 32; ++kk) yj[kk] = kc + kk < d ? y[j * d + kc + kk] : 0.f;
#pragma unroll
        for (int r = 0; r < 32; r += 4) {
#pragma unroll
            for (int kk = 0; kk < 32; ++kk) {
                const float4 xv = *reinterpret_cast<const float4 *>(&sx[kc + kk][r]);
                const float2 yy = make_float2(yj[kk], yj[kk]);
                const float2 t01 = sub2(make_float2(xv.x, xv.y), yy), t23 = sub2(make_float2(xv.z, xv.w), yy);
                acc[r / 2] = fma2(t01, t01, acc[r / 2]);
                acc[r / 2 + 1] = fma2(t23, t23, acc[r / 2 + 1]);
            }
        }
    }
    const int rows = (int)min(32LL, n - i0);
#pragma unroll
    for (int r = 0; r < 32; r += 2) {
        float *out = C + (i0 + r) * m + j;
        if (r < rows) out[0] = acc[r / 2].x;
        if (r + 1 < rows) out[m] = acc[r / 2].y;
    }
}

cudaError_t launch_build_cost(const float *x, const float *y, long long n, long long m, int d, float *C,
                              cudaStream_t st) {
    dim3 grid((unsigned)((m + 255) / 256), (unsigned)((n + 31) / 32));
    if (d <= 4) k_build_cost<4><<<grid, 256, 0, st>>>(x, y, n, m, d, C);
    else if (d <= 8) k_build_cost<8><<<grid, 256, 0, st>>>(x, y, n, m, d, C);
    else if (d <= 16) k_build_cost<16><<<grid, 256, 0, st>>>(x, y, n, m, d, C);
    else if (d <= 32) k_build_cost<32><<<grid, 256, 0, st>>>(x, y, n, m, d, C);
    else if (d <= 64) k_build_cost<64><<<grid, 256, 0, st>>>(x, y, n, m, d, C);
    else if (d <= 128) k_build_cost_wide<128><<<grid, 256, 0, st>>>(x, y, n, m, d, C);
    else if (d <= 256) k_build_cost_wide<256><<<grid, 256, 0, st>>>(x, y, n, m, d, C);
    else return cudaErrorInvalidValue;
    return cudaGetLastError();
}

__device__ __forceinline__ float4 ldg_stream(const float4 *p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}

// ------------------------------------------------------------------ K5r
// One warp per row; each lane handles float4 groups j4 = lane + 32 t; 4 groups per step.
__global__ void __launch_bounds__(256) k_rows(StoredPass S) {
    if (S.stop && *(volatile const int *)S.stop) return;
    const long long row = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= S.n) return;
    const float kap = kLog2e / S.eps;
    const float4 *Cr = reinterpret_cast<const float4 *>(S.C + row * S.m);
    const float4 *W = reinterpret_cast<const float4 *>(S.wq);
    const long long m4 = S.m >> 2;
    float M = -INFINITY, Sx = 0.f, Sy = 0.f;
    long long j4 = lane;
    for (; j4 + 96 < m4; j4 += 128) {
        float4 c[4], w[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) c[u] = ldg_stream(Cr + j4 + 32 * u);
#pragma unroll
        for (int u = 0; u < 4; ++u) w[u] = __ldg(W + j4 + 32 * u);
        float t[16];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            t[4 * u + 0] = fmaf(c[u].x, -kap, w[u].x);
            t[4 * u + 1] = fmaf(c[u].y, -kap, w[u].y);
            t[4 * u + 2] = fmaf(c[u].z, -kap, w[u].z);
            t[4 * u + 3] = fmaf(c[u].w, -kap, w[u].w);
        }
        float cm = t[0];
#pragma unroll
        for (int q = 1; q < 16; ++q) cm = fmaxf(cm, t[q]);
        if (cm > M) {
            const float sc = ex2(M - cm);
            Sx *= sc; Sy *= sc; M = cm;
        }
#pragma unroll
        for (int q = 0; q < 16; q += 2) {
            Sx += ex2(t[q] - M);
            Sy += ex2(t[q + 1] - M);
        }
    }
    for (; j4 < m4; j4 += 32) {
        const float4 c = ldg_stream(Cr + j4), w = __ldg(W + j4);
        const float t0 = fmaf(c.x, -kap, w.x), t1 = fmaf(c.y, -kap, w.y),
                    t2 = fmaf(c.z, -kap, w.z), t3 = fmaf(c.w, -kap, w.w);
        const float cm = fmaxf(fmaxf(t0, t1), fmaxf(t2, t3));
        if (cm > M) { const float sc = ex2(M - cm); Sx *= sc; Sy *= sc; M = cm; }
        Sx += ex2(t0 - M) + ex2(t2 - M);
        Sy += ex2(t1 - M) + ex2(t3 - M);
    }
    for (long long j = (m4 << 2) + lane; j < S.m; j += 32) {  // scalar tail (m % 4)
        const float t = fmaf(S.C[row * S.m + j], -kap, S.wq[j]);
        if (t > M) { const float sc = ex2(M - t); Sx *= sc; Sy *= sc; M = t; }
        Sx += ex2(t - M);
    }
    float Sv = Sx + Sy;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float M2 = __shfl_xor_sync(0xffffffffu, M, o);
        const float S2 = __shfl_xor_sync(0xffffffffu, Sv, o);
        lse_merge(M, Sv, M2, S2);
    }
    if (lane == 0) S.part[row] = make_float2(M, Sv);
}

cudaError_t launch_stored_rows(const StoredPass &S, cudaStream_t st) {
    if (S.m % 4) return cudaErrorInvalidValue;  // float4 rows need m % 4 == 0 (checked by the API)
    k_rows<<<(unsigned)((S.n + 7) / 8), 256, 0, st>>>(S);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ K5c
constexpr int kCT = 128;  // threads; 4 columns each -> 512 columns per CTA
__global__ void __launch_bounds__(kCT) k_cols(StoredPass S) {
    if (S.stop && *(volatile const int *)S.stop) return;
    if (S.only_if && !*(volatile const int *)S.only_if) return;
    const long long j0 = ((long long)blockIdx.x * kCT + threadIdx.x) * 4;
    const int s = blockIdx.y;
    const int bq = s / S.split_q, u = s % S.split_q;
    const long long bs = S.blk_rows > 0 ? S.blk_rows : S.n;
    const long long b0 = bq * bs, nb = max(0LL, min(bs, S.n - b0));
    const long long r0 = b0 + nb * u / S.split_q, r1 = b0 + nb * (u + 1) / S.split_q;
    const float kap = kLog2e / S.eps;
    float M[4], Sx[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) { M[c] = -INFINITY; Sx[c] = 0.f; }
    const bool ok = j0 < S.m;
    long long i = r0;
    for (; i + 8 <= r1; i += 8) {
        float4 c[8];
        float w[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            c[u] = ok ? ldg_stream(reinterpret_cast<const float4 *>(S.C + (i + u) * S.m + j0))
                      : make_float4(0.f, 0.f, 0.f, 0.f);
            w[u] = __ldg(S.wq + i + u);
        }
        float t[4][8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            t[0][u] = fmaf(c[u].x, -kap, w[u]);
            t[1][u] = fmaf(c[u].y, -kap, w[u]);
            t[2][u] = fmaf(c[u].z, -kap, w[u]);
            t[3][u] = fmaf(c[u].w, -kap, w[u]);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            float cm = t[q][0];
#pragma unroll
            for (int u = 1; u < 8; ++u) cm = fmaxf(cm, t[q][u]);
            if (cm > M[q]) { Sx[q] *= ex2(M[q] - cm); M[q] = cm; }
            float a0 = 0.f, a1 = 0.f;
#pragma unroll
            for (int u = 0; u < 8; u += 2) { a0 += ex2(t[q][u] - M[q]); a1 += ex2(t[q][u + 1] - M[q]); }
            Sx[q] += a0 + a1;
        }
    }
    for (; i < r1; ++i) {
        const float4 c = ok ? ldg_stream(reinterpret_cast<const float4 *>(S.C + i * S.m + j0))
                            : make_float4(0.f, 0.f, 0.f, 0.f);
        const float w = __ldg(S.wq + i);
        const float tv[4] = {fmaf(c.x, -kap, w), fmaf(c.y, -kap, w), fmaf(c.z, -kap, w), fmaf(c.w, -kap, w)};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (tv[q] > M[q]) { Sx[q] *= ex2(M[q] - tv[q]); M[q] = tv[q]; }
            Sx[q] += ex2(tv[q] - M[q]);
        }
    }
    if (!ok) return;
#pragma unroll
    for (int q = 0; q < 4; ++q)
        if (j0 + q < S.m) S.part[(long long)s * S.m + j0 + q] = make_float2(M[q], Sx[q]);
}

cudaError_t launch_stored_cols(const StoredPass &S, cudaStream_t st) {
    if (S.m % 4) return cudaErrorInvalidValue;
    dim3 grid((unsigned)((S.m + kCT * 4 - 1) / (kCT * 4)), (unsigned)(S.nblk * S.split_q));
    k_cols<<<grid, kCT, 0, st>>>(S);
    return cudaGetLastError();
}

}  // namespace sk

namespace sk {

// ------------------------------------------------------------------ K5 fused
// One HBM read of C per sweep, one exponential per cost entry.
// CTA s owns the rows of split s (same fixed block structure as k_cols); thread t owns the
// columns of float4 groups t, t + 512, ... (CPT columns) in both phases, so every value it
// needs stays in registers.  Rows stream HBM -> shared memory through a ring of whole-row
// buffers (1D bulk TMA, mbarrier complete_tx), refilled as soon as a row is in registers.
// Per row i (log2 units, kappa = log2(e)/eps, t_ij = g_j kappa - C_ij kappa):
//   row:    e_ij = 2^(t_ij - sigma_i), S_i = sum_j e_ij (fixed reduction tree), with the shift
//           sigma_i = the row's previous LSE + 4 (validated: S_i in [2^-100, 2^100]; otherwise,
//           and in the first sweep, the exact row maximum);  lse_i = sigma_i + log2 S_i,
//           f_i = eps log a_i - eps ln2 lse_i (Alg. 1 l.4), w_i = f_i kappa;
//   column: the next g-update needs sum_i 2^((f_i - C_ij) kappa)
//             = 2^(-g_j kappa) sum_i e_ij 2^(sigma_i + w_i)          (the Sinkhorn scaling
//           identity P = diag(u) K diag(v)), so A_j += e_ij v_i with v_i = 2^(sigma_i + w_i),
//           the same exponential serving both passes.  sum_j A_j = sum_i a_i, so A_j cannot
//           overflow; a column whose total mass leaves [2^-100, 2^100] (an unmatched column
//           early in a solve) is caught by the merge, which redoes the column pass exactly.
// Output partial (M, S) = (-g_j kappa, A_j) for the standard merge (all M equal).
// Deterministic: fixed reduction tree per row, sequential row order per column.
constexpr int kFT = 512;
constexpr int kFW = kFT / 32;            // warps
constexpr int kFRingBytes = 3 * 65536;   // row ring (3 rows of m = 16384)
constexpr float kFusedSeedMargin = 4.f;

struct FusedArgs {
    const float *C; long long n, m;
    float eps;
    const float *gw;        // g log2(e)/eps (Y side D = 0 pack), m
    const float *xc;        // eps log a_i (X side c), n
    float *xpot[2];         // X potential buffers (parity = iteration)
    float *xw;              // X side w pack (f log2(e)/eps), n
    float *xlse;            // per-row LSE seeds (in/out), n
    float2 *part;           // column partials [nblk * split_q][m]
    long long blk_rows;
    int split_q, stages;
    DevStatus *st;
    int sharded, no_iter_inc;
};

__device__ __forceinline__ float warp_sum_tree(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Row LSE of one staged row (all threads of the CTA; uniform control flow): t receives
// e_j = 2^(t_j - sig) for this thread's columns, S = sum_j e_j over the row (fixed tree), with
// sig = seed + margin when that keeps S in [2^-100, 2^100], else the exact row maximum.
template <int CPT, int FT = kFT, class W>
__device__ __forceinline__ void fused_row_lse(const float4 *row4, int m4, float kap, const W &w,
                                              float seed, float (&t)[CPT], float *red, float *redm, float &sig,
                                              float &S) {
    constexpr int G = CPT / 4;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int q = 0; q < G; ++q) {
        const int g = threadIdx.x + q * FT;
        const float4 c = g < m4 ? row4[g] : make_float4(0.f, 0.f, 0.f, 0.f);
        t[4 * q] = fmaf(c.x, -kap, w(4 * q)); t[4 * q + 1] = fmaf(c.y, -kap, w(4 * q + 1));
        t[4 * q + 2] = fmaf(c.z, -kap, w(4 * q + 2)); t[4 * q + 3] = fmaf(c.w, -kap, w(4 * q + 3));
    }
    sig = seed + kFusedSeedMargin;
    S = 0.f;
    bool exact = !isfinite(seed);
    if (!exact) {
        float p = 0.f;
#pragma unroll
        for (int c = 0; c < CPT; ++c) { t[c] = ex2(t[c] - sig); p += t[c]; }   // t now holds e
        p = warp_sum_tree(p);
        if (lane == 0) red[warp] = p;
        __syncthreads();
#pragma unroll
        for (int x = 0; x < FT / 32; ++x) S += red[x];
        exact = !(S >= 0x1p-100f && S <= 0x1p100f);
        if (exact) {   // rare: rebuild t from the row (still in shared memory until refilled)
#pragma unroll
            for (int q = 0; q < G; ++q) {
                const int g = threadIdx.x + q * FT;
                const float4 c = g < m4 ? row4[g] : make_float4(0.f, 0.f, 0.f, 0.f);
                t[4 * q] = fmaf(c.x, -kap, w(4 * q)); t[4 * q + 1] = fmaf(c.y, -kap, w(4 * q + 1));
                t[4 * q + 2] = fmaf(c.z, -kap, w(4 * q + 2)); t[4 * q + 3] = fmaf(c.w, -kap, w(4 * q + 3));
            }
        }
    }
    if (exact) {   // exact maximum as the shift (first sweep, or the seed was off)
        float mx = -INFINITY;
#pragma unroll
        for (int c = 0; c < CPT; ++c) mx = fmaxf(mx, t[c]);
        mx = warp_max(mx);
        if (lane == 0) redm[warp] = mx;
        __syncthreads();
        sig = -INFINITY;
#pragma unroll
        for (int x = 0; x < FT / 32; ++x) sig = fmaxf(sig, redm[x]);
        float p = 0.f;
#pragma unroll
        for (int c = 0; c < CPT; ++c) { t[c] = ex2(t[c] - sig); p += t[c]; }
        p = warp_sum_tree(p);
        if (lane == 0) red[warp] = p;
        __syncthreads();
        S = 0.f;
#pragma unroll
        for (int x = 0; x < FT / 32; ++x) S += red[x];
    }
}

template <int CPT>
__global__ void __launch_bounds__(kFT, 1) k_stored_fused(FusedArgs A) {
    constexpr int G = CPT / 4;                     // float4 groups per thread
    extern __shared__ __align__(128) float ring[];   // stages x m floats
    __shared__ __align__(8) uint64_t full[8];
    __shared__ float red[2][kFW], redm[kFW];
    __shared__ int s_last;
    if (*(volatile const int *)&A.st->stop) return;
    const int l = A.st->iter;                      // producing f^{l+1}
    float *fnew = ((l + 1) & 1) ? A.xpot[1] : A.xpot[0];   // no dynamic param indexing
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float kap = kLog2e / A.eps, epsln2 = A.eps * kLn2;
    const int s = blockIdx.x;
    const int bq = s / A.split_q, u = s % A.split_q;
    const long long bs = A.blk_rows > 0 ? A.blk_rows : A.n;
    const long long b0 = bq * bs, nb = max(0LL, min(bs, A.n - b0));
    const long long r0 = b0 + nb * u / A.split_q, r1 = b0 + nb * (u + 1) / A.split_q;
    const int m = (int)A.m, m4 = m >> 2;
    const int NS = A.stages;
    const uint32_t rowb = (uint32_t)m * 4u;

    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) mbar_init(&full[i], 1);
        fence_mbar_init();
        for (int k = 0; k < NS && r0 + k < r1; ++k) {
            mbar_expect_tx(&full[k], rowb);
            bulk_g2s(ring + (size_t)k * m, A.C + (r0 + k) * A.m, rowb, &full[k]);
        }
    }
    __syncthreads();

    // this thread's columns: w_j = g_j kappa (-inf padding) and the column accumulators
    float w[CPT], acc[CPT];
    const float4 *Gw = reinterpret_cast<const float4 *>(A.gw);
#pragma unroll
    for (int q = 0; q < G; ++q) {
        const int g = threadIdx.x + q * kFT;
        const float4 v = g < m4 ? __ldg(Gw + g) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
        w[4 * q] = v.x; w[4 * q + 1] = v.y; w[4 * q + 2] = v.z; w[4 * q + 3] = v.w;
    }
#pragma unroll
    for (int c = 0; c < CPT; ++c) acc[c] = 0.f;
    int bad = 0;   // non-finite f in this CTA's rows (thread 0)

    for (long long i = r0; i < r1; ++i) {
        const int k = (int)(i - r0);
        const int st = k % NS;
        const float4 *row4 = reinterpret_cast<const float4 *>(ring + (size_t)st * m);
        const float seed = A.xlse[i];
        mbar_wait(&full[st], (k / NS) & 1);
        float t[CPT], sig, S;
        fused_row_lse<CPT>(row4, m4, kap, [&](int c) { return w[c]; }, seed, t, red[k & 1], redm, sig, S);
        const float lse = sig + log2f(S);
        const float fn = A.xc[i] - epsln2 * lse;
        const float wv = fn * kap;
        if (threadIdx.x == 0) {
            fnew[i] = fn;
            bad |= !isfinite(fn);
            A.xw[i] = wv;
            A.xlse[i] = lse;
            // every thread has row i in registers (a barrier passed since): refill its slot
            const long long nx = i + NS;
            if (nx < r1) {
                fence_proxy_async();
                mbar_expect_tx(&full[st], rowb);
                bulk_g2s(ring + (size_t)st * m, A.C + nx * A.m, rowb, &full[st]);
            }
        }
        // ---- column partials with the same exponentials
        const float v = ex2(sig + wv);
#pragma unroll
        for (int c = 0; c < CPT; ++c) acc[c] = fmaf(t[c], v, acc[c]);
    }
#pragma unroll
    for (int q = 0; q < G; ++q) {
        const int g = threadIdx.x + q * kFT;
        if (g < m4) {
#pragma unroll
            for (int e = 0; e < 4; ++e)
                A.part[(long long)s * A.m + 4 * g + e] = make_float2(-w[4 * q + e], acc[4 * q + e]);
        }
    }
    // row bookkeeping (what MERGE_ROW does for the separate passes): the last CTA advances the
    // sweep counter, or stops on a non-finite f (unsharded; sharded ranks rely on the column merge)
    if (threadIdx.x == 0) {
        if (bad) atomicOr(&A.st->nonfinite, 2);   // bit 1: pending, promoted below
        __threadfence();
        s_last = atomicAdd(&A.st->ticket_row, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (threadIdx.x == 0 && s_last) {
        __threadfence();
        DevStatus *st = A.st;
        st->ticket_row = 0;
        const int nf = *(volatile int *)&st->nonfinite;
        if ((nf & 2) && !A.sharded) { st->nonfinite = 1; st->stop = 1; st->final_iter = l; }
        else {
            st->nonfinite = nf & 1;
            if (!A.no_iter_inc) st->iter = l + 1;
        }
        __threadfence();
    }
}

bool stored_fused_supported(long long m) { return m % 4 == 0 && m >= 4 && m <= (long long)kFT * 32; }

cudaError_t launch_stored_fused(const FusedLaunch &L, cudaStream_t st) {
    FusedArgs A;
    A.C = L.C; A.n = L.n; A.m = L.m; A.eps = L.eps; A.gw = L.gw; A.xc = L.xc;
    A.xpot[0] = L.xpot[0]; A.xpot[1] = L.xpot[1]; A.xw = L.xw; A.xlse = L.xlse; A.part = L.part;
    A.blk_rows = L.blk_rows; A.split_q = L.split_q; A.st = L.st;
    A.sharded = L.sharded; A.no_iter_inc = L.no_iter_inc;
    if (!stored_fused_supported(L.m) || !L.xlse) return cudaErrorInvalidValue;
    // ring depth: as many whole rows as fit (2 .. 8)
    const long long rb = L.m * 4;
    A.stages = (int)std::min<long long>(8, kFRingBytes / rb);
    const size_t smem = (size_t)A.stages * rb;
    const int grid = L.nblk * L.split_q;
    const long long cpt = (L.m / 4 + kFT - 1) / kFT * 4;
    cudaError_t e = cudaSuccess;
#define SK_FUSED_LAUNCH(CP)                                                                                   \
    {                                                                                                         \
        e = cudaFuncSetAttribute(k_stored_fused<CP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        if (e != cudaSuccess) return e;                                                                       \
        k_stored_fused<CP><<<grid, kFT, smem, st>>>(A);                                                       \
    }
    if (cpt <= 4) SK_FUSED_LAUNCH(4)
    else if (cpt <= 8) SK_FUSED_LAUNCH(8)
    else if (cpt <= 16) SK_FUSED_LAUNCH(16)
    else if (cpt <= 32) SK_FUSED_LAUNCH(32)
    else return cudaErrorInvalidValue;
#undef SK_FUSED_LAUNCH
    return cudaGetLastError();
}

}  // namespace sk
