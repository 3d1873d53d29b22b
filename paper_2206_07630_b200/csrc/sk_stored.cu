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
#include "sk_internal.h"
#include "sk_common.cuh"

namespace sk {

// ------------------------------------------------------------------- K4
__global__ void __launch_bounds__(256) k_build_cost(const float *__restrict__ x, const float *__restrict__ y,
                                                    long long n, long long m, int d, float *C) {
    extern __shared__ float sxy[];  // [32][d] rows of x
    const long long i0 = (long long)blockIdx.y * 32;
    const long long j = (long long)blockIdx.x * 256 + threadIdx.x;
    for (int t = threadIdx.x; t < 32 * d; t += 256) {
        const long long i = i0 + t / d;
        sxy[t] = i < n ? x[i * d + t % d] : 0.f;
    }
    __syncthreads();
    if (j >= m) return;
    float yj[64];
#pragma unroll
    for (int k = 0; k < 64; ++k)
        if (k < d) yj[k] = y[j * d + k];
    for (int r = 0; r < 32 && i0 + r < n; ++r) {
        float s = 0.f;
#pragma unroll
        for (int k = 0; k < 64; ++k)
            if (k < d) {
                const float t = sxy[r * d + k] - yj[k];
                s = fmaf(t, t, s);
            }
        C[(i0 + r) * m + j] = s;
    }
}

cudaError_t launch_build_cost(const float *x, const float *y, long long n, long long m, int d, float *C,
                              cudaStream_t st) {
    if (d > 64) return cudaErrorInvalidValue;
    dim3 grid((unsigned)((m + 255) / 256), (unsigned)((n + 31) / 32));
    k_build_cost<<<grid, 256, 32 * d * sizeof(float), st>>>(x, y, n, m, d, C);
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
// One HBM read of C per sweep.  CTA s owns the rows of split s (same
// fixed block structure as k_cols) and, in registers, the (max, sum) state of every column:
// thread t owns the float4 groups t, t + 512, ... (CPT columns).  Per group of 4 rows:
//   phase A  warps 4r..4r+3 stream row r (a quarter each) from HBM: exact online
//            (max, sum) of t = g_j log2(e)/eps - C_ij log2(e)/eps, combined in fixed order
//            -> f_i = eps log a_i - eps ln2 (M + log2 S) (Alg. 1 l.4), written with its w;
//   phase B  every thread re-reads its columns of the 4 rows (L2 hits: the group was
//            bulk-prefetched into L2 one group ahead) and updates the column state with
//            t = f_i log2(e)/eps - C_ij log2(e)/eps (the partials of g^{l+2}, Alg. 1 l.5).
// Deterministic: fixed per-row quarter order, per-column sequential row order.
constexpr int kFT = 512;

struct FusedArgs {
    const float *C; long long n, m;
    float eps;
    const float *gw;        // g log2(e)/eps (Y side D = 0 pack), m
    const float *xc;        // eps log a_i (X side c), n
    float *xpot[2];         // X potential buffers (parity = iteration)
    float *xw;              // X side w pack (f log2(e)/eps), n
    float2 *part;           // column partials [nblk * split_q][m]
    long long blk_rows;
    int split_q;
    DevStatus *st;
};

__device__ __forceinline__ void prefetch_l2(const void *p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

constexpr int kFR = 2;                  // rows per group
constexpr int kFWR = (kFT / 32) / kFR;  // warps per row in phase A (8)

template <int CPT>
__global__ void __launch_bounds__(kFT, 1) k_stored_fused(FusedArgs A) {
    __shared__ float2 red[kFT / 32];
    __shared__ float wrow[kFR];
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
    const long long m4 = A.m >> 2;
    const float4 *Gw = reinterpret_cast<const float4 *>(A.gw);

    float cM[CPT], cS[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) { cM[c] = -INFINITY; cS[c] = 0.f; }

    // L2 prefetch two groups ahead (the TMA engine streams HBM while the warps compute)
    if (threadIdx.x == 0)
        for (long long i = r0; i < min(r1, r0 + 2 * kFR); ++i) prefetch_l2(A.C + i * A.m, (uint32_t)(A.m * 4));

    for (long long i0 = r0; i0 < r1; i0 += kFR) {
        const int rows = (int)min((long long)kFR, r1 - i0);
        if (threadIdx.x == 0)
            for (long long i = i0 + 2 * kFR; i < min(r1, i0 + 3 * kFR); ++i)
                prefetch_l2(A.C + i * A.m, (uint32_t)(A.m * 4));
        // ---- phase A: row r = warp / kFWR, segment q = warp % kFWR (exact online LSE)
        {
            const int r = warp / kFWR, q = warp % kFWR;
            float M = -INFINITY, S0 = 0.f, S1 = 0.f;
            if (r < rows) {
                const float4 *Cr = reinterpret_cast<const float4 *>(A.C + (i0 + r) * A.m);
                const long long g0 = m4 * q / kFWR, g1 = m4 * (q + 1) / kFWR;
                long long g = g0 + lane;
                for (; g + 96 < g1; g += 128) {
                    float4 c[4], w[4];
#pragma unroll
                    for (int v = 0; v < 4; ++v) c[v] = Cr[g + 32 * v];
#pragma unroll
                    for (int v = 0; v < 4; ++v) w[v] = __ldg(Gw + g + 32 * v);
                    float t[16];
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        t[4 * v + 0] = fmaf(c[v].x, -kap, w[v].x); t[4 * v + 1] = fmaf(c[v].y, -kap, w[v].y);
                        t[4 * v + 2] = fmaf(c[v].z, -kap, w[v].z); t[4 * v + 3] = fmaf(c[v].w, -kap, w[v].w);
                    }
                    float cm = t[0];
#pragma unroll
                    for (int v = 1; v < 16; ++v) cm = fmaxf(cm, t[v]);
                    if (cm > M) { const float sc = ex2(M - cm); S0 *= sc; S1 *= sc; M = cm; }
#pragma unroll
                    for (int v = 0; v < 16; v += 2) { S0 += ex2(t[v] - M); S1 += ex2(t[v + 1] - M); }
                }
                for (; g < g1; g += 32) {
                    const float4 c = Cr[g], w = __ldg(Gw + g);
                    const float t0 = fmaf(c.x, -kap, w.x), t1 = fmaf(c.y, -kap, w.y),
                                t2 = fmaf(c.z, -kap, w.z), t3 = fmaf(c.w, -kap, w.w);
                    const float cm = fmaxf(fmaxf(t0, t1), fmaxf(t2, t3));
                    if (cm > M) { const float sc = ex2(M - cm); S0 *= sc; S1 *= sc; M = cm; }
                    S0 += ex2(t0 - M) + ex2(t2 - M);
                    S1 += ex2(t1 - M) + ex2(t3 - M);
                }
            }
            float Sv = S0 + S1;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const float M2 = __shfl_xor_sync(0xffffffffu, M, o);
                const float S2 = __shfl_xor_sync(0xffffffffu, Sv, o);
                lse_merge(M, Sv, M2, S2);
            }
            if (lane == 0) red[warp] = make_float2(M, Sv);
        }
        __syncthreads();
        if (threadIdx.x < rows) {
            const int r = threadIdx.x;
            float M = red[kFWR * r].x, Sv = red[kFWR * r].y;
            for (int q = 1; q < kFWR; ++q) lse_merge(M, Sv, red[kFWR * r + q].x, red[kFWR * r + q].y);
            const long long i = i0 + r;
            const float fn = A.xc[i] - epsln2 * (M + log2f(Sv));
            fnew[i] = fn;
            const float wv = fn * kap;
            A.xw[i] = wv;
            wrow[r] = wv;
        }
        __syncthreads();
        // ---- phase B: column state over the rows of this group (L2 / L1 re-read)
        float wr[kFR];
#pragma unroll
        for (int r = 0; r < kFR; ++r) wr[r] = r < rows ? wrow[r] : -INFINITY;
#pragma unroll
        for (int k = 0; k < CPT / 4; ++k) {
            const long long g = threadIdx.x + (long long)k * kFT;
            if (g < m4) {
                float t[4][kFR];
#pragma unroll
                for (int r = 0; r < kFR; ++r) {
                    const long long rr = r < rows ? r : 0;   // duplicate row 0 as padding, masked by wr
                    const float4 c = *reinterpret_cast<const float4 *>(A.C + (i0 + rr) * A.m + 4 * g);
                    t[0][r] = fmaf(c.x, -kap, wr[r]); t[1][r] = fmaf(c.y, -kap, wr[r]);
                    t[2][r] = fmaf(c.z, -kap, wr[r]); t[3][r] = fmaf(c.w, -kap, wr[r]);
                }
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const float cm = fmaxf(t[c][0], t[c][1]);
                    if (cm > cM[4 * k + c]) { cS[4 * k + c] *= ex2(cM[4 * k + c] - cm); cM[4 * k + c] = cm; }
                    const float mm = cM[4 * k + c];
                    cS[4 * k + c] += ex2(t[c][0] - mm) + ex2(t[c][1] - mm);
                }
            }
        }
        __syncthreads();   // red / wrow reuse
    }
#pragma unroll
    for (int k = 0; k < CPT / 4; ++k) {
        const long long g = threadIdx.x + (long long)k * kFT;
        if (g < m4) {
#pragma unroll
            for (int c = 0; c < 4; ++c)
                A.part[(long long)s * A.m + 4 * g + c] = make_float2(cM[4 * k + c], cS[4 * k + c]);
        }
    }
}

bool stored_fused_supported(long long m) { return m % 4 == 0 && m <= (long long)kFT * 32; }

cudaError_t launch_stored_fused(const FusedLaunch &L, cudaStream_t st) {
    FusedArgs A;
    A.C = L.C; A.n = L.n; A.m = L.m; A.eps = L.eps; A.gw = L.gw; A.xc = L.xc;
    A.xpot[0] = L.xpot[0]; A.xpot[1] = L.xpot[1]; A.xw = L.xw; A.part = L.part;
    A.blk_rows = L.blk_rows; A.split_q = L.split_q; A.st = L.st;
    const int grid = L.nblk * L.split_q;
    const long long cpt = (L.m / 4 + kFT - 1) / kFT * 4;
    if (cpt <= 8) k_stored_fused<8><<<grid, kFT, 0, st>>>(A);
    else if (cpt <= 16) k_stored_fused<16><<<grid, kFT, 0, st>>>(A);
    else if (cpt <= 32) k_stored_fused<32><<<grid, kFT, 0, st>>>(A);
    else return cudaErrorInvalidValue;
    return cudaGetLastError();
}

}  // namespace sk
