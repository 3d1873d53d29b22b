// sk_online.cu — the multi-kernel online-cost Sinkhorn path for large problems.
//
//  K1 pack_side   : per point |p|^2, eps log w_p + |p|^2 and the tile-packed
//                   operand [coords | w] with w = (h - |p|^2) log2(e)/eps.
//  K2 k_lse<D,R>  : one LSE pass (row pass for f, column pass for g; Alg. 1
//                   l.4-5 with reading R-1): for every output point p, the
//                   (max, sum 2^(t - max)) partial over one split of the other
//                   side, t = w_q + <2 log2(e)/eps p, q>; the q tiles stream
//                   global -> shared through a 4-stage 1D bulk-TMA ring with
//                   mbarrier completion; the cross term is packed FFMA2, the
//                   exponentials MUFU.EX2 (sk_lse_tile.cuh).
//  K6 k_merge     : stable LSE merge of the split partials in fixed order ->
//                   new potential (+ packed w for the next pass), the fused
//                   marginal error err_l = sum_j b_j |expm1((g^l - g^{l+1})/eps)|
//                   (H5; threshold appendix), non-finite
//                   detection and the stop flag, decided by the last block.
//  K7 k_report    : E = <f,a> + <g,b> - eps sum(a) (Eq. 2 right after an
//                   f-update, H6) in fp64.
#include "sk_internal.h"
#include "sk_lse_tile.cuh"

#include <cstdlib>

namespace sk {

constexpr int kLT = 128;      // LSE kernel threads
constexpr int kStages = 4;    // bulk-copy ring depth
constexpr int kLseEmu = 1;
constexpr int kWideTQ = 32;   // D > 64: reduction points per tile
constexpr int kWideStages = 2;    // exp2 pairs (of 4 per chunk) on the FMA pipe when D <= 4

int lse_dpad(int d) {
    if (d <= 4) return d < 1 ? 0 : d;
    if (d <= 8) return 8;
    if (d <= 16) return 16;
    if (d <= 32) return 32;
    if (d <= 64) return 64;
    if (d <= 128) return 128;
    if (d <= 256) return 256;
    return 0;
}

int lse_tq(int D) { return D <= 4 ? 256 : (D <= 16 ? 128 : (D <= 64 ? 64 : kWideTQ)); }

template <int D> constexpr int kR = D <= 4 ? 4 : (D <= 16 ? 2 : 1);

// ------------------------------------------------------------------- K1
__global__ void k_pack_side(Side S, const float *__restrict__ pts, const float *__restrict__ wts,
                            float logw_const, const float *__restrict__ pot0, float eps, int mode) {
    const long long tiles = lse_tiles(S.P, S.tq);
    const long long total = tiles * S.tq;
    const float kap = kLog2e / eps;
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < total;
         p += (long long)gridDim.x * blockDim.x) {
        const long long t = p / S.tq, o = p % S.tq;
        float *tile = S.pack + t * (long long)(S.D + 1) * S.tq;
        if (p < S.P) {
            float s = 0.f;
            for (int k = 0; k < S.D; ++k) {
                const float v = k < S.d ? pts[p * S.d + k] : 0.f;
                tile[k * S.tq + o] = v;
                s = fmaf(v, v, s);
            }
            if (mode == PACK_TC)
                for (int k = 0; k < S.d; ++k) s = fmaf(pts[p * S.d + k], pts[p * S.d + k], s);
            if (mode == PACK_STORED) s = 0.f;  // stored cost: no |p|^2 folding
            const float lw = wts ? logf(wts[p]) : logw_const;
            S.c[p] = fmaf(eps, lw, s);
            S.nk[p] = s * kap;
            const float h = pot0 ? pot0[p] : 0.f;
            S.pot[0][p] = h;
            if (S.lse) S.lse[p] = -INFINITY;
            tile[S.D * S.tq + o] = fmaf(h, kap, -s * kap);
        } else {
            for (int k = 0; k < S.D; ++k) tile[k * S.tq + o] = 0.f;
            tile[S.D * S.tq + o] = -INFINITY;
        }
    }
}

cudaError_t pack_side(const Side &S, const float *pts, const float *wts, float logw_const,
                      const float *pot0, float eps, cudaStream_t st, int mode) {
    const long long total = lse_tiles(S.P, S.tq) * S.tq;
    int blocks = (int)((total + 255) / 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (mode < 0) mode = S.D == 0 ? PACK_STORED : PACK_ONLINE;
    k_pack_side<<<blocks, 256, 0, st>>>(S, pts, wts, logw_const, pot0, eps, mode);
    return cudaGetLastError();
}

// ------------------------------------------------------------------- K2
struct LseArgs {
    const float *Ppack; int P; int Ptq;
    const float *Qpack; int Qtiles;
    int blk_tiles, split_q;
    float2 *part;
    float tk;
    const int *stop;
    const int *only_if;     // run only if *only_if != 0 (nullable)
    const float *seed;      // SEEDED: P side last LSE
    float margin;           // SEEDED: shift = seed + margin (log2 units)
    float2 *xchg;           // non-null: the last CTA of each (P tile, block) merges the block's
    int *cnt;               //   split_q partials into xchg [nblk][P] (K6a fused); cnt [nblk][P tiles]
    int ptiles;             // P tiles (the 1D grid of the fused premerge)
};


// K6a: one point's block partial from its split_q sub-split partials src[u * P], merged in split
// order (L2 loads: other CTAs wrote them)
__device__ __forceinline__ float2 premerge_point(const float2 *src, int split_q, long long P) {
    float M = -INFINITY;
    for (int u = 0; u < split_q; ++u) M = fmaxf(M, __ldcg(src + u * P).x);
    float S = 0.f;
    for (int u = 0; u < split_q; ++u) {
        const float2 v = __ldcg(src + u * P);
        if (v.x != -INFINITY) S = fmaf(v.y, ex2(v.x - M), S);
    }
    return make_float2(M, S);
}

// The same merge (the same max, the same fmaf order) with all partials in flight at once: one L2
// round trip instead of 2 x split_q dependent ones.  For the standalone premerge kernel only (its
// 64 extra registers would cut K2's occupancy if inlined into the fused premerge).
__device__ __forceinline__ float2 premerge_point_r(const float2 *src, int split_q, long long P) {
    if (split_q > 32) return premerge_point(src, split_q, P);
    float2 v[32];
#pragma unroll
    for (int u = 0; u < 32; ++u) v[u] = u < split_q ? __ldcg(src + u * P) : make_float2(-INFINITY, 0.f);
    float M = -INFINITY;
#pragma unroll
    for (int u = 0; u < 32; ++u) M = fmaxf(M, v[u].x);
    float S = 0.f;
#pragma unroll
    for (int u = 0; u < 32; ++u)
        if (u < split_q && v[u].x != -INFINITY) S = fmaf(v[u].y, ex2(v[u].x - M), S);
    return make_float2(M, S);
}

// K2 item of this CTA: P tile px and Q range [t0, t0 + nt) of split s -> block b, sub-split u.
// 2D grid (P tiles, splits); with the fused premerge a 1D grid with the sub-split fastest, so
// that a (P tile, block)'s split_q CTAs run back to back and their partials are merged (and
// discarded) from L2
__device__ __forceinline__ void lse_item(const LseArgs &A, int &s, int &px, int &b, int &t0, int &nt) {
    if (A.xchg) {
        const int id = blockIdx.x, uu = id % A.split_q, rr = id / A.split_q;
        px = rr % A.ptiles;
        s = (rr / A.ptiles) * A.split_q + uu;
    } else {
        s = blockIdx.y;
        px = blockIdx.x;
    }
    b = s / A.split_q;
    const int u = s % A.split_q;
    const int bt = A.blk_tiles > 0 ? A.blk_tiles : A.Qtiles;
    const int base = b * bt;
    const int nt_b = max(0, min(bt, A.Qtiles - base));
    t0 = base + (int)((long long)nt_b * u / A.split_q);
    nt = base + (int)((long long)nt_b * (u + 1) / A.split_q) - t0;
}

// K2 tail: the CTA's split partials, then (fused K6a) the block premerge by the last CTA of
// each (P tile, block)
// (act: this thread owns output points - threadIdx.x < kLT; the others only join the barriers)
template <int R>
__device__ __forceinline__ void lse_store(const LseArgs &A, int s, int b, int px, const float (&M)[R],
                                          const float2 (&Sx)[R], bool act = true) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int p = px * (kLT * R) + r * kLT + threadIdx.x;
        if (act && p < A.P) A.part[(long long)s * A.P + p] = make_float2(M[r], Sx[r].x + Sx[r].y);
    }
    if (A.xchg) {
        // K6a fused: the last of the block's split_q CTAs for this P tile merges their partials in
        // split order (the premerge arithmetic) while they are still in L2, and writes the block
        // partial - the exchange payload - directly
        __shared__ int s_last;
        __threadfence();
        __syncthreads();
        int *c = A.cnt + (long long)b * A.ptiles + px;
        if (threadIdx.x == 0) s_last = atomicAdd(c, 1) == A.split_q - 1;
        __syncthreads();
        if (!s_last) return;
        __threadfence();
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int p = px * (kLT * R) + r * kLT + threadIdx.x;
            if (act && p < A.P) A.xchg[(long long)b * A.P + p] = premerge_point(A.part + (long long)b * A.split_q * A.P + p,
                                                                               A.split_q, A.P);
        }
        if (threadIdx.x == 0) *c = 0;   // (ready for the next launch)
        // the group's sub-split partials are dead: drop their L2 lines without writing them back
        // (only whole 128-byte lines inside the group's partial rows)
        // (per sub-split row: the whole 128-byte lines inside [p0, p1) - rows start anywhere)
        __syncthreads();
        const int p0 = px * kLT * R, p1 = min(A.P, p0 + kLT * R);
        for (int uu = 0; uu < A.split_q; ++uu) {
            const float2 *rowp = A.part + ((long long)b * A.split_q + uu) * A.P;
            const unsigned long long a0 = (reinterpret_cast<unsigned long long>(rowp + p0) + 127ull) & ~127ull;
            const unsigned long long a1 = reinterpret_cast<unsigned long long>(rowp + p1) & ~127ull;
            if (act)
                for (unsigned long long a = a0 + 128ull * threadIdx.x; a < a1; a += 128ull * kLT)
                    asm volatile("discard.global.L2 [%0], 128;" ::"l"(a) : "memory");
        }
    }
}

// EMU8: exponential pairs (of every 8 pairs = 2 chunks) evaluated on the FMA pipe in the
// seeded pass (D <= 4); balances MUFU against the FMA pipe (measured by SK_LSE_EMU8 sweeps)
template <int D, int R, bool SEEDED, int EMU8 = 2>
__global__ void __launch_bounds__(kLT) k_lse(LseArgs A) {
    constexpr int TQ = D <= 4 ? 256 : (D <= 16 ? 128 : 64);
    constexpr int TF = (D + 1) * TQ;  // floats per tile
    extern __shared__ __align__(128) float ring[];  // [kStages][TF]
    __shared__ __align__(8) uint64_t full[kStages];
    if (A.stop && *(volatile const int *)A.stop) return;
    if (A.only_if && !*(volatile const int *)A.only_if) return;

    int s, px, b, t0, nt;
    lse_item(A, s, px, b, t0, nt);

    // ---- output points: R per thread
    float2 pd[R][D];
    float M[R];
    float2 Sx[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int p = px * (kLT * R) + r * kLT + threadIdx.x;
        const int pt = p / A.Ptq, po = p % A.Ptq;
        const float *tile = A.Ppack + (long long)pt * (D + 1) * A.Ptq;
#pragma unroll
        for (int k = 0; k < D; ++k) {
            const float v = p < A.P ? tile[k * A.Ptq + po] * A.tk : 0.f;
            pd[r][k] = make_float2(v, v);
        }
        M[r] = (SEEDED && p < A.P) ? A.seed[p] + A.margin : -INFINITY;
        Sx[r] = make_float2(0.f, 0.f);
    }

    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i) mbar_init(&full[i], 1);
        fence_mbar_init();
        for (int i = 0; i < kStages && i < nt; ++i) {
            mbar_expect_tx(&full[i], TF * 4);
            bulk_g2s(ring + i * TF, A.Qpack + (long long)(t0 + i) * TF, TF * 4, &full[i]);
        }
    }
    __syncthreads();

    for (int i = 0; i < nt; ++i) {
        const int st = i % kStages;
        mbar_wait(&full[st], (i / kStages) & 1);
        const float *qt = ring + st * TF;
#pragma unroll 2
        if (SEEDED) {
            for (int q = 0; q < TQ; q += 2 * kChunk) {
                lse_chunk_seeded<D, R, (D <= 4 ? (EMU8 + 1) / 2 : 0)>(qt, TQ, qt + D * TQ, q, pd, M, Sx);
                lse_chunk_seeded<D, R, (D <= 4 ? EMU8 / 2 : 0)>(qt, TQ, qt + D * TQ, q + kChunk, pd, M, Sx);
            }
        } else {
            for (int q = 0; q < TQ; q += kChunk) lse_chunk<D, R, (D <= 4 ? kLseEmu : 0)>(qt, TQ, qt + D * TQ, q, pd, M, Sx);
        }
        __syncthreads();  // everyone is done with stage st
        if (threadIdx.x == 0 && i + kStages < nt) {
            fence_proxy_async();
            mbar_expect_tx(&full[st], TF * 4);
            bulk_g2s(ring + st * TF, A.Qpack + (long long)(t0 + i + kStages) * TF, TF * 4, &full[st]);
        }
    }

    lse_store<R>(A, s, b, px, M, Sx);
}

// D in {128, 256} (d in (64, 256]): the output points' scaled coordinates do not fit registers;
// they are staged once in shared memory as [D/4][kLT][4] (four consecutive coordinates of a point
// in one 16-byte word).  Register tiles: thread (pg, qg) of 32 x 8 takes the points pg + 32 r
// (r < 4) and the reduction points 4 qg .. 4 qg + 3 of every 32-point tile, so four coordinates
// of four points and of four reduction points (eight 128-bit shared loads, the latter broadcast
// across the warp) feed 64 FFMAs.  Each thread keeps a running (max, sum) per point over its
// share of the reduction points; the eight shares of a point are merged in qg order at the end.
// Always unseeded (exact running max per tile); the partials and the fused premerge are K2's.
// Large problems with d > 64 run on the tensor cores (K3); this kernel serves small problems with
// the tensor cores off, coordinates outside the fp16 fold, and the subsample initializer's
// extension pass.
constexpr int kWideT = 2 * kLT;
template <int D>
__global__ void __launch_bounds__(kWideT) k_lse_wide(LseArgs A) {
    constexpr int TQ = kWideTQ, TF = (D + 1) * TQ;
    extern __shared__ __align__(128) float ring[];   // [kWideStages][TF], then sP [D/4][kLT][4]
    float *sP = ring + kWideStages * TF;
    __shared__ __align__(8) uint64_t full[kWideStages];
    __shared__ float2 share[8][kLT];
    if (A.stop && *(volatile const int *)A.stop) return;
    if (A.only_if && !*(volatile const int *)A.only_if) return;
    int s, px, b, t0, nt;
    lse_item(A, s, px, b, t0, nt);
    const int pg = threadIdx.x & 31, qg = threadIdx.x >> 5;
    for (int e = threadIdx.x; e < D * kLT; e += kWideT) {
        const int k = e / kLT, q = e % kLT;
        const int p = px * kLT + q;
        const int pt = p / A.Ptq, po = p % A.Ptq;
        sP[((k >> 2) * kLT + q) * 4 + (k & 3)] =
            p < A.P ? A.Ppack[(long long)pt * (D + 1) * A.Ptq + k * A.Ptq + po] * A.tk : 0.f;
    }
    if (threadIdx.x == 0) {
        for (int i = 0; i < kWideStages; ++i) mbar_init(&full[i], 1);
        fence_mbar_init();
        for (int i = 0; i < kWideStages && i < nt; ++i) {
            mbar_expect_tx(&full[i], TF * 4);
            bulk_g2s(ring + i * TF, A.Qpack + (long long)(t0 + i) * TF, TF * 4, &full[i]);
        }
    }
    __syncthreads();
    float M[4], S[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) { M[r] = -INFINITY; S[r] = 0.f; }
    const float4 *sP4 = reinterpret_cast<const float4 *>(sP);
    for (int i = 0; i < nt; ++i) {
        const int st = i % kWideStages;
        mbar_wait(&full[st], (i / kWideStages) & 1);
        const float *qt = ring + st * TF + 4 * qg;
        float t[4][4];
        {
            const float4 w = *reinterpret_cast<const float4 *>(qt + D * TQ);
#pragma unroll
            for (int r = 0; r < 4; ++r) { t[r][0] = w.x; t[r][1] = w.y; t[r][2] = w.z; t[r][3] = w.w; }
        }
#pragma unroll 2
        for (int k4 = 0; k4 < D / 4; ++k4) {
            float4 pv[4], c[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) pv[r] = sP4[k4 * kLT + pg + 32 * r];
#pragma unroll
            for (int u = 0; u < 4; ++u) c[u] = *reinterpret_cast<const float4 *>(qt + (4 * k4 + u) * TQ);
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const float pk[4] = {pv[r].x, pv[r].y, pv[r].z, pv[r].w};
                float2 a = make_float2(t[r][0], t[r][1]), bq = make_float2(t[r][2], t[r][3]);
#pragma unroll
                for (int u = 0; u < 4; ++u) {   // coordinate 4 k4 + u, in k order per entry (FFMA2)
                    const float2 pp = make_float2(pk[u], pk[u]);
                    a = fma2(pp, make_float2(c[u].x, c[u].y), a);
                    bq = fma2(pp, make_float2(c[u].z, c[u].w), bq);
                }
                t[r][0] = a.x; t[r][1] = a.y; t[r][2] = bq.x; t[r][3] = bq.y;
            }
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const float cm = fmaxf(fmaxf(t[r][0], t[r][1]), fmaxf(t[r][2], t[r][3]));
            if (cm > M[r]) { S[r] *= ex2(M[r] - cm); M[r] = cm; }
            if (M[r] != -INFINITY)   // (four padding points keep M = -inf)
                S[r] += (ex2(t[r][0] - M[r]) + ex2(t[r][1] - M[r])) + (ex2(t[r][2] - M[r]) + ex2(t[r][3] - M[r]));
        }
        __syncthreads();  // everyone is done with stage st
        if (threadIdx.x == 0 && i + kWideStages < nt) {
            fence_proxy_async();
            mbar_expect_tx(&full[st], TF * 4);
            bulk_g2s(ring + st * TF, A.Qpack + (long long)(t0 + i + kWideStages) * TF, TF * 4, &full[st]);
        }
    }
    // point q's eight shares (qg = 0 .. 7) merged in qg order by thread q
#pragma unroll
    for (int r = 0; r < 4; ++r) share[qg][pg + 32 * r] = make_float2(M[r], S[r]);
    __syncthreads();
    float Mo[1] = {-INFINITY};
    float2 So[1] = {make_float2(0.f, 0.f)};
    const bool act = threadIdx.x < kLT;
    if (act) {
        float m = -INFINITY;
#pragma unroll
        for (int g = 0; g < 8; ++g) m = fmaxf(m, share[g][threadIdx.x].x);
        float sum = 0.f;
        if (m != -INFINITY)
#pragma unroll
            for (int g = 0; g < 8; ++g) {
                const float2 v = share[g][threadIdx.x];
                if (v.x != -INFINITY) sum = fmaf(v.y, ex2(v.x - m), sum);
            }
        Mo[0] = m;
        So[0] = make_float2(sum, 0.f);
    }
    lse_store<1>(A, s, b, px, Mo, So, act);
}

template <int D>
constexpr size_t wide_smem() { return (size_t)(kWideStages * (D + 1) * kWideTQ + D * kLT) * sizeof(float); }

template <int D>
static cudaError_t launch_lse_wide(const LsePass &L, cudaStream_t st) {
    const size_t smem = wide_smem<D>();
    cudaError_t e = cudaFuncSetAttribute(k_lse_wide<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    LseArgs A;
    A.Ppack = L.Pside->pack; A.P = L.Pside->P; A.Ptq = L.Pside->tq;
    A.Qpack = L.Qside->pack; A.Qtiles = (int)lse_tiles(L.Qside->P, L.Qside->tq);
    A.blk_tiles = L.blk_tiles; A.split_q = L.split_q;
    A.part = L.part;
    A.tk = 2.f * kLog2e / L.eps;
    A.stop = L.stop;
    A.only_if = L.only_if;
    A.seed = nullptr;
    A.margin = 0.f;
    A.xchg = L.xchg;
    A.cnt = L.cnt;
    A.ptiles = (A.P + kLT - 1) / kLT;
    dim3 grid(A.ptiles, L.nblk * L.split_q);
    if (A.xchg) grid = dim3((unsigned)A.ptiles * L.nblk * L.split_q, 1);
    k_lse_wide<D><<<grid, kWideT, smem, st>>>(A);
    return cudaGetLastError();
}

template <int D, int R>
static cudaError_t launch_lse_dr(const LsePass &L, cudaStream_t st) {
    constexpr int TQ = D <= 4 ? 256 : (D <= 16 ? 128 : 64);
    const size_t smem = (size_t)kStages * (D + 1) * TQ * sizeof(float);
    cudaError_t e = cudaFuncSetAttribute(k_lse<D, R, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    const int emu8 = L.emu8;
    auto seeded_fn = emu8 == 0 ? k_lse<D, R, true, 0> : (emu8 == 1 ? k_lse<D, R, true, 1> : k_lse<D, R, true, 2>);
    e = cudaFuncSetAttribute(seeded_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    LseArgs A;
    A.Ppack = L.Pside->pack; A.P = L.Pside->P; A.Ptq = L.Pside->tq;
    A.Qpack = L.Qside->pack; A.Qtiles = (int)lse_tiles(L.Qside->P, L.Qside->tq);
    A.blk_tiles = L.blk_tiles; A.split_q = L.split_q;
    A.part = L.part;
    A.tk = 2.f * kLog2e / L.eps;
    A.stop = L.stop;
    A.only_if = L.only_if;
    A.seed = L.Pside->lse;
    A.margin = L.margin;
    A.xchg = L.xchg;
    A.cnt = L.cnt;
    A.ptiles = (A.P + kLT * R - 1) / (kLT * R);
    dim3 grid(A.ptiles, L.nblk * L.split_q);
    if (A.xchg) grid = dim3((unsigned)A.ptiles * L.nblk * L.split_q, 1);
    if (L.seeded && A.seed) seeded_fn<<<grid, kLT, smem, st>>>(A);
    else k_lse<D, R, false><<<grid, kLT, smem, st>>>(A);
    return cudaGetLastError();
}

// R: output points per thread (small problems: one, so that their few P tiles still fill the
// SMs; a point's sum does not depend on R - only the split structure fixes the order)
template <int D>
static cudaError_t launch_lse_d(const LsePass &L, cudaStream_t st) {
    if constexpr (kR<D> > 1)
        if (L.R == 1) return launch_lse_dr<D, 1>(L, st);
    return launch_lse_dr<D, kR<D>>(L, st);
}

cudaError_t launch_lse(const LsePass &L, cudaStream_t st) {
    switch (L.Pside->D) {
        case 1: return launch_lse_d<1>(L, st);
        case 2: return launch_lse_d<2>(L, st);
        case 3: return launch_lse_d<3>(L, st);
        case 4: return launch_lse_d<4>(L, st);
        case 8: return launch_lse_d<8>(L, st);
        case 16: return launch_lse_d<16>(L, st);
        case 32: return launch_lse_d<32>(L, st);
        case 64: return launch_lse_d<64>(L, st);
        case 128: return launch_lse_wide<128>(L, st);
        case 256: return launch_lse_wide<256>(L, st);
        default: return cudaErrorInvalidValue;
    }
}

template <int D, int R = kR<D>>
static int occ_d() {
    constexpr int TQ = D <= 4 ? 256 : (D <= 16 ? 128 : 64);
    const size_t smem = (size_t)kStages * (D + 1) * TQ * sizeof(float);
    cudaFuncSetAttribute(k_lse<D, R, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_lse<D, R, false>, kLT, smem) != cudaSuccess) n = 1;
    return n > 0 ? n : 1;
}

template <int D>
static int occ_wide() {
    const size_t smem = wide_smem<D>();
    cudaFuncSetAttribute(k_lse_wide<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_lse_wide<D>, kWideT, smem) != cudaSuccess) n = 1;
    return n > 0 ? n : 1;
}

int lse_occupancy_ctas(int D, int R) {
    if (R == 1 && D <= 4) {
        switch (D) {
            case 1: return occ_d<1, 1>();
            case 2: return occ_d<2, 1>();
            case 3: return occ_d<3, 1>();
            default: return occ_d<4, 1>();
        }
    }
    switch (D) {
        case 1: return occ_d<1>();
        case 2: return occ_d<2>();
        case 3: return occ_d<3>();
        case 4: return occ_d<4>();
        case 8: return occ_d<8>();
        case 16: return occ_d<16>();
        case 32: return occ_d<32>();
        case 64: return occ_d<64>();
        case 128: return occ_wide<128>();
        case 256: return occ_wide<256>();
        default: return 1;
    }
}

// ------------------------------------------------------------------- K6
constexpr int kMT = 256;
int merge_blocks(int P) {
    int b = (P + kMT - 1) / kMT;
    return b < 1 ? 1 : (b > kMergeMaxBlocks ? kMergeMaxBlocks : b);
}

// Exact (online max) LSE of output point p of side S over every point of side Q, from the
// packed tiles (coordinates + w): the fallback of a seeded pass.
__device__ void exact_lse_point(const Side &S, const Side &Q, int p, float eps, float &M, float &Ssum) {
    const float tk = 2.f * kLog2e / eps;
    if (S.D == 0) {
        // tensor-core pass (PACK_TC): coordinates from the caller's fp32 arrays, w from the plain
        // [P] array (tiles of tq points, no coordinates)
        M = -INFINITY;
        Ssum = 0.f;
        const float *pp = S.raw + (long long)p * S.d;
        for (long long q = 0; q < Q.P; ++q) {
            const float *qq = Q.raw + q * Q.d;
            float dot = 0.f;
            for (int k = 0; k < S.d; ++k) dot = fmaf(pp[k], qq[k], dot);
            const float v = fmaf(dot, tk, Q.pack[q]);
            if (v > M) { Ssum = Ssum * ex2(M - v); M = v; }
            Ssum += ex2(v - M);
        }
        return;
    }
    const long long pt = p / S.tq, po = p % S.tq;
    const float *ptile = S.pack + pt * (long long)(S.D + 1) * S.tq;
    M = -INFINITY;
    Ssum = 0.f;
    const long long qt = lse_tiles(Q.P, Q.tq);
    for (long long t = 0; t < qt; ++t) {
        const float *tile = Q.pack + t * (long long)(Q.D + 1) * Q.tq;
        for (int o = 0; o < Q.tq; ++o) {
            float v = tile[Q.D * Q.tq + o];
            if (v == -INFINITY) continue;
            for (int k = 0; k < Q.D; ++k) v = fmaf(ptile[k * S.tq + po] * tk, tile[k * Q.tq + o], v);
            if (v > M) { Ssum = Ssum * ex2(M - v); M = v; }
            Ssum += ex2(v - M);
        }
    }
}

// Merge of point p given its (M, Ssum) over all splits: new potential (+ packed w), fused
// error term, non-finite and column-range flags.
__device__ __forceinline__ void merge_point(const MergePass &Mp, const Side &S, const Side &Qs, int p, float M, float Ssum,
                                            bool check, float om, bool rterms, const float *hold, float *hnew,
                                            double &e, double &e2, int &bad) {
    const float eps = Mp.eps, kap = kLog2e / eps, epsln2 = eps * kLn2;
    const double wu = 1.0 / (double)(Mp.n_uniform > 0 ? Mp.n_uniform : S.P);   // uniform weight
    if (Mp.range_redo && !(Ssum >= 0x1p-100f && Ssum <= 0x1p100f)) {
        // seeded column pass: the fixed shift was far from this column's true maximum.  The exact
        // pass is redone for every column (k_lse / k_lse_tc2 + premerge + merge, gated on
        // st->colfail) so that every partition of the rows takes the same path.
        bad |= 2;
        return;
    }
    if (Mp.Q && !(Ssum >= 0x1p-100f && Ssum <= 0x1p100f)) {
        // seeded pass: the fixed shift was far from the true maximum -> exact recompute of
        // this point over the whole reduced side (rare; one thread, online max)
        exact_lse_point(S, Qs, p, eps, M, Ssum);   // (Mp.Q is a host pointer: only a flag here)
    }
    if (Mp.scaled && !(Ssum >= 0x1p-100f && Ssum <= 0x1p100f)) {
        // fused stored sweep: the scaled column mass left the safe range (an almost unmatched
        // column).  Unsharded: exact online LSE of column p over all rows of the stored C here;
        // sharded (rows on other ranks): the column pass is redone exactly (k_cols + merge,
        // gated on st->colfail).
        if (!Mp.Cst) { bad |= 2; return; }
        const float kap = kLog2e / Mp.eps;
        M = -INFINITY;
        Ssum = 0.f;
        for (long long i = 0; i < Mp.n_rows; ++i) {
            const float t = fmaf(Mp.Cst[i * S.P + p], -kap, Mp.xw[i]);
            if (t > M) { Ssum = Ssum * ex2(M - t); M = t; }
            Ssum += ex2(t - M);
        }
    }
    const float lse2 = M + log2f(Ssum);
    if (S.lse) S.lse[p] = lse2;
    if (Mp.mode == MERGE_OUT) {
        const float v = Mp.out_const + (S.c[p] - epsln2 * lse2);
        Mp.out[p] = v;
        bad |= !isfinite(v);
        return;
    }
    const float hsk = S.c[p] - epsln2 * lse2;   // the Sinkhorn (omega = 1) update
    // Alg. 1 with relaxation (R-1): h <- (1 - omega) h_old + omega h_sk
    const float hn = om == 1.f ? hsk : fmaf(om, hsk - hold[p], hold[p]);
    hnew[p] = hn;
    if (rterms && Mp.mode == MERGE_ROW) {
        // rows are no longer exact after a relaxed f-update: sum_j P_ij = a_i exp((f_i - fsk_i)/eps)
        const double ai = Mp.wts ? (double)Mp.wts[p] : wu;
        const double dv = (double)expm1f((hn - hsk) / eps);
        e += ai * fabs(dv);
        e2 += ai * dv;
    }
    const long long t = p / S.tq, o = p % S.tq;
    const float wn = fmaf(hn, kap, -S.nk[p]);
    S.pack[t * (long long)(S.D + 1) * S.tq + (long long)S.D * S.tq + o] = wn;
    if (S.tcimg) {   // K3 side: w into the B-role extra columns, the next row shift into the A role
        tc_put_w(S.tcimg, S.P, p, wn, S.tc_c, S.tc_rb);
        if (Mp.tc_fold) tc_put_shift(S.tcimg, S.P, p, lse2 + Mp.tc_margin, S.tc_c, S.tc_rb);
    }
    bad |= !isfinite(hn);
    if (Mp.anderson && Mp.mode == MERGE_ROW) {   // row term of err_l for (f^l, g~): columns are exact
        const double ai = Mp.wts ? (double)Mp.wts[p] : wu;
        e += ai * fabs((double)expm1f((hold[p] - hsk) / eps));
    }
    if (check) {
        const double bj = Mp.wts ? (double)Mp.wts[p] : wu;
        e += bj * fabs((double)expm1f((hold[p] - hsk) / eps));   // column term of err_l (H5)
    }
}

constexpr int kWideMax = 32;      // splits per warp in the WIDE merge (nsplit <= 8 * 32)

// WIDE (many splits): 32 points per block step; warp w reduces splits w, w + 8, ... of the 32
// points (coalesced rows of the partial array), the 8 warp partials are combined in a fixed
// order by warp 0 (max first, then the rescaled sums) — deterministic.
template <bool WIDE>
__global__ void __launch_bounds__(kMT) k_merge(MergePass Mp, Side S, Side Qs) {
    __shared__ double red[kMT / 32];
    __shared__ int redi[kMT / 32];
    __shared__ int s_last;
    __shared__ double red2[kMT / 32];
    __shared__ float wM[kMT / 32][32], wS[kMT / 32][32];
    DevStatus *st = Mp.st;
    if (st && *(volatile int *)&st->stop) return;
    if (Mp.only_if && !*(volatile const int *)Mp.only_if) return;
    const int l = st ? st->iter : 0;
    const bool check = Mp.mode == MERGE_COL && !Mp.anderson && l >= 1 &&
                       (l % st->check_every == 0 || l == st->max_iter);
    // adaptive momentum (R-31): err_l also at the end of every window; omega of this sweep from
    // the status (rewritten only by the last block of a row merge, after every block has read it)
    const bool chk_ad = Mp.mode == MERGE_COL && Mp.adapt > 0 && l >= 1 && l % Mp.adapt == 0;
    const float om = (st && Mp.adapt > 0) ? st->omega : Mp.omega;
    const bool rterms = Mp.adapt > 0 || Mp.omega != 1.f;
    const float *hold = (l & 1) ? S.pot[1] : S.pot[0];      // no dynamic param indexing
    float *hnew = (l & 1) ? S.pot[0] : S.pot[1];
    double e = 0.0, e2 = 0.0;
    int bad = 0;
    if (WIDE) {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        constexpr int NW = kMT / 32;
        for (int pb = blockIdx.x * 32; pb < S.P; pb += gridDim.x * 32) {
            const int p = pb + lane;
            // this warp's splits, all loads in flight at once (kWideMax per warp), kept for pass 2
            float2 v[kWideMax];
#pragma unroll
            for (int q = 0; q < kWideMax; ++q) {
                const int s = warp + q * NW;
                v[q] = (p < S.P && s < Mp.nsplit) ? Mp.part[(long long)s * S.P + p] : make_float2(-INFINITY, 0.f);
            }
            float M = -INFINITY;
#pragma unroll
            for (int q = 0; q < kWideMax; ++q) M = fmaxf(M, v[q].x);
            wM[warp][lane] = M;
            __syncthreads();
            M = wM[0][lane];
#pragma unroll
            for (int w = 1; w < NW; ++w) M = fmaxf(M, wM[w][lane]);
            float Ssum = 0.f;
#pragma unroll
            for (int q = 0; q < kWideMax; ++q)
                if (v[q].x != -INFINITY) Ssum += v[q].y * ex2(v[q].x - M);
            wS[warp][lane] = Ssum;
            __syncthreads();
            if (warp == 0 && p < S.P) {
                Ssum = wS[0][lane];
#pragma unroll
                for (int w = 1; w < NW; ++w) Ssum += wS[w][lane];
                if (Mp.precomputed) bad |= !isfinite(hnew[p]);
                else merge_point(Mp, S, Qs, p, M, Ssum, check || chk_ad, om, rterms, hold, hnew, e, e2, bad);
            }
            __syncthreads();
        }
    } else {
        for (int p = blockIdx.x * kMT + threadIdx.x; p < S.P; p += gridDim.x * kMT) {
            if (Mp.precomputed) {  // fused stored sweep wrote f and w; only check finiteness
                bad |= !isfinite(hnew[p]);
                continue;
            }
            float M = -INFINITY;
            float Ssum = 0.f;
            if (Mp.nsplit <= 16) {   // (all partials in flight at once; the same arithmetic)
                float2 v[16];
#pragma unroll
                for (int s = 0; s < 16; ++s)
                    v[s] = s < Mp.nsplit ? Mp.part[(long long)s * S.P + p] : make_float2(-INFINITY, 0.f);
#pragma unroll
                for (int s = 0; s < 16; ++s) M = fmaxf(M, v[s].x);
#pragma unroll
                for (int s = 0; s < 16; ++s)
                    if (s < Mp.nsplit && v[s].x != -INFINITY) Ssum += v[s].y * ex2(v[s].x - M);
            } else {
                for (int s = 0; s < Mp.nsplit; ++s) M = fmaxf(M, Mp.part[(long long)s * S.P + p].x);
                for (int s = 0; s < Mp.nsplit; ++s) {
                    const float2 v = Mp.part[(long long)s * S.P + p];
                    if (v.x != -INFINITY) Ssum += v.y * ex2(v.x - M);
                }
            }
            merge_point(Mp, S, Qs, p, M, Ssum, check || chk_ad, om, rterms, hold, hnew, e, e2, bad);
        }
    }
    if (!st) return;
    // block partials -> last block decides (fixed order => deterministic)
    for (int o = 16; o > 0; o >>= 1) {
        e += __shfl_xor_sync(0xffffffffu, e, o);
        e2 += __shfl_xor_sync(0xffffffffu, e2, o);
        bad |= __shfl_xor_sync(0xffffffffu, bad, o);
    }
    if ((threadIdx.x & 31) == 0) { red[threadIdx.x >> 5] = e; red2[threadIdx.x >> 5] = e2; redi[threadIdx.x >> 5] = bad; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double be = 0.0, be2 = 0.0; int bb = 0;
        for (int w = 0; w < kMT / 32; ++w) { be += red[w]; be2 += red2[w]; bb |= redi[w]; }
        Mp.blk_err[blockIdx.x] = be;
        Mp.blk_err[kMergeMaxBlocks + blockIdx.x] = be2;
        Mp.blk_bad[blockIdx.x] = bb;
        __threadfence();
        unsigned *tk = Mp.mode == MERGE_COL ? &st->ticket_col : &st->ticket_row;
        s_last = atomicAdd(tk, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // the last block sums the block partials: thread t takes blocks t, t + 256, ... in order,
    // then a fixed tree (lanes by xor, the 8 warps in order) - deterministic, and parallel (a
    // serial sum over ~1000 blocks by one thread took tens of microseconds)
    double et = 0.0, et2 = 0.0; int bt = 0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += kMT) {
        et += __ldcg(Mp.blk_err + i);
        et2 += __ldcg(Mp.blk_err + kMergeMaxBlocks + i);
        bt |= __ldcg(Mp.blk_bad + i);
    }
    for (int o = 16; o > 0; o >>= 1) {
        et += __shfl_xor_sync(0xffffffffu, et, o);
        et2 += __shfl_xor_sync(0xffffffffu, et2, o);
        bt |= __shfl_xor_sync(0xffffffffu, bt, o);
    }
    __syncthreads();   // (red / red2 / redi reused)
    if ((threadIdx.x & 31) == 0) { red[threadIdx.x >> 5] = et; red2[threadIdx.x >> 5] = et2; redi[threadIdx.x >> 5] = bt; }
    __syncthreads();
    if (threadIdx.x != 0) return;
    et = 0.0; et2 = 0.0; bt = 0;
    for (int w = 0; w < kMT / 32; ++w) { et += red[w]; et2 += red2[w]; bt |= redi[w]; }
    if (Mp.mode == MERGE_COL) {
        st->ticket_col = 0;
        if (bt & 2) { st->colfail = 1; __threadfence(); return; }   // decisions left to the exact redo
        if (Mp.only_if) st->colfail = 0;
        if (bt) {
            st->nonfinite = 1;
            st->stop = 1;
            if (Mp.anderson) {
                // g~ = g_sk(f^l) is the non-finite one: (f^{l-1}, g~_{l-1}) are still in their
                // buffers (sweep l wrote the other ones); at l = 0, (f^0, g^0 = 0)
                if (l >= 1) st->final_iter = l - 1;
                else { st->final_iter = 0; st->g_off = 0; }
            } else {
                // sharded: f^l may be the non-finite one (rows are not checked locally), so fall
                // back to (f^{l-1}, g^{l-1}), both finite
                st->final_iter = Mp.sharded ? max(l - 1, 0) : l;
            }
        } else if (check || chk_ad) {
            if (rterms) et += st->row_err;   // relaxed: the rows of (f^l, g^l) are off too
            const float en = (float)et;
            if (check) {
                st->err = en;
                if (en < st->tol) { st->converged = 1; st->stop = 1; st->final_iter = l; }
                else if (l >= st->max_iter) { st->stop = 1; st->final_iter = l; }
            }
            if (chk_ad) {   // a window ends at sweep l: omega from sweep l + 2 on (R-31)
                if (l >= 2 * Mp.adapt)
                    st->omega_next = adaptive_omega((double)en / (double)st->err_win, Mp.adapt, st->omega);
                st->err_win = en;
            }
        }
    } else if (Mp.mode == MERGE_ROW && Mp.anderson) {
        // Anderson: this slice's row term of err_l; K19's k_and_decide sums the slices (ranks),
        // decides and advances the sweep counter
        st->ticket_row = 0;
        *Mp.and_err = et;
        if (bt && !Mp.sharded) { st->nonfinite = 1; st->stop = 1; st->final_iter = l; }
    } else if (Mp.mode == MERGE_ROW) {
        st->ticket_row = 0;
        if (rterms) {   // (row shards: summed over the slices here, over ranks by an allreduce)
            if (Mp.accum) { st->row_err += et; st->mass_dev += et2; }
            else { st->row_err = et; st->mass_dev = et2; }
        }
        if (bt && !Mp.sharded) { st->nonfinite = 1; st->stop = 1; st->final_iter = l; }
        else if (!Mp.no_iter_inc) {
            st->iter = l + 1;
            if (Mp.adapt > 0) st->omega = st->omega_next;   // the next sweep's relaxation
        }
    } else {
        st->ticket_row = 0;
        if (bt) st->nonfinite = 1;
    }
    __threadfence();
}

constexpr int kWideSplits = 12;   // splits from which the merge uses the warp-per-split-group layout

cudaError_t launch_merge(const MergePass &M, cudaStream_t st) {
    const Side Qs = M.Q ? *M.Q : Side{};   // the reduced side by value (the fallback runs on the device)
    if (M.nsplit >= kWideSplits && M.nsplit <= kWideMax * (kMT / 32)) {
        int b = (M.S->P + 31) / 32;
        if (b > kMergeMaxBlocks) b = kMergeMaxBlocks;
        k_merge<true><<<b, kMT, 0, st>>>(M, *M.S, Qs);
    } else {
        k_merge<false><<<merge_blocks(M.S->P), kMT, 0, st>>>(M, *M.S, Qs);
    }
    return cudaGetLastError();
}

// ------------------------------------------------------------------- K6a
// One (M, S) per point per fixed row block from its split_q sub-split partials, merged in split
// order (the first step of the column pass's fixed merge tree; k_merge then merges the blocks in
// block order).  Sharded solves exchange exactly these block partials: 8 B per column per block.
__global__ void __launch_bounds__(256) k_premerge(const float2 *__restrict__ part, int nblk, int split_q,
                                                  long long P, float2 *__restrict__ out, const int *stop,
                                                  const int *only_if) {
    if (stop && *(volatile const int *)stop) return;
    if (only_if && !*(volatile const int *)only_if) return;
    const long long total = (long long)nblk * P;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const long long b = t / P, p = t - b * P;
        out[t] = premerge_point_r(part + b * split_q * P + p, split_q, P);
    }
}

cudaError_t launch_premerge(const float2 *part, int nblk, int split_q, long long P, float2 *out, const int *stop,
                            const int *only_if, cudaStream_t st) {
    const long long total = (long long)nblk * P;
    long long b = (total + 255) / 256;
    if (b > 148 * 8) b = 148 * 8;
    k_premerge<<<(int)(b < 1 ? 1 : b), 256, 0, st>>>(part, nblk, split_q, P, out, stop, only_if);
    return cudaGetLastError();
}

// ------------------------------------------------------------------- K7
__global__ void __launch_bounds__(1024) k_report(Side X, Side Y, const float *a, const float *b,
                                                  float eps, DevStatus *st, int local_only,
                                                  long long n_uniform) {
    __shared__ double red[32];
    const int l = st->final_iter, lg = l + st->g_off;
    const float *f = (l & 1) ? X.pot[1] : X.pot[0], *g = (lg & 1) ? Y.pot[1] : Y.pot[0];
    double s = 0.0;
    if (!local_only)   // (local_only: <f,a> comes from k_report_blocks)
        for (int i = threadIdx.x; i < X.P; i += 1024) {
            const double ai = a ? (double)a[i] : 1.0 / n_uniform;
            s += (double)f[i] * ai - (double)eps * ai;
        }
    double s2 = 0.0;
    for (int j = threadIdx.x; j < Y.P; j += 1024) s2 += (double)g[j] * (b ? (double)b[j] : 1.0 / Y.P);
    const double fa = block_sum_d<1024>(s, red);
    const double gb = block_sum_d<1024>(s2, red);
    if (threadIdx.x == 0) {
        st->fa_local = fa;
        st->E = local_only ? gb : fa + gb;
    }
}

cudaError_t launch_report(const Side &X, const Side &Y, const float *a, const float *b, float eps,
                          DevStatus *st, int local_only, long long n_uniform, cudaStream_t s) {
    k_report<<<1, 1024, 0, s>>>(X, Y, a, b, eps, st, local_only, n_uniform);
    return cudaGetLastError();
}

__global__ void k_status_init(DevStatus *st, int max_iter, int check_every, float tol, int g_off, float omega0) {
    DevStatus z = {};
    z.g_off = g_off;
    z.omega = omega0;
    z.omega_next = omega0;
    z.max_iter = max_iter;
    z.check_every = check_every;
    z.tol = tol;
    z.err = INFINITY;
    *st = z;
}

// <f,a> - eps sum(a) per fixed row block (partition-invariant): block b of the global
// partition covers rows [b*bs, (b+1)*bs); this slice holds rows [row0, row0 + X.P).  CTA k
// reduces global block (row0 / bs + k) in a fixed order and writes out[block].
__global__ void __launch_bounds__(1024) k_report_blocks(Side X, const float *a, float eps, DevStatus *st,
                                                         long long n_uniform, long long row0, long long bs,
                                                         double *out) {
    __shared__ double red[32];
    const int l = st->final_iter;
    const float *f = (l & 1) ? X.pot[1] : X.pot[0];
    const long long b = row0 / bs + blockIdx.x;
    const long long lo = max(b * bs, row0) - row0, hi = min((b + 1) * bs, row0 + (long long)X.P) - row0;
    double s = 0.0;
    for (long long i = lo + threadIdx.x; i < hi; i += 1024) {
        const double ai = a ? (double)a[i] : 1.0 / n_uniform;
        s += (double)f[i] * ai - (double)eps * ai;
    }
    const double tot = block_sum_d<1024>(s, red);
    if (threadIdx.x == 0) out[b] = tot;
}

cudaError_t launch_report_blocks(const Side &X, const float *a, float eps, DevStatus *st, long long n_uniform,
                                 long long row0, long long bs, double *out, cudaStream_t s) {
    const long long b0 = row0 / bs, b1 = (row0 + X.P - 1) / bs;
    k_report_blocks<<<(unsigned)(b1 - b0 + 1), 1024, 0, s>>>(X, a, eps, st, n_uniform, row0, bs, out);
    return cudaGetLastError();
}

cudaError_t launch_status_init(DevStatus *st, int max_iter, int check_every, float tol,
                               cudaStream_t s, int g_off, float omega0) {
    k_status_init<<<1, 1, 0, s>>>(st, max_iter, check_every, tol, g_off, omega0);
    return cudaGetLastError();
}

// ------------------------------------------------------------ misc kernels
__global__ void k_fill(float *p, long long n, float v) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        p[i] = v;
}

cudaError_t launch_fill(float *p, long long n, float v, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    long long b = (n + 255) / 256;
    k_fill<<<(int)(b > 4096 ? 4096 : b), 256, 0, st>>>(p, n, v);
    return cudaGetLastError();
}

__global__ void k_check(const float *p, long long n, int *flag, int positive) {
    int bad = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const float v = p[i];
        bad |= !isfinite(v) || (positive && !(v > 0.f));
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// All of a call's input checks in one launch: entry e covers [off_e, off_e + n_e) of the
// concatenated index range (finite, or finite and > 0).
__global__ void k_check_multi(CheckList L, int *flag) {
    int bad = 0;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < L.total;
         t += (long long)gridDim.x * blockDim.x) {
        int e = 0;
        long long o = t;
        while (o >= L.n[e]) { o -= L.n[e]; ++e; }
        const float v = L.p[e][o];
        bad |= !isfinite(v) || (L.positive[e] && !(v > 0.f));
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

cudaError_t launch_check_multi(const CheckList &L, int *flag, cudaStream_t st) {
    if (L.total <= 0) return cudaSuccess;
    long long b = (L.total + 255) / 256;
    k_check_multi<<<(int)(b > 2048 ? 2048 : b), 256, 0, st>>>(L, flag);
    return cudaGetLastError();
}

cudaError_t launch_check_finite(const float *p, long long n, int *flag, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    long long b = (n + 255) / 256;
    k_check<<<(int)(b > 2048 ? 2048 : b), 256, 0, st>>>(p, n, flag, 0);
    return cudaGetLastError();
}

cudaError_t launch_check_positive(const float *p, long long n, int *flag, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    long long b = (n + 255) / 256;
    k_check<<<(int)(b > 2048 ? 2048 : b), 256, 0, st>>>(p, n, flag, 1);
    return cudaGetLastError();
}

__global__ void k_gather(const float *src, const int *idx, long long cnt, int d, float *dst) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < cnt * d;
         t += (long long)gridDim.x * blockDim.x) {
        const long long r = t / d, k = t % d;
        dst[t] = src[(long long)idx[r] * d + k];
    }
}

cudaError_t launch_gather_rows(const float *src, const int *idx, long long cnt, int d, float *dst,
                               cudaStream_t st) {
    long long b = (cnt * d + 255) / 256;
    k_gather<<<(int)(b > 4096 ? 4096 : (b < 1 ? 1 : b)), 256, 0, st>>>(src, idx, cnt, d, dst);
    return cudaGetLastError();
}

// indices in range and distinct: mark[idx] counting via atomics on an int scratch of size n
__global__ void k_check_idx(const int *idx, long long cnt, long long n, int *flag, int *mark) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < cnt;
         t += (long long)gridDim.x * blockDim.x) {
        const int v = idx[t];
        if (v < 0 || v >= n) { atomicOr(flag, 1); continue; }
        if (atomicAdd(&mark[v], 1) != 0) atomicOr(flag, 2);
    }
}

cudaError_t launch_check_indices(const int *idx, long long cnt, long long n, int *flag, int *scratch,
                                 cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(scratch, 0, sizeof(int) * n, st);
    if (e != cudaSuccess) return e;
    long long b = (cnt + 255) / 256;
    k_check_idx<<<(int)(b > 4096 ? 4096 : (b < 1 ? 1 : b)), 256, 0, st>>>(idx, cnt, n, flag, scratch);
    return cudaGetLastError();
}

}  // namespace sk
