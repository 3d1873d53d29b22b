// sk_lse_tile.cuh — the inner online log-sum-exp loop shared by the on-chip
// solver (K13) and the multi-kernel LSE pass (K2).
//
// For output points p (R per thread) and reduction points q it accumulates, in
// log2 units,
//     t_pq = w_q + <p~, q>,     p~ = 2 log2(e)/eps * p,
//     w_q  = (h_q - ||q||^2) * log2(e)/eps      (h = the other potential),
// i.e. t_pq = (h_q - C_pq) log2(e)/eps + ||p||^2 log2(e)/eps: the per-p constant
// ||p||^2 is folded out of the LSE and added back by the caller's finalize.
// State per p: running max M and sum S of 2^(t - M), updated once per chunk of 8
// q's (chunk max first, then one rescale only if the max grew).  The cross term
// uses packed FFMA2 over pairs of q; exponentials are MUFU.EX2.
#pragma once
#include "sk_common.cuh"

namespace sk {

constexpr int kChunk = 8;  // q's per online-max chunk (4 FFMA2 pairs)

// 2^x for x <= 0 on the FMA pipe (two lanes per instruction): Cody-Waite split
// x = n + r, n = rint(x) via the 1.5*2^23 magic add, r in [-1/2, 1/2]; 2^r by a degree-5
// near-minimax polynomial (max rel. error 2.1e-7 in fp32 Horner, on par with
// ex2.approx); 2^n by adding n to the exponent field.  Inputs below -125 are clamped
// (2^-125 is ~1e-38 relative to the chunk maximum, which is exactly 1).
__device__ __forceinline__ float2 ex2_emu2(float2 x) {
    x.x = fmaxf(x.x, -125.f);
    x.y = fmaxf(x.y, -125.f);
    const float2 magic = make_float2(12582912.f, 12582912.f);
    const float2 t = add2(x, magic);
    const float2 r = sub2(x, sub2(t, magic));
    float2 p = fma2(make_float2(1.32764654699713e-3f, 1.32764654699713e-3f), r,
                    make_float2(9.675540961325169e-3f, 9.675540961325169e-3f));
    p = fma2(p, r, make_float2(5.550713464617729e-2f, 5.550713464617729e-2f));
    p = fma2(p, r, make_float2(2.4022120237350464e-1f, 2.4022120237350464e-1f));
    p = fma2(p, r, make_float2(6.931469440460205e-1f, 6.931469440460205e-1f));
    p = fma2(p, r, make_float2(1.0000001192092896f, 1.0000001192092896f));
    // bits(t) << 23 == n << 23 (mod 2^32): the magic's own mantissa bit shifts out
    p.x = __int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23));
    p.y = __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23));
    return p;
}

// One chunk of 8 q's for R output points.  qc: coords [D][stride] (SoA), qw: w.
// EMU of the 4 exponential pairs go to the FMA pipe (ex2_emu2), the rest to MUFU.
template <int D, int R, int EMU = 0>
__device__ __forceinline__ void lse_chunk(const float *__restrict__ qc, int qstride,
                                          const float *__restrict__ qw, int q,
                                          const float2 (&pd)[R][D], float (&M)[R],
                                          float2 (&S)[R]) {
    float2 w[4], c[D][4];
    {
        const float4 w0 = *reinterpret_cast<const float4 *>(qw + q);
        const float4 w1 = *reinterpret_cast<const float4 *>(qw + q + 4);
        w[0] = make_float2(w0.x, w0.y); w[1] = make_float2(w0.z, w0.w);
        w[2] = make_float2(w1.x, w1.y); w[3] = make_float2(w1.z, w1.w);
    }
#pragma unroll
    for (int k = 0; k < D; ++k) {
        const float4 c0 = *reinterpret_cast<const float4 *>(qc + k * qstride + q);
        const float4 c1 = *reinterpret_cast<const float4 *>(qc + k * qstride + q + 4);
        c[k][0] = make_float2(c0.x, c0.y); c[k][1] = make_float2(c0.z, c0.w);
        c[k][2] = make_float2(c1.x, c1.y); c[k][3] = make_float2(c1.z, c1.w);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
        float2 t[4];
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
            t[jj] = w[jj];
#pragma unroll
            for (int k = 0; k < D; ++k) t[jj] = fma2(pd[r][k], c[k][jj], t[jj]);
        }
        float cm = fmaxf(fmaxf(fmaxf(t[0].x, t[0].y), fmaxf(t[1].x, t[1].y)),
                         fmaxf(fmaxf(t[2].x, t[2].y), fmaxf(t[3].x, t[3].y)));
        if (cm > M[r]) {  // rare after the first chunks
            const float sc = ex2(M[r] - cm);
            S[r].x *= sc;
            S[r].y *= sc;
            M[r] = cm;
        }
        const float2 mm = make_float2(M[r], M[r]);
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
            float2 e = sub2(t[jj], mm);
            if (jj >= 4 - EMU) {
                e = ex2_emu2(e);
            } else {
                e.x = ex2(e.x);
                e.y = ex2(e.y);
            }
            S[r] = add2(S[r], e);
        }
    }
}

// Seeded variant: the shift M is fixed for the whole pass (the point's previous LSE plus
// a margin), so no chunk max and no rescale are needed: S += 2^(t - M).  The caller
// validates S in [2^-100, 2^100] (no overflow, no underflow of the dominant terms) and
// recomputes the point with lse_chunk otherwise.  EMU of every 4 pairs go to FMA.
template <int D, int R, int EMU = 0>
__device__ __forceinline__ void lse_chunk_seeded(const float *__restrict__ qc, int qstride,
                                                 const float *__restrict__ qw, int q,
                                                 const float2 (&pd)[R][D], const float (&M)[R],
                                                 float2 (&S)[R]) {
    float2 w[4], c[D][4];
    {
        const float4 w0 = *reinterpret_cast<const float4 *>(qw + q);
        const float4 w1 = *reinterpret_cast<const float4 *>(qw + q + 4);
        w[0] = make_float2(w0.x, w0.y); w[1] = make_float2(w0.z, w0.w);
        w[2] = make_float2(w1.x, w1.y); w[3] = make_float2(w1.z, w1.w);
    }
#pragma unroll
    for (int k = 0; k < D; ++k) {
        const float4 c0 = *reinterpret_cast<const float4 *>(qc + k * qstride + q);
        const float4 c1 = *reinterpret_cast<const float4 *>(qc + k * qstride + q + 4);
        c[k][0] = make_float2(c0.x, c0.y); c[k][1] = make_float2(c0.z, c0.w);
        c[k][2] = make_float2(c1.x, c1.y); c[k][3] = make_float2(c1.z, c1.w);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const float2 mm = make_float2(M[r], M[r]);
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
            float2 t = sub2(w[jj], mm);
#pragma unroll
            for (int k = 0; k < D; ++k) t = fma2(pd[r][k], c[k][jj], t);
            if (jj >= 4 - EMU) {
                t = ex2_emu2(t);
            } else {
                t.x = ex2(t.x);
                t.y = ex2(t.y);
            }
            S[r] = add2(S[r], t);
        }
    }
}

}  // namespace sk
