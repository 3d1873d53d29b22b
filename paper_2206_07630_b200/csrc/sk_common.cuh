// sk_common.cuh — shared device helpers of the sm_100a Sinkhorn library.
// (PTX wrappers: MUFU ex2, packed FP32x2 FFMA2/FADD2, mbarrier + 1D bulk TMA.)
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace sk {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr double kLn2d = 0.6931471805599453094;
constexpr double kLog2ed = 1.4426950408889634074;

// ---------------------------------------------------------------- MUFU.EX2
__device__ __forceinline__ float ex2(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// ---------------------------------------------------------- packed f32x2 ops
// Blackwell FFMA2 / FADD2: two fp32 lanes per instruction (sm_100+).
union f2u {
    float2 f;
    unsigned long long u;
};

__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    f2u A, B, C, D;
    A.f = a; B.f = b; C.f = c;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(D.u) : "l"(A.u), "l"(B.u), "l"(C.u));
    return D.f;
}

__device__ __forceinline__ float2 add2(float2 a, float2 b) {
    f2u A, B, D;
    A.f = a; B.f = b;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(D.u) : "l"(A.u), "l"(B.u));
    return D.f;
}

__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
    f2u A, B, D;
    A.f = a; B.f = b;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(D.u) : "l"(A.u), "l"(B.u));
    return D.f;
}

// ------------------------------------------------------- (max, sum) merging
// Online log-sum-exp state in log2 units: value = M + log2(S).
__device__ __forceinline__ void lse_merge(float &M, float &S, float M2, float S2) {
    float Mn = fmaxf(M, M2);
    if (Mn == -INFINITY) return;  // both empty
    S = S * ex2(M - Mn) + S2 * ex2(M2 - Mn);
    M = Mn;
}

// ----------------------------------------------------- mbarrier + bulk copy
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

// 1D bulk TMA: global -> shared, completion via mbarrier transaction count.
__device__ __forceinline__ void bulk_g2s(void *dst_smem, const void *src_gmem, uint32_t bytes,
                                         uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst_smem)),
        "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t addr = smem_u32(bar);
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(addr),
        "r"(parity)
        : "memory");
}

// Consumer-side wait that suspends the thread (suspendTimeHint, ns) instead of re-polling the
// barrier: many waiting warps otherwise steal shared-memory cycles from the tensor core's
// operand reads.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity) {
    uint32_t addr = smem_u32(bar);
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAITS_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAITS_%=;\n\t}" ::"r"(addr),
        "r"(parity), "r"(0x989680)
        : "memory");
}

// --------------------------------------------------------- block reductions
// Deterministic (fixed-order) block sum of doubles; all threads get the result.
template <int NT>
__device__ __forceinline__ double block_sum_d(double v, double *scratch /* NT/32 */) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) scratch[w] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < NT / 32; ++i) s += scratch[i];
    return s;
}

template <int NT>
__device__ __forceinline__ int block_or(int v, int *scratch /* NT/32 */) {
    v = __any_sync(0xffffffffu, v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) scratch[w] = v;
    __syncthreads();
    int s = 0;
#pragma unroll
    for (int i = 0; i < NT / 32; ++i) s |= scratch[i];
    return s;
}

}  // namespace sk

// ------------------------------------------- K3 tensor-core image layout (shared with K6)
// One side of P points as images for tcgen05.mma (tiles of 128 points, padded to a multiple of
// 256 = one CTA-pair tile), in one allocation:
//   [T x (hi | lo)]   T = tc_tiles(P) tiles of 2 x 128 rb bytes: fp16 hi/lo split of alpha x,
//                     K-major; rb = 128: SWIZZLE_128B (row r of a tile: 64 halves, d <= 64);
//                     rb = 32: SWIZZLE_32B (16 halves, d <= 16 - a quarter of the bytes)
//   [T x EA]          4 KB per tile, K-major SWIZZLE_32B (16 halves per row): the "A role" extra
//                     columns [-sh/c, 0, 0, c, c, c, 0 ..]    (sh: the point's folded shift)
//   [T x EB]          4 KB per tile: the "B role" extra columns [c, 0, 0, w1, w2, w3, 0 ..]
//                     with w1 + w2 + w3 = w / c (three fp16 pieces, ~33 bits)
//   [T x 128 floats]  sh, exact (= -c * EA[0])
// so that one extra K = 16 MMA of EA(p) against EB(q) adds w_q - sh_p to the accumulator.
namespace sk {
constexpr int kTcImgBytes = 128 * 128;   // one SW128 image tile (128 rows x 128 bytes)
constexpr int kTcExtBytes = 128 * 32;    // one SW32 extra tile (128 rows x 32 bytes)
__host__ __device__ inline long long tc_tiles(long long P) { return (P + 255) / 256 * 2; }
__host__ __device__ inline long long tc_ea_off(long long P, int rb = 128) { return tc_tiles(P) * 2 * 128LL * rb; }
__host__ __device__ inline long long tc_eb_off(long long P, int rb = 128) { return tc_ea_off(P, rb) + tc_tiles(P) * kTcExtBytes; }
__host__ __device__ inline long long tc_sh_off(long long P, int rb = 128) { return tc_eb_off(P, rb) + tc_tiles(P) * kTcExtBytes; }
__host__ __device__ inline long long tc_side_bytes(long long P, int rb = 128) { return tc_sh_off(P, rb) + tc_tiles(P) * 128 * 4; }
// byte offset of half `slot` (0..15) of point p inside an extra image (SW32: the 16-byte chunk
// index is XORed with bit 2 of the row)
__device__ __forceinline__ long long tc_ext_at(long long p, int slot) {
    const long long t = p >> 7;
    const int r = (int)(p & 127), ch = slot >> 3;
    return t * kTcExtBytes + (r >> 3) * 256 + (r & 7) * 32 + ((ch ^ ((r >> 2) & 1)) << 4) + (slot & 7) * 2;
}
// EB slots 3..5 of point p: w / c as three fp16 pieces (w = -inf: [-inf, 0, 0])
__device__ __forceinline__ void tc_put_w(unsigned char *img, long long P, long long p, float w, float c,
                                         int rb = 128) {
    unsigned char *eb = img + tc_eb_off(P, rb);
    __half h1, h2 = __float2half_rn(0.f), h3 = h2;
    if (w == -INFINITY) {
        h1 = __float2half_rn(-INFINITY);
    } else {
        const float v = w / c;
        h1 = __float2half_rn(v);
        const float r1 = v - __half2float(h1);
        h2 = __float2half_rn(r1);
        h3 = __float2half_rn(r1 - __half2float(h2));
    }
    *reinterpret_cast<__half *>(eb + tc_ext_at(p, 3)) = h1;
    *reinterpret_cast<__half *>(eb + tc_ext_at(p, 4)) = h2;
    *reinterpret_cast<__half *>(eb + tc_ext_at(p, 5)) = h3;
}
// EA slot 0 of point p: the shift rounded to c * fp16; returns the exact shift stored in sh[p]
__device__ __forceinline__ float tc_put_shift(unsigned char *img, long long P, long long p, float sh, float c,
                                             int rb = 128) {
    const __half h = __float2half_rn(isfinite(sh) ? sh / c : 0.f);
    const float exact = __half2float(h) * c;
    *reinterpret_cast<__half *>(img + tc_ea_off(P, rb) + tc_ext_at(p, 0)) = __hneg(h);
    reinterpret_cast<float *>(img + tc_sh_off(P, rb))[p] = exact;
    return exact;
}

}  // namespace sk
