// sk_tc.cu — K3: the online LSE pass with the cross term on the 5th-generation tensor
// cores (tcgen05, kind::tf32, fp32 accumulators in TMEM), for d in (16, 64].
//
// BJ.ns: "computes the -2<x,y> cross term on tensor cores only when d >= 32, using an
// error-compensated 3xTF32 split".  Every point is split once per solve into
// hi = tf32(x), lo = tf32(x - hi) and stored as MMA-ready images (K-major, 128-byte
// swizzle, tiles of 128 points); acc = <p, q> is accumulated as
//     lo_p . hi_q + hi_p . lo_q + hi_p . hi_q      (3 MMAs per K step; lo.lo dropped)
// which is fp32-accurate (error ~2^-22 |p||q|; the potential error is 2 |d acc|).
//
// CTA = one tile of 128 output points (TMEM lanes) x one split of the other side:
//   warp 0   producer: 1D bulk TMA of the A image (once) and of B tile images + w tiles
//            into a 2-stage ring (mbarrier complete_tx);
//   warp 1   TMEM allocation and the MMA issuer (one elected thread): 3*K/8 MMAs
//            128x128xK per tile into one of two TMEM accumulators, tcgen05.commit to
//            the smem-slot and accumulator-ready barriers;
//   warps 2-5 epilogue: tcgen05.ld of the thread's row (= TMEM lane), t = 2 log2(e)/eps
//            * acc + w_q, online (max, sum 2^(t - max)) per 32 columns, MUFU.EX2.
// The output is the same (max, sum) partial as the FFMA kernel (K2), merged by K6.
#include "sk_internal.h"
#include "sk_common.cuh"

namespace sk {

constexpr int kTcM = 128;       // points per tile (MMA M and N)
constexpr int kTcEpiWarps = 8;  // two per TMEM lane quadrant, each half of the columns
constexpr int kTcThreads = 64 + 32 * kTcEpiWarps;
constexpr int kTcStages = 2;

__host__ __device__ constexpr int tc_img_bytes(int katoms) { return 16 * katoms * 1024; }  // one of hi/lo

// ------------------------------------------------------------ operand images
__device__ __forceinline__ float tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// img: tiles of 128 points, each [hi image | lo image], K-major SWIZZLE_128B canonical
// layout: 8-row x 128-byte atoms, atom (mi, kj) at (mi + 16 kj) * 1024 bytes, the 16-byte
// chunk c of row r stored at chunk c ^ (r % 8).
__global__ void k_pack_tc(const float *__restrict__ pts, long long P, int d, int katoms, float *img) {
    const long long tiles = (P + kTcM - 1) / kTcM;
    const int K = 32 * katoms;
    const long long total = tiles * kTcM * K;
    const int IMG = tc_img_bytes(katoms);
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long p = e / K;
        const int k = (int)(e % K);
        const long long t = p / kTcM;
        const int r = (int)(p % kTcM);
        const float x = (p < P && k < d) ? pts[p * d + k] : 0.f;
        const float hi = tf32_rna(x);
        const float lo = tf32_rna(x - hi);
        const int kj = k / 32, kb = (k % 32) * 4;
        const int chunk = (kb >> 4) ^ (r & 7);
        const long long off = (long long)((r >> 3) + 16 * kj) * 1024 + (r & 7) * 128 + chunk * 16 + (kb & 15);
        char *base = reinterpret_cast<char *>(img) + t * 2LL * IMG;
        *reinterpret_cast<float *>(base + off) = hi;
        *reinterpret_cast<float *>(base + IMG + off) = lo;
    }
}

// --------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
    uint64_t desc = 0;
    desc |= (uint64_t)((saddr >> 4) & 0x3FFF);          // start address
    desc |= (uint64_t)1 << 16;                           // LBO (unused for swizzled K-major)
    desc |= (uint64_t)(1024 >> 4) << 32;                 // SBO: 8-row group stride
    desc |= (uint64_t)1 << 46;                           // version (sm_100)
    desc |= (uint64_t)2 << 61;                           // SWIZZLE_128B
    return desc;
}

// kind::tf32, D = F32, A = B = TF32, both K-major, M = 128, N = 128
constexpr uint32_t kIdescTf32 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kTcM >> 3) << 17) |
                                ((uint32_t)(kTcM >> 4) << 24);

__device__ __forceinline__ void umma_tf32(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtmem),
        "l"(adesc), "l"(bdesc), "r"(kIdescTf32), "r"(accum));
}

__device__ __forceinline__ void umma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

#define TMEM_LD32(taddr, r)                                                                                    \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15," \
                 "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                     \
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),          \
                   "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),      \
                   "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),   \
                   "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),   \
                   "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                                           \
                 : "r"(taddr))

__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ------------------------------------------------------------------ the kernel
struct TcArgs {
    const float *Aimg;      // P side images
    const float *Bimg;      // Q side images
    const float *Bw;        // Q side packed w, [Qtiles][128] (D = 0 style plain array, padded -inf)
    int P, Qtiles;
    int blk_tiles, split_q; // Q split structure (as K2)
    float2 *part;
    float tk;               // 2 log2(e)/eps
    const int *stop;
    float *debug_acc;       // if non-null: write raw acc of the first Q tile, [128][128]
    int mma_only;           // K14 microbenchmark: epilogue only releases the buffers
};

template <int KATOMS>
__global__ void __launch_bounds__(kTcThreads, 1) k_lse_tc(TcArgs A) {
    constexpr int IMG = tc_img_bytes(KATOMS);
    constexpr int KSTEPS = KATOMS * 4;              // K = 8 tf32 per MMA
    constexpr int STAGE = 2 * IMG;                  // B hi + lo (1024-aligned slots)
    extern __shared__ __align__(1024) unsigned char smraw[];
    // 1024-byte alignment of the dynamic smem window for the swizzled operands
    unsigned char *sm = smraw + ((1024 - (smem_u32(smraw) & 1023)) & 1023);
    unsigned char *sA = sm;                          // [hi | lo] of this CTA's 128 points
    unsigned char *sB = sm + 2 * IMG;                // kTcStages x STAGE
    float *sW = reinterpret_cast<float *>(sB + kTcStages * STAGE);  // kTcStages x 128 w values
    __shared__ __align__(8) uint64_t bar_a, full[kTcStages], empty[kTcStages], tfull[2], tempty[2];
    __shared__ uint32_t tmem_base;

    if (A.stop && *(volatile const int *)A.stop) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    const int s = blockIdx.y;
    const int bq = s / A.split_q, u = s % A.split_q;
    const int bt = A.blk_tiles > 0 ? A.blk_tiles : A.Qtiles;
    const int base = bq * bt;
    const int nt_b = max(0, min(bt, A.Qtiles - base));
    const int t0 = base + (int)((long long)nt_b * u / A.split_q);
    const int nt = base + (int)((long long)nt_b * (u + 1) / A.split_q) - t0;

    if (threadIdx.x == 0) {
        mbar_init(&bar_a, 1);
        for (int i = 0; i < kTcStages; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1 + kTcEpiWarps); }
        for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], kTcEpiWarps); }
        fence_mbar_init();
    }
    if (warp == 1) {  // 256 TMEM columns: two 128x128 fp32 accumulators
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = tmem_base;

    if (warp == 0) {
        if (lane == 0) {
            // A images (the CTA's own points), then the B ring
            mbar_expect_tx(&bar_a, 2 * IMG);
            bulk_g2s(sA, reinterpret_cast<const char *>(A.Aimg) + (long long)blockIdx.x * 2 * IMG, 2 * IMG, &bar_a);
            for (int i = 0; i < nt; ++i) {
                const int st = i % kTcStages;
                if (i >= kTcStages) mbar_wait(&empty[st], ((i / kTcStages) - 1) & 1);
                unsigned char *dst = sB + st * STAGE;
                mbar_expect_tx(&full[st], STAGE + kTcM * 4);
                bulk_g2s(dst, reinterpret_cast<const char *>(A.Bimg) + (long long)(t0 + i) * 2 * IMG, 2 * IMG,
                         &full[st]);
                bulk_g2s(sW + st * kTcM, A.Bw + (long long)(t0 + i) * kTcM, kTcM * 4, &full[st]);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            mbar_wait(&bar_a, 0);
            const uint32_t a_hi = smem_u32(sA), a_lo = a_hi + IMG;
            for (int i = 0; i < nt; ++i) {
                const int st = i % kTcStages, b = i & 1;
                mbar_wait(&full[st], (i / kTcStages) & 1);
                if (i >= 2) mbar_wait(&tempty[b], ((i >> 1) - 1) & 1);
                tc_fence_after();
                const uint32_t b_hi = smem_u32(sB + st * STAGE), b_lo = b_hi + IMG;
                const uint32_t d = tbase + (uint32_t)(b * kTcM);
#pragma unroll
                for (int k = 0; k < KSTEPS; ++k) {
                    const uint32_t koff = (uint32_t)((k >> 2) * 16 * 1024 + (k & 3) * 32);
                    umma_tf32(d, umma_desc_sw128(a_lo + koff), umma_desc_sw128(b_hi + koff), k > 0);
                    umma_tf32(d, umma_desc_sw128(a_hi + koff), umma_desc_sw128(b_lo + koff), 1);
                }
#pragma unroll
                for (int k = 0; k < KSTEPS; ++k) {
                    const uint32_t koff = (uint32_t)((k >> 2) * 16 * 1024 + (k & 3) * 32);
                    umma_tf32(d, umma_desc_sw128(a_hi + koff), umma_desc_sw128(b_hi + koff), 1);
                }
                umma_commit(&empty[st]);   // smem slot free once these MMAs retire
                umma_commit(&tfull[b]);    // accumulator b ready
            }
        }
    } else {
        // epilogue: warp w reads TMEM lanes 32*(w%4) .. +31 (its quadrant) and the column half
        // h = (w-2)/4 of every accumulator; thread = one output point, (M, S) over its half.
        const int q4 = warp & 3, h = (warp - 2) >> 2;
        const int row = q4 * 32 + lane;
        const int p = blockIdx.x * kTcM + row;
        float M = -INFINITY, S = 0.f;
        for (int i = 0; i < nt; ++i) {
            const int st = i % kTcStages, b = i & 1;
            mbar_wait(&tfull[b], (i >> 1) & 1);
            tc_fence_after();
            if (A.mma_only) {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) { mbar_arrive(&tempty[b]); mbar_arrive(&empty[st]); }
                continue;
            }
            const float *w = sW + st * kTcM + h * 64;
            uint32_t r[64];
            const uint32_t taddr = tbase + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(b * kTcM + h * 64);
            TMEM_LD32(taddr, r);
            TMEM_LD32(taddr + 32, (r + 32));
            tmem_ld_wait();
            if (A.debug_acc && i == 0 && blockIdx.x == 0 && blockIdx.y == 0) {
#pragma unroll
                for (int j = 0; j < 64; ++j) A.debug_acc[row * kTcM + h * 64 + j] = __uint_as_float(r[j]);
            }
            float t[64];
#pragma unroll
            for (int j = 0; j < 64; ++j) t[j] = fmaf(__uint_as_float(r[j]), A.tk, w[j]);
            // accumulator b and the w slot are no longer needed: release them early
            tc_fence_before();
            __syncwarp();
            if (lane == 0) { mbar_arrive(&tempty[b]); mbar_arrive(&empty[st]); }
            float cm = t[0];
#pragma unroll
            for (int j = 1; j < 64; ++j) cm = fmaxf(cm, t[j]);
            if (cm > M) { S *= ex2(M - cm); M = cm; }
            if (M == -INFINITY) continue;  // only padding seen so far (ragged last tile's upper half)
            float s0 = 0.f, s1 = 0.f;
#pragma unroll
            for (int j = 0; j < 64; j += 2) { s0 += ex2(t[j] - M); s1 += ex2(t[j + 1] - M); }
            S += s0 + s1;
        }
        // combine the two column halves of each row (fixed order: half 0 then half 1)
        float2 *xch = reinterpret_cast<float2 *>(sW + kTcStages * kTcM);  // 128 x float2
        if (h == 1) xch[row] = make_float2(M, S);
        asm volatile("bar.sync 1, %0;" ::"r"(32 * kTcEpiWarps));
        if (h == 0) {
            const float2 o = xch[row];
            lse_merge(M, S, o.x, o.y);
            if (p < A.P) A.part[(long long)s * A.P + p] = make_float2(M, S);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tbase));
    }
}

// --------------------------------------------------------------------- host side
size_t tc_image_floats(long long P, int katoms) {
    return (size_t)((P + kTcM - 1) / kTcM) * 2 * tc_img_bytes(katoms) / 4;
}

cudaError_t launch_pack_tc(const float *pts, long long P, int d, int katoms, float *img, cudaStream_t st) {
    const long long total = ((P + kTcM - 1) / kTcM) * kTcM * 32LL * katoms;
    long long b = (total + 255) / 256;
    k_pack_tc<<<(int)(b > 148 * 16 ? 148 * 16 : b), 256, 0, st>>>(pts, P, d, katoms, img);
    return cudaGetLastError();
}

template <int KATOMS>
static cudaError_t launch_tc_k(const TcArgs &A, int ptiles, int nsplit, cudaStream_t st) {
    const size_t smem = 1024 + 2 * (size_t)tc_img_bytes(KATOMS) + kTcStages * (2 * (size_t)tc_img_bytes(KATOMS) + kTcM * 4)
                        + kTcM * 8;   // half-combination exchange
    cudaError_t e = cudaFuncSetAttribute(k_lse_tc<KATOMS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid(ptiles, nsplit);
    k_lse_tc<KATOMS><<<grid, kTcThreads, smem, st>>>(A);
    return cudaGetLastError();
}

cudaError_t launch_lse_tc(const TcPass &L, cudaStream_t st) {
    TcArgs A;
    A.Aimg = L.Aimg; A.Bimg = L.Bimg; A.Bw = L.Bw;
    A.P = L.P; A.Qtiles = (int)((L.Q + kTcM - 1) / kTcM);
    A.blk_tiles = L.blk_tiles; A.split_q = L.split_q;
    A.part = L.part; A.tk = 2.f * kLog2e / L.eps; A.stop = L.stop; A.debug_acc = L.debug_acc;
    A.mma_only = L.mma_only;
    const int ptiles = (L.P + kTcM - 1) / kTcM;
    const int nsplit = L.nblk * L.split_q;
    return L.katoms == 1 ? launch_tc_k<1>(A, ptiles, nsplit, st) : launch_tc_k<2>(A, ptiles, nsplit, st);
}

}  // namespace sk
