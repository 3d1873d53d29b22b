// sk_tc.cu — K3: the online LSE pass with the cross term on the 5th-generation tensor
// cores (tcgen05.mma kind::f16, fp16 operands, fp32 accumulators in TMEM), for d in (16, 256]
// (d > 64 in K chunks of 64, template KC) and for every d on large problems.
//
// BJ.ns: "computes the -2<x,y> cross term on tensor cores only when d >= 32, using an
// error-compensated 3xTF32/bf16x3 split".  This kernel uses the same three-product split with
// IEEE fp16 pieces (twice the TF32 tensor rate, the same 22-bit significand).  Per solve, each
// side is scaled once — x by alpha_x = 2^s, y by alpha_y = tk 2^-s with tk = 2 log2(e)/eps and
// the integer s balancing the two magnitudes (K3a absmax) — and split into
//     hi = fp16(alpha x),  lo = fp16(alpha x - hi)        (11 + 11 significand bits)
// stored as MMA-ready images (K-major, 128-byte swizzle, tiles of 128 points, K padded to 64).
// The accumulator of a (p, q) entry is
//     lo_p . hi_q + hi_p . lo_q + hi_p . hi_q  +  EA_p . EB_q
//   = tk <p, q>  +  w_q - sh_p          (3 x ksteps + 1 MMAs of K = 16; lo.lo dropped)
// where the extra K = 16 step multiplies the output point's "A role" columns (its shift sh_p)
// against the reduced point's "B role" columns (w_q = (h_q - |q|^2) log2(e)/eps in three fp16
// pieces; layout in sk_common.cuh).  So the accumulator IS the log2-domain exponent minus the
// row shift: the epilogue is one tcgen05.ld and one exponential per entry (seeded passes: no
// max, no multiply, no w load).  K6 rewrites w and sh of a side after every merge.
//
// CTA pair (cta_group::2), persistent: the pair computes 256 x 256 tiles (A: 128 output points
// per CTA; B: 128 reduction points per CTA), two TMEM accumulator buffers of 256 columns.
// The output is the same (max, sum) partial as the FFMA kernel (K2), merged by K6.
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "sk_internal.h"
#include "sk_common.cuh"
#include "sk_lse_tile.cuh"

namespace sk {

constexpr int kTcM = 128;                 // points per image tile (MMA rows per CTA)
constexpr int kTcImg = kTcImgBytes;       // bytes of one fp16 image: 128 rows x 64 halves (16 SW128 atoms)
constexpr float kTcFoldC = 16.f;          // c of the extra columns (sh and w range |.| < 2^20)

// ------------------------------------------------------------ operand images
// K3a: max |x| over all coordinates (non-negative floats order like their bit patterns).
__global__ void k_absmax(const float *__restrict__ pts, long long cnt, unsigned *out) {
    float mx = 0.f;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < cnt;
         i += (long long)gridDim.x * blockDim.x)
        mx = fmaxf(mx, fabsf(pts[i]));
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0 && mx > 0.f) atomicMax(out, __float_as_uint(mx));
}

// exponent e with max = f 2^e, f in [1/2, 1) (0 for an all-zero side)
__host__ __device__ inline int tc_exp_of(float mx) {
    int e = 0;
    if (mx > 0.f) frexpf(mx, &e);
    return e;
}
// the balancing exponent s: max |alpha_x x| ~ 2^(ex + s), max |alpha_y y| ~ tk 2^(ey - s)
__host__ __device__ inline int tc_fold_s(float ax, float ay, float tk) {
    return (int)rintf(0.5f * (log2f(tk) + (float)tc_exp_of(ay) - (float)tc_exp_of(ax)));
}

// img: tiles of 128 points, each [hi image | lo image] of alpha * x, K-major SWIZZLE_128B
// canonical layout: 8-row x 128-byte atoms, atom mi at mi * 1024 bytes, the 16-byte chunk c
// (halves 8c .. 8c+7) of row r stored at chunk c ^ (r % 8).  One thread per (point, chunk).
// role 0 (x side): alpha = 2^s; role 1 (y side): alpha = tk 2^-s.
__global__ void k_pack_tc(const float *__restrict__ pts, long long P, long long P2, int d, const unsigned *amax2,
                          int role, float tk, unsigned char *img, int rb) {
    // rb = 128: SW128 (8 chunks of 8 halves per row); rb = 128 KC (d in (64, 256]): KC such SW128
    // K chunks per tile, each chunk's hi and lo images adjacent; rb = 32: SW32 (2 chunks,
    // d <= 16), the 16-byte chunk index XORed with bit 2 of the row, 8-row groups of 256 bytes
    const int cpr = rb / 16;
    const long long total = P2 * cpr;
    const int s = tc_fold_s(__uint_as_float(amax2[0]), __uint_as_float(amax2[1]), tk);
    const float alpha = role == 0 ? ldexpf(1.f, s) : ldexpf(tk, -s);
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long p = e / cpr;
        const int c = (int)(e % cpr);
        const long long t = p / kTcM;
        const int r = (int)(p % kTcM);
        __align__(16) __half hi[8], lo[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int k = 8 * c + j;
            const float x = (p < P && k < d) ? pts[p * d + k] * alpha : 0.f;
            hi[j] = __float2half_rn(x);
            lo[j] = __float2half_rn(x - __half2float(hi[j]));
        }
        const long long ib = 128LL * rb;   // bytes of one image tile (all K chunks)
        unsigned char *base = img + t * 2LL * ib;
        if (rb >= 128) {
            // K chunk kc = c / 8 (64 halves) at kc * 32 KB: [hi 16 KB | lo 16 KB] (rb = 128: one chunk)
            const int kc = c >> 3, cc = c & 7;
            const long long off = (long long)kc * 2 * kTcImgBytes + (r >> 3) * 1024 + (r & 7) * 128 + ((cc ^ (r & 7)) << 4);
            *reinterpret_cast<uint4 *>(base + off) = *reinterpret_cast<const uint4 *>(hi);
            *reinterpret_cast<uint4 *>(base + kTcImgBytes + off) = *reinterpret_cast<const uint4 *>(lo);
        } else {
            const long long off = (long long)(r >> 3) * 256 + (r & 7) * 32 + ((c ^ ((r >> 2) & 1)) << 4);
            *reinterpret_cast<uint4 *>(base + off) = *reinterpret_cast<const uint4 *>(hi);
            *reinterpret_cast<uint4 *>(base + ib + off) = *reinterpret_cast<const uint4 *>(lo);
        }
    }
}

// K3b: the extra columns of every point: EA = [0, 0, 0, c, c, c, 0 ..] (shift 0), EB = [c, 0, 0,
// w pieces, 0 ..] from the plain w array (w == nullptr: 0; padding points: w = -inf), sh = 0.
__global__ void k_pack_tc_ext(long long P, long long P2, const float *__restrict__ w, float c, unsigned char *img,
                              int rb) {
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < P2; p += (long long)gridDim.x * blockDim.x) {
        unsigned char *ea = img + tc_ea_off(P, rb), *eb = img + tc_eb_off(P, rb);
        const __half z = __float2half_rn(0.f), ch = __float2half_rn(c);
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            *reinterpret_cast<__half *>(ea + tc_ext_at(p, k)) = (k >= 3 && k <= 5) ? ch : z;
            *reinterpret_cast<__half *>(eb + tc_ext_at(p, k)) = (k == 0) ? ch : z;
        }
        reinterpret_cast<float *>(img + tc_sh_off(P, rb))[p] = 0.f;
        tc_put_w(img, P, p, p < P ? (w ? w[p] : 0.f) : -INFINITY, c, rb);
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

// SWIZZLE_32B K-major (the 16-half extra images): 8-row groups of 256 bytes
__device__ __forceinline__ uint64_t umma_desc_sw32(uint32_t saddr) {
    uint64_t desc = 0;
    desc |= (uint64_t)((saddr >> 4) & 0x3FFF);
    desc |= (uint64_t)1 << 16;
    desc |= (uint64_t)(256 >> 4) << 32;                  // SBO: 8 rows x 32 bytes
    desc |= (uint64_t)1 << 46;
    desc |= (uint64_t)6 << 61;                           // SWIZZLE_32B
    return desc;
}

// kind::f16, D = F32, A = B = F16, both K-major, M = 128, N = 128 (K14 probe shape)
constexpr uint32_t kIdescF16 = (1u << 4) | ((uint32_t)(kTcM >> 3) << 17) | ((uint32_t)(kTcM >> 4) << 24);

__device__ __forceinline__ void umma_f16(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtmem),
        "l"(adesc), "l"(bdesc), "r"(kIdescF16), "r"(accum));
}

__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
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
    const unsigned char *Aimg;  // output side images (P points) incl. EA, sh
    const unsigned char *Bimg;  // reduced side images (Q points) incl. EB
    int P, Q, Qtiles, ksteps, ptiles;
    int nblk, blk_tiles, split_q;   // Q split structure (as K2), in tiles of 256 points
    float2 *part;
    float tk;                   // 2 log2(e)/eps (only the selftest's unscale uses it)
    const int *stop;
    const int *only_if;         // run only if *only_if != 0 (nullable; the exact column redo)
    float *debug_acc;           // if non-null: write <p, q> of the first 128 x 128 block, [128][128]
    int mma_only;               // K14 probes: 1, 2, 4 = the epilogue only releases the buffers
                                //   (2: and the B ring is not reloaded); 3 = no MMAs, full epilogue
    long long *cyc;             // K14: SM cycles of CTA 0 (clock64 around the work), nullable
};

// which exponential pairs of a chunk go to the FMA pipe: EMU < 100: the last EMU of every 8;
// EMU >= 100: the last EMU - 100 of every 16 (finer balances)
template <int EMU>
__device__ __forceinline__ constexpr bool tc_emu_pair(int j) {
    return EMU >= 100 ? (j & 15) >= 16 - (EMU - 100) : (j & 7) >= 8 - EMU;
}

// sum of 2^(t - M) over one 64-column chunk (32 pairs), EMU of every 8 pairs on the FMA pipe;
// SUB = false: M = 0 (seeded passes: the shift is already in the accumulator)
template <int EMU, bool SUB>
__device__ __forceinline__ float2 tc_sum_chunk(const float2 (&t)[32], float M) {
    const float2 mm = make_float2(M, M);
    float2 s0 = make_float2(0.f, 0.f), s1 = s0;
#pragma unroll
    for (int j = 0; j < 32; j += 2) {
        float2 e0 = t[j], e1 = t[j + 1];
        if constexpr (SUB) { e0 = sub2(e0, mm); e1 = sub2(e1, mm); }
        if (tc_emu_pair<EMU>(j)) e0 = ex2_emu2(e0); else { e0.x = ex2(e0.x); e0.y = ex2(e0.y); }
        if (tc_emu_pair<EMU>(j + 1)) e1 = ex2_emu2(e1); else { e1.x = ex2(e1.x); e1.y = ex2(e1.y); }
        s0 = add2(s0, e0);
        s1 = add2(s1, e1);
    }
    return add2(s0, s1);
}

// the same over one 32-column chunk (16 pairs; seeded: M = 0), the FMA-pipe pairs as above
template <int EMU>
__device__ __forceinline__ float2 tc_sum_half(const uint32_t (&r)[32]) {
    float2 s0 = make_float2(0.f, 0.f), s1 = s0;
#pragma unroll
    for (int j = 0; j < 16; j += 2) {
        float2 e0 = make_float2(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1]));
        float2 e1 = make_float2(__uint_as_float(r[2 * j + 2]), __uint_as_float(r[2 * j + 3]));
        if (tc_emu_pair<EMU>(j)) e0 = ex2_emu2(e0); else { e0.x = ex2(e0.x); e0.y = ex2(e0.y); }
        if (tc_emu_pair<EMU>(j + 1)) e1 = ex2_emu2(e1); else { e1.x = ex2(e1.x); e1.y = ex2(e1.y); }
        s0 = add2(s0, e0);
        s1 = add2(s1, e1);
    }
    return add2(s0, s1);
}

// cta_group::2: the pair computes a 256 x 256 tile per MMA group (M = 256 split over the two
// SMs' A halves, N = 256 split over their B halves).  Roles per CTA (rank r of the pair):
//   warp 0   producer: A half (points 256 pt + 128 r: [hi | lo | EA], 36 KB) once per item, B
//            halves (points 256 bt + 128 r: [hi | lo | EB]) into a kT2Stages ring;
//   warp 1   leader: TMEM allocation (both CTAs allocate, cta_group::2) and the MMA issuer;
//            peer: relay — waits for its own A/B arrivals and arrives remotely on the leader's
//            pair barriers (1D bulk copies signal their own CTA's mbarrier);
//   warps 2.. epilogue (NE warps) on this CTA's 128 accumulator rows: warp w = lane quadrant
//            w % 4, column group (w - 2) / 4 (256 / (NE / 4) columns); releases accumulator b
//            remotely on the leader's tempty.  MMA completion is multicast to both CTAs' barriers.
constexpr int kT2Stages = 4;                  // B ring depth (36 KB stages)
constexpr int kT2N = 256;                     // MMA N (B points per tile) and A points per item
constexpr uint32_t kIdescF16M256N256 = (1u << 4) | ((uint32_t)(kT2N >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);

__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
    return pred != 0;
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
// Relaxed: the arrivals only signal that a TMEM buffer was drained (tcgen05.wait::ld already
// retired the loads) or that an async-proxy copy completed; no generic-proxy data is published,
// and .release.cluster would cost a MEMBAR.ALL.GPU per arrive (measured: 12 % of stall samples).
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void umma2_f16(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtmem),
        "l"(adesc), "l"(bdesc), "r"(kIdescF16M256N256), "r"(accum));
}
__device__ __forceinline__ void umma2_commit_mc(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(smem_u32(bar)), "h"((uint16_t)3) : "memory");
}


// KC > 1 (d in (64, 256], RB = 128): the images hold KC K chunks of 64 halves; the A half of an
// item is staged whole (KC chunks, one buffer when KC > 2), the B half of a tile arrives chunk by
// chunk through a two-stage ring of K3's 36 KB stages (the extra columns with the last chunk), and
// the tile's accumulator takes 3 x 4 MMAs per chunk plus the extra-column MMA after the last.
template <int EMU, int NE, bool SEEDED, int G, int PL = 0, bool DBG = false, int RB = 128, int KC = 1>
__global__ void __launch_bounds__(64 + 32 * NE, 1) k_lse_tc2(TcArgs A) {
    constexpr int NQ = NE / 4;                       // epilogue warps per TMEM lane quadrant
    // G tile groups: group k's warps take the tiles g with g % G == k (accumulator buffer k when
    // G = 2), so one group's TMEM loads overlap the other group's exponentials
    constexpr int NQG = NQ / G;                      // warps per lane quadrant and group
    constexpr int CW = kT2N / NQG;                   // accumulator columns per epilogue warp
    static_assert(KC == 1 || RB == 128, "K chunks use the SW128 images");
    constexpr int ABUF = KC > 2 ? 1 : 2;
    constexpr int NBS = KC > 1 ? 2 : kT2Stages;       // B ring depth
    constexpr int RBX = RB * KC;                      // image row bytes (the side's offsets)
    // [hi | lo | extra] of 128 points: 36 KB (RB = 128), 12 KB (RB = 32: the compact d <= 16 images)
    constexpr int IMG = 128 * RB;
    constexpr int STAGE = 2 * IMG + kTcExtBytes;      // B stage: one K chunk (+ the extra columns)
    constexpr int ASTAGE = 2 * KC * IMG + kTcExtBytes;
    extern __shared__ __align__(1024) unsigned char smraw[];
    unsigned char *sm = smraw + ((1024 - (smem_u32(smraw) & 1023)) & 1023);
    unsigned char *sA = sm;                           // ABUF x ASTAGE: this CTA's 128 A rows
    unsigned char *sB = sm + ABUF * ASTAGE;           // NBS x STAGE: this CTA's 128 B rows
    float2 *xch = reinterpret_cast<float2 *>(sB + NBS * STAGE);   // (NQ - 1) x 128 partials
    __shared__ __align__(8) uint64_t full[NBS], pfull[NBS], empty[NBS], tfull[2], tempty[2],
        afull[ABUF], pafull[ABUF], aempty[ABUF];
    __shared__ uint32_t tmem_base;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    // uniform over the pair (same flags)
    const bool stopped = (A.stop && *(volatile const int *)A.stop) || (A.only_if && !*(volatile const int *)A.only_if);
    if (stopped) return;
    const int nsplit = A.nblk * A.split_q;
    const int items = A.ptiles * nsplit;
    const int bt_blk = A.blk_tiles > 0 ? A.blk_tiles : A.Qtiles;
    auto range = [&](int s, int &t0, int &nt) {
        const int bq = s / A.split_q, u = s % A.split_q;
        const int base = bq * bt_blk;
        const int nt_b = max(0, min(bt_blk, A.Qtiles - base));
        t0 = base + (int)((long long)nt_b * u / A.split_q);
        nt = base + (int)((long long)nt_b * (u + 1) / A.split_q) - t0;
    };
    const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;

    if (threadIdx.x == 0) {
        for (int i = 0; i < NBS; ++i) {
            mbar_init(&full[i], 1); mbar_init(&pfull[i], 1); mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 2 * NE / G); }
        for (int i = 0; i < ABUF; ++i) { mbar_init(&afull[i], 1); mbar_init(&pafull[i], 1); mbar_init(&aempty[i], 1); }
        fence_mbar_init();
    }
    if (warp == 1) {  // both CTAs: 512 TMEM columns = 2 accumulator buffers x 256 columns
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    cluster_sync_all();   // barriers initialised in both CTAs before any remote arrive
    tc_fence_after();
    const uint32_t tbase = tmem_base;
    const long long clk0 = clock64();

    if (warp == 0) {
        if (lane == 0) {
            const unsigned char *aext = A.Aimg + tc_ea_off(A.P, RBX), *bext = A.Bimg + tc_eb_off(A.Q, RBX);
            int g = 0, c = 0;
            for (int it = cid; it < items; it += ncl, ++c) {
                const int s = it / A.ptiles, pt = it % A.ptiles;
                int t0, nt;
                range(s, t0, nt);
                const int ab = c % ABUF;
                const long long at = 2LL * pt + rank;   // this CTA's 128-point A tile
                if (c >= ABUF) mbar_wait_sleep(&aempty[ab], ((c / ABUF) - 1) & 1);
                mbar_expect_tx(&afull[ab], ASTAGE);
                bulk_g2s(sA + ab * ASTAGE, A.Aimg + at * 2 * KC * IMG, 2 * KC * IMG, &afull[ab]);
                bulk_g2s(sA + ab * ASTAGE + 2 * KC * IMG, aext + at * kTcExtBytes, kTcExtBytes, &afull[ab]);
                for (int i = 0; i < nt; ++i) {
                    const long long bt = 2LL * (t0 + i) + rank;
                    for (int kc = 0; kc < KC; ++kc, ++g) {
                        const int st = g % NBS;
                        const bool last = kc == KC - 1;
                        if (g >= NBS) mbar_wait_sleep(&empty[st], ((g / NBS) - 1) & 1);
                        if (A.mma_only == 2 && g >= NBS) {   // K14 probe: MMA rate without the B stream
                            mbar_arrive(&full[st]);
                            continue;
                        }
                        mbar_expect_tx(&full[st], 2 * IMG + (last ? kTcExtBytes : 0));
                        bulk_g2s(sB + st * STAGE, A.Bimg + (bt * KC + kc) * 2 * IMG, 2 * IMG, &full[st]);
                        if (last) bulk_g2s(sB + st * STAGE + 2 * IMG, bext + bt * kTcExtBytes, kTcExtBytes, &full[st]);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && !leader) {
            // relay: own arrivals -> the leader's pair barriers
            const uint32_t r_pafull = mapa_u32(smem_u32(&pafull[0]), 0), r_pfull = mapa_u32(smem_u32(&pfull[0]), 0);
            int g = 0, c = 0;
            for (int it = cid; it < items; it += ncl, ++c) {
                int t0, nt;
                range(it / A.ptiles, t0, nt);
                const int ab = c % ABUF;
                mbar_wait(&afull[ab], (c / ABUF) & 1);
                mbar_arrive_cluster(r_pafull + 8 * ab);
                for (int i = 0; i < nt * KC; ++i, ++g) {
                    const int st = g % NBS;
                    mbar_wait(&full[st], (g / NBS) & 1);
                    mbar_arrive_cluster(r_pfull + 8 * st);
                }
            }
        } else if (leader) {
            // MMA issuer: the whole warp runs the (warp-uniform) loop, so the descriptors live in
            // uniform registers; one elected lane issues each tcgen05 instruction
            const int ks = (A.mma_only == 3 || A.mma_only == 5) ? 0 : A.ksteps;
            int g = 0, c = 0, gc = 0;   // tiles, items, B chunks
            for (int it = cid; it < items; it += ncl, ++c) {
                int t0, nt;
                range(it / A.ptiles, t0, nt);
                const int ab = c % ABUF;
                mbar_wait(&afull[ab], (c / ABUF) & 1);
                mbar_wait(&pafull[ab], (c / ABUF) & 1);
                if constexpr (KC == 1) {
                    const uint32_t a_hi = smem_u32(sA + ab * STAGE);
                    const uint64_t da_hi = RB == 128 ? umma_desc_sw128(a_hi) : umma_desc_sw32(a_hi),
                                   da_lo = RB == 128 ? umma_desc_sw128(a_hi + IMG) : umma_desc_sw32(a_hi + IMG),
                                   da_ex = umma_desc_sw32(a_hi + 2 * IMG);
                    for (int i = 0; i < nt; ++i, ++g) {
                        const int st = g % kT2Stages, b = g & 1;
                        mbar_wait(&full[st], (g / kT2Stages) & 1);
                        mbar_wait(&pfull[st], (g / kT2Stages) & 1);
                        if (g >= 2) mbar_wait_sleep(&tempty[b], ((g >> 1) - 1) & 1);
                        tc_fence_after();
                        const uint32_t b_hi = smem_u32(sB + st * STAGE);
                        const uint64_t db_hi = RB == 128 ? umma_desc_sw128(b_hi) : umma_desc_sw32(b_hi),
                                       db_lo = RB == 128 ? umma_desc_sw128(b_hi + IMG) : umma_desc_sw32(b_hi + IMG),
                                       db_ex = umma_desc_sw32(b_hi + 2 * IMG);
                        const uint32_t d = tbase + (uint32_t)(b * kT2N);
                        if (elect_one()) {
                            // smallest magnitudes first (each MMA rounds at the running accumulator's
                            // scale): the lo cross products, then hi . hi, then the extra columns
                            // w_q - sh_p, which bring the sum down to t - sh_p in one rounding.
                            // K = 16 halves = 32 bytes per step = +2 in the descriptor's address field.
                            for (int k = 0; k < ks; ++k) {
                                umma2_f16(d, da_lo + 2 * k, db_hi + 2 * k, k > 0);
                                umma2_f16(d, da_hi + 2 * k, db_lo + 2 * k, 1);
                            }
                            for (int k = 0; k < ks; ++k) umma2_f16(d, da_hi + 2 * k, db_hi + 2 * k, 1);
                            if (A.mma_only != 3 && A.mma_only != 5) umma2_f16(d, da_ex, db_ex, 1);
                            umma2_commit_mc(&empty[st]);   // both CTAs' B slots free once these MMAs retire
                            umma2_commit_mc(&tfull[b]);    // accumulator b ready in both CTAs
                        }
                        __syncwarp();
                    }
                } else {
                    // K chunks: per tile, KC ring stages; the lo cross products then hi . hi of
                    // each chunk (the chunk's 4 K steps), the extra columns after the last chunk
                    const uint32_t a0 = smem_u32(sA + ab * ASTAGE);
                    const uint64_t da_ex = umma_desc_sw32(a0 + 2 * KC * IMG);
                    for (int i = 0; i < nt; ++i, ++g) {
                        const int b = g & 1;
                        const uint32_t d = tbase + (uint32_t)(b * kT2N);
                        for (int kc = 0; kc < KC; ++kc, ++gc) {
                            const int st = gc % NBS;
                            mbar_wait(&full[st], (gc / NBS) & 1);
                            mbar_wait(&pfull[st], (gc / NBS) & 1);
                            if (kc == 0 && g >= 2) mbar_wait_sleep(&tempty[b], ((g >> 1) - 1) & 1);
                            tc_fence_after();
                            const uint32_t a_hi = a0 + kc * 2 * IMG, b_hi = smem_u32(sB + st * STAGE);
                            const uint64_t da_hi = umma_desc_sw128(a_hi), da_lo = umma_desc_sw128(a_hi + IMG),
                                           db_hi = umma_desc_sw128(b_hi), db_lo = umma_desc_sw128(b_hi + IMG),
                                           db_ex = umma_desc_sw32(b_hi + 2 * IMG);
                            const int kn = min(4, ks - 4 * kc);
                            if (elect_one()) {
                                for (int k = 0; k < kn; ++k) {
                                    umma2_f16(d, da_lo + 2 * k, db_hi + 2 * k, kc > 0 || k > 0);
                                    umma2_f16(d, da_hi + 2 * k, db_lo + 2 * k, 1);
                                }
                                for (int k = 0; k < kn; ++k) umma2_f16(d, da_hi + 2 * k, db_hi + 2 * k, 1);
                                if (kc == KC - 1 && A.mma_only != 3 && A.mma_only != 5) umma2_f16(d, da_ex, db_ex, 1);
                                umma2_commit_mc(&empty[st]);
                                if (kc == KC - 1) umma2_commit_mc(&tfull[b]);
                            }
                            __syncwarp();
                        }
                    }
                }
                if (elect_one()) umma2_commit_mc(&aempty[ab]);   // both CTAs' A buffers free
                __syncwarp();
            }
        }
    } else {
        // epilogue: this CTA's accumulator rows (TMEM lanes) q4*32 + lane, columns hc*CW ..+CW-1
        // in 64-column chunks; the accumulator is t - sh (log2 units).  (A software-pipelined
        // variant — the next chunk's TMEM load in flight under the current chunk's
        // exponentials — measured slower: the epilogue is issue-bound next to MUFU.)
        const int q4 = warp & 3, h = (warp - 2) >> 2;
        const int grp = h / NQG, hc = h % NQG;   // tile group, column group
        const int row = q4 * 32 + lane;
        const float *sh = reinterpret_cast<const float *>(A.Aimg + tc_sh_off(A.P, RBX));
        const uint32_t r_tempty = leader ? smem_u32(&tempty[0]) : mapa_u32(smem_u32(&tempty[0]), 0);
        const bool full_epi = A.mma_only == 0 || A.mma_only == 3 || A.mma_only == 5;   // 3, 5: probes without MMAs
        int g = 0;
        for (int it = cid; it < items; it += ncl) {
            const int s = it / A.ptiles, pt = it % A.ptiles;
            int t0, nt;
            range(s, t0, nt);
            const int p = pt * kT2N + (int)rank * kTcM + row;
            // (DBG: the selftest's raw accumulator dump - its own instantiation, so that the
            // division code stays out of the solver's epilogue loop and instruction cache)
            const bool dbg = DBG && A.debug_acc && leader && it == 0 && grp == 0 && hc * CW < kTcM;
            // seeded: the row shift sh_p (previous LSE + margin, folded by K6) is already
            // subtracted by the MMA: no running max (k_merge recomputes a point exactly if its
            // sum leaves [2^-100, 2^100]); unseeded: running max of t - sh_p
            float M = SEEDED ? 0.f : -INFINITY, S = 0.f;
            for (int i = 0; i < nt; ++i, ++g) {
                // tile group by the tile's index within the item (not the CTA's stream position):
                // which group sums which tiles - and so the item's result - is a function of the
                // item alone, whatever the launch's item schedule (bit-identity across world sizes)
                if (G > 1 && i % G != grp) continue;
                const int b = g & 1;
                mbar_wait_sleep(&tfull[b], (g >> 1) & 1);
                tc_fence_after();
                if (!full_epi) {   // K14 probes 1, 2, 4: the epilogue only releases the buffers
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(r_tempty + 8 * b);
                    continue;
                }
                const uint32_t taddr = tbase + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(b * kT2N + hc * CW);
                if constexpr (SEEDED && PL) {
                    // software-pipelined: 32-column chunks double-buffered in registers - the next
                    // chunk's tcgen05.ld is in flight while this chunk's exponentials run (the
                    // wait::ld at the end of an iteration only covers that one load)
                    uint32_t ra[32], rb[32];
                    TMEM_LD32(taddr, ra);
                    tmem_ld_wait();
#pragma unroll
                    for (int c = 0; c < CW / 32; c += 2) {
                        TMEM_LD32(taddr + (c + 1) * 32, rb);
                        {
                            const float2 sc = tc_sum_half<EMU>(ra);
                            S += sc.x + sc.y;
                        }
                        tmem_ld_wait();
                        if (c + 2 < CW / 32) TMEM_LD32(taddr + (c + 2) * 32, ra);
                        else {   // every load of accumulator b has retired: release it
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive_cluster(r_tempty + 8 * b);
                        }
                        {
                            const float2 sc = tc_sum_half<EMU>(rb);
                            S += sc.x + sc.y;
                        }
                        if (c + 2 < CW / 32) tmem_ld_wait();
                    }
                    continue;
                }
#pragma unroll
                for (int hh = 0; hh < CW / 64; ++hh) {   // 64-column chunks
                    uint32_t r[64];
                    if (A.mma_only == 5) {   // K14 probe: the epilogue's arithmetic without TMEM loads
#pragma unroll
                        for (int j = 0; j < 64; ++j) r[j] = __float_as_uint(-4.f - 0.01f * (float)((j + lane + i) & 15));
                    } else {
                        TMEM_LD32(taddr + hh * 64, r);
                        TMEM_LD32(taddr + hh * 64 + 32, (r + 32));
                        tmem_ld_wait();
                    }
                    if (hh == CW / 64 - 1) {
                        // accumulator b (this warp's columns) is in registers: release it
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive_cluster(r_tempty + 8 * b);
                    }
                    if (DBG && dbg && i == 0) {
#pragma unroll
                        for (int j = 0; j < 64; ++j)
                            A.debug_acc[row * kTcM + hc * CW + hh * 64 + j] = __fdiv_rn(__uint_as_float(r[j]), A.tk);
                    }
                    float2 tt[32];
#pragma unroll
                    for (int j = 0; j < 32; ++j) tt[j] = make_float2(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1]));
                    if constexpr (!SEEDED) {
                        float m8[8];
#pragma unroll
                        for (int j = 0; j < 8; ++j)
                            m8[j] = fmax3(fmaxf(tt[4 * j].x, tt[4 * j].y), fmax3(tt[4 * j + 1].x, tt[4 * j + 1].y, tt[4 * j + 2].x),
                                          fmax3(tt[4 * j + 2].y, tt[4 * j + 3].x, tt[4 * j + 3].y));
                        const float cm = fmax3(fmax3(m8[0], m8[1], m8[2]), fmax3(m8[3], m8[4], m8[5]), fmaxf(m8[6], m8[7]));
                        if (cm > M) { S *= ex2(M - cm); M = cm; }
                        if (M == -INFINITY) continue;  // only padding seen so far
                    }
                    const float2 sc = tc_sum_chunk<EMU, !SEEDED>(tt, M);
                    S += sc.x + sc.y;
                }
            }
            // combine the (tile, column) groups of each row in fixed order (h = 0, 1, ..)
            if (h > 0) xch[(h - 1) * kTcM + row] = make_float2(M, S);
            asm volatile("bar.sync 1, %0;" ::"r"(32 * NE));
            if (h == 0) {
#pragma unroll
                for (int k = 1; k < NQ; ++k) {
                    const float2 o = xch[(k - 1) * kTcM + row];
                    lse_merge(M, S, o.x, o.y);
                }
                if (p < A.P && !A.mma_only) A.part[(long long)s * A.P + p] = make_float2(M + sh[p], S);
            }
            asm volatile("bar.sync 1, %0;" ::"r"(32 * NE));   // xch reuse
        }
    }
    tc_fence_before();
    cluster_sync_all();
    if (A.cyc && blockIdx.x == 0 && threadIdx.x == 0) *A.cyc = clock64() - clk0;   // both CTAs done: no remote arrive or MMA still targets this CTA
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tbase));
    }
}

// ------------------------------------------------------------- K14 MMA probe
// Raw tcgen05.mma issue rate of one shape (M = 128, N, K = 32 bytes, SS operands on smem
// garbage), one CTA per SM, groups of 12 MMAs into alternating accumulators, at most two
// groups in flight.  Writes the SM cycles of CTA 0 (clock64) to cyc.  mode bits (diagnosis of
// the K3 loop): 1 = operands alternate between two A and two B images (hi/lo pattern);
// 2 = 24 MMAs per group into two accumulators; 4 = 8 extra warps wait on every group's
// completion barrier (as K3's epilogue warps do); 8 = they wait with a suspend-time hint.
template <int N, int TF32>
__global__ void __launch_bounds__(320, 1) k_mb_mma(int groups, int mode, long long *cyc) {
    extern __shared__ __align__(1024) unsigned char smraw[];
    unsigned char *sm = smraw + ((1024 - (smem_u32(smraw) & 1023)) & 1023);
    __shared__ __align__(8) uint64_t done[2];
    __shared__ uint32_t tmem_base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) { mbar_init(&done[0], 1); mbar_init(&done[1], 1); fence_mbar_init(); }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = tmem_base;
    constexpr uint32_t idesc = (1u << 4) | (TF32 ? ((2u << 7) | (2u << 10)) : 0u) | ((uint32_t)(N >> 3) << 17) |
                               ((uint32_t)(128 >> 4) << 24);
    const int per = (mode & 2) ? 24 : 12;
    long long c0 = clock64();
    if (warp == 0 && lane == 0) {
        const uint32_t a = smem_u32(sm), b = a + 32768;
        for (int g = 0; g < groups; ++g) {
            const int buf = g & 1;
            if (g >= 2) mbar_wait(&done[buf], ((g >> 1) - 1) & 1);
            tc_fence_after();
            for (int k = 0; k < per; ++k) {
                const uint32_t d = tb + (uint32_t)(buf * 2 * 128 + ((mode & 2) && k >= 12 ? 128 : 0));
                const uint32_t ko = (uint32_t)(k & 3) * 32;
                const uint32_t ao = (mode & 1) ? (uint32_t)((k & 1) * 16384) : 0u;
                const uint32_t bo = (mode & 1) ? (uint32_t)(((k >> 1) & 1) * 16384) : 0u;
                const uint64_t ad = umma_desc_sw128(a + ao + ko), bd = umma_desc_sw128(b + bo + ko);
                if constexpr (TF32)
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                        "l"(ad), "l"(bd), "r"(idesc), "r"((k % 12) > 0 ? 1 : 0));
                else
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                        "l"(ad), "l"(bd), "r"(idesc), "r"((k % 12) > 0 ? 1 : 0));
            }
            umma_commit(&done[buf]);
        }
        for (int g = groups - 2 > 0 ? groups - 2 : 0; g < groups; ++g) mbar_wait(&done[g & 1], (g >> 1) & 1);
    } else if (warp >= 2 && (mode & 4)) {
        for (int g = 0; g < groups; ++g) {
            if (mode & 8) mbar_wait_sleep(&done[g & 1], (g >> 1) & 1);
            else mbar_wait(&done[g & 1], (g >> 1) & 1);
        }
    }
    __syncthreads();
    long long c1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) *cyc = c1 - c0;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}

// flops per SM clock of the probe shape (kind & 3 -> 0: f16 N=128, 1: f16 N=256, 2: tf32 N=128,
// 3: tf32 N=256; kind >> 2 = mode bits)
cudaError_t microbench_mma(int kind, void *scratch, cudaStream_t st, double *flop_per_clk) {
    const int groups = 4096;
    const int mode = kind >> 2;
    long long *cyc = (long long *)scratch;
    const size_t smem = 1024 + 65536;
    int nsm = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    int N = 128, kk = 16;
#define SK_MMA_PROBE(NN, TF)                                                                              \
    {                                                                                                     \
        cudaError_t e = cudaFuncSetAttribute(k_mb_mma<NN, TF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        if (e != cudaSuccess) return e;                                                                   \
        k_mb_mma<NN, TF><<<nsm, 320, smem, st>>>(64, mode, cyc);                                          \
        k_mb_mma<NN, TF><<<nsm, 320, smem, st>>>(groups, mode, cyc);                                      \
        N = NN; kk = TF ? 8 : 16;                                                                         \
    }
    switch (kind & 3) {
        case 0: SK_MMA_PROBE(128, 0); break;
        case 1: SK_MMA_PROBE(256, 0); break;
        case 2: SK_MMA_PROBE(128, 1); break;
        default: SK_MMA_PROBE(256, 1); break;
    }
#undef SK_MMA_PROBE
    long long c = 0;
    cudaError_t e = cudaMemcpyAsync(&c, cyc, sizeof c, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return e;
    *flop_per_clk = 2.0 * 128 * N * kk * ((mode & 2) ? 24.0 : 12.0) * groups / (double)(c > 0 ? c : 1);
    return cudaGetLastError();
}


// --------------------------------------------------------------------- host side
size_t tc_image_bytes(long long P, int rb) { return (size_t)tc_side_bytes(P, rb); }

cudaError_t launch_absmax(const float *pts, long long cnt, unsigned *out, cudaStream_t st) {
    long long b = (cnt + 255) / 256;
    k_absmax<<<(int)(b > 148 * 8 ? 148 * 8 : (b < 1 ? 1 : b)), 256, 0, st>>>(pts, cnt, out);
    return cudaGetLastError();
}

cudaError_t launch_pack_tc(const float *pts, long long P, int d, const unsigned *amax2, int role, float eps,
                           void *img, cudaStream_t st, int rb) {
    if (!((rb % 128 == 0 && rb >= 128 && rb <= 512 && d <= rb / 2) || (rb == 32 && d <= 16))) return cudaErrorInvalidValue;
    const long long P2 = tc_tiles(P) * kTcM;   // zero images up to the pair tile
    const long long total = P2 * (rb / 16);
    long long b = (total + 255) / 256;
    k_pack_tc<<<(int)(b > 148 * 16 ? 148 * 16 : b), 256, 0, st>>>(pts, P, P2, d, amax2, role, 2.f * kLog2e / eps,
                                                                    (unsigned char *)img, rb);
    return cudaGetLastError();
}

cudaError_t launch_pack_tc_ext(long long P, const float *w, void *img, cudaStream_t st, int rb) {
    const long long P2 = tc_tiles(P) * kTcM;
    long long b = (P2 + 255) / 256;
    k_pack_tc_ext<<<(int)(b > 148 * 8 ? 148 * 8 : b), 256, 0, st>>>(P, P2, w, kTcFoldC, (unsigned char *)img, rb);
    return cudaGetLastError();
}

float tc_fold_c() { return kTcFoldC; }

bool tc_fold_ok(float amax_x, float amax_y, float eps) {
    // both scaled sides within fp16 range with headroom: max |alpha x|, max |alpha y| <= 2^13
    const float tk = 2.f * kLog2e / eps;
    if (!(tk > 0.f) || !std::isfinite(tk)) return false;
    const int s = tc_fold_s(amax_x, amax_y, tk);
    const double mx = amax_x > 0.f ? std::ldexp((double)amax_x, s) : 0.0;
    const double my = amax_y > 0.f ? (double)amax_y * tk * std::ldexp(1.0, -s) : 0.0;
    return mx <= 8192.0 && my <= 8192.0;
}

template <int EMU, int NE, bool SEEDED, int G, int PL = 0, bool DBG = false, int RB = 128, int KC = 1>
static cudaError_t launch_tc2(const TcArgs &A, int items, cudaStream_t st) {
    constexpr int ABUF = KC > 2 ? 1 : 2;
    constexpr int NBS = KC > 1 ? 2 : kT2Stages;
    constexpr size_t STAGE = 2 * (size_t)(128 * RB) + kTcExtBytes;
    constexpr size_t ASTAGE = 2 * (size_t)KC * (128 * RB) + kTcExtBytes;
    const size_t smem = 1024 + ABUF * ASTAGE + NBS * STAGE + (NE / 4 - 1) * kTcM * 8;
    static_assert(1024 + ABUF * ASTAGE + NBS * STAGE + (NE / 4 - 1) * kTcM * 8 <= 227 * 1024, "K3 shared memory");
    cudaError_t e = cudaFuncSetAttribute(k_lse_tc2<EMU, NE, SEEDED, G, PL, DBG, RB, KC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int nsm = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int ncl = std::max(1, std::min(items, nsm / 2));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * ncl);
    cfg.blockDim = dim3(64 + 32 * NE);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_lse_tc2<EMU, NE, SEEDED, G, PL, DBG, RB, KC>, A);
}

template <int EMU>
static cudaError_t launch_tc2_ne(const TcArgs &A, int items, bool seeded, int ne, int pipe, cudaStream_t st) {
    // epilogue organisation (sk_set_tuning "tc_epi"): 162 = 16 warps in two tile groups (even /
    // odd tiles, 128 columns per warp); 16 = four warps per TMEM lane quadrant on every tile
    if (seeded) {
        if (pipe && ne != 16) return launch_tc2<EMU, 16, true, 2, 1>(A, items, st);
        return ne == 16 ? launch_tc2<EMU, 16, true, 1>(A, items, st) : launch_tc2<EMU, 16, true, 2>(A, items, st);
    }
    return ne == 16 ? launch_tc2<EMU, 16, false, 1>(A, items, st) : launch_tc2<EMU, 16, false, 2>(A, items, st);
}

int tc_points_per_tile() { return kT2N; }

cudaError_t launch_lse_tc(const TcPass &L, cudaStream_t st) {
    // exponential pairs (of every 8) evaluated on the FMA pipe (sk_set_tuning "tc_emu")
    const int emu = L.emu, ne = L.epi;
    TcArgs A;
    A.Aimg = (const unsigned char *)L.Aimg; A.Bimg = (const unsigned char *)L.Bimg;
    A.P = L.P; A.Q = (int)L.Q; A.ksteps = L.ksteps;
    A.split_q = L.split_q;
    A.part = L.part; A.tk = 2.f * kLog2e / L.eps; A.stop = L.stop; A.only_if = L.only_if; A.debug_acc = L.debug_acc;
    A.mma_only = L.mma_only;
    A.cyc = L.cyc;
    if (A.ksteps < 1 || A.ksteps > 16) return cudaErrorInvalidValue;
    A.ptiles = (L.P + kT2N - 1) / kT2N;
    A.nblk = L.nblk;
    A.Qtiles = (int)((L.Q + kT2N - 1) / kT2N);
    A.blk_tiles = L.blk_tiles;
    const int items = A.ptiles * L.nblk * L.split_q;
    const bool seeded = L.seeded != 0;
    if (L.rb == 32) {
        // compact K = 16 images (d <= 16): the solver's variants (tc_emu 1..3, both epilogues)
        if (A.ksteps != 1) return cudaErrorInvalidValue;
        if (L.debug_acc) return launch_tc2<2, 16, false, 2, 0, true, 32>(A, items, st);   // (selftest)
        const bool g1 = ne == 16;
#define SK_TC32(E) \
        return seeded ? (g1 ? launch_tc2<E, 16, true, 1, 0, false, 32>(A, items, st) : launch_tc2<E, 16, true, 2, 0, false, 32>(A, items, st)) \
                      : (g1 ? launch_tc2<E, 16, false, 1, 0, false, 32>(A, items, st) : launch_tc2<E, 16, false, 2, 0, false, 32>(A, items, st));
        if (emu <= 1) { SK_TC32(1) }
        if (emu == 3) { SK_TC32(3) }
        SK_TC32(2)
#undef SK_TC32
    }
    if (L.rb > 128) {
        // d in (64, 256]: KC = rb / 128 K chunks; the MMAs grow with d while the epilogue does not,
        // so every exponential stays on MUFU (EMU 0) and the tile groups alternate (G = 2)
        const int kc = L.rb / 128;
        if (L.rb % 128 || kc > 4 || (A.ksteps + 3) / 4 != kc) return cudaErrorInvalidValue;
#define SK_TCK(KC) \
        return L.debug_acc ? launch_tc2<0, 16, false, 2, 0, true, 128, KC>(A, items, st) \
                           : (seeded ? launch_tc2<0, 16, true, 2, 0, false, 128, KC>(A, items, st) \
                                     : launch_tc2<0, 16, false, 2, 0, false, 128, KC>(A, items, st));
        if (kc == 2) { SK_TCK(2) }
        if (kc == 3) { SK_TCK(3) }
        SK_TCK(4)
#undef SK_TCK
    }
    if (A.ksteps > 4) return cudaErrorInvalidValue;
    if (L.debug_acc) return launch_tc2<2, 16, false, 2, 0, true>(A, items, st);   // (selftest)
    switch (emu) {
        case 0: return launch_tc2_ne<0>(A, items, seeded, ne, L.pipe, st);
        case 1: return launch_tc2_ne<1>(A, items, seeded, ne, L.pipe, st);
        case 3: return launch_tc2_ne<3>(A, items, seeded, ne, L.pipe, st);
        case 4: return launch_tc2_ne<4>(A, items, seeded, ne, L.pipe, st);
        case 5: return launch_tc2_ne<5>(A, items, seeded, ne, L.pipe, st);
        case 6: return launch_tc2_ne<6>(A, items, seeded, ne, L.pipe, st);
        default: return launch_tc2_ne<2>(A, items, seeded, ne, L.pipe, st);
    }
}

}  // namespace sk
