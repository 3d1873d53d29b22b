// sk_grid.cu — K20: one medium problem solved by one grid-persistent kernel.
//
// The subsample initializer's inner problem (Sec. 3.4: 4096 x 4096 at C4) is too large for
// one CTA's shared memory (K13) and too small for the multi-kernel path, whose six launches per
// sweep each fill only part of the GPU (57 us per sweep, ~7 us of it arithmetic).  K20 runs the
// whole solve in ONE cooperative launch, one CTA per SM, with a grid barrier between the passes:
//     column pass  g_j <- eps log b_j - eps LSE_i((f_i - C_ij)/eps)      (Alg. 1 l.5, R-1)
//     [err_l = sum_j b_j |expm1((g_j^l - g_j^{l+1})/eps)| every check_every sweeps (H5)]
//     row pass     f_i <- eps log a_i - eps LSE_j((g_j - C_ij)/eps)      (Alg. 1 l.4)
// the same sweep, stop rule and returned pair (f^l, g^l) as the on-chip solver K13.  Every CTA
// holds both point clouds in shared memory (static) and reloads the other side's w = (h -
// |q|^2) log2(e)/eps from L2 after each barrier; CTA c owns a fixed range of output points of
// each side (<= 32 per round: lane = output point, warp = slice of the reduction points, the 32
// slices' (M, S) combined in a fixed order).  Passes from the second sweep on are seeded (shift =
// the point's previous LSE + 4, no max), with the exact recompute of a point group whose sum left
// [2^-100, 2^100].  Deterministic: fixed ownership, fixed reduction shapes, and every CTA sums
// the per-CTA partials in CTA order (identical stop decisions everywhere).
#include "sk_internal.h"
#include "sk_lse_tile.cuh"

#include <algorithm>

namespace sk {

namespace {

constexpr int kGT = 1024;               // threads per CTA (32 warps = 32 reduction slices)
constexpr int kGW = kGT / 32;
constexpr float kGSeedMargin = 4.f;     // log2 units above the previous LSE (as K13)

struct GridArgs {
    int n, m;
    const float *x, *y;                 // [n][d], [m][d]
    const float *a, *b;                 // nullable: uniform weights
    const float *finit;                 // nullable: f^0 = 0
    float eps, tol;
    int max_iter, check_every;
    float *fbuf, *gbuf;                 // [2][n], [2][m]: (f^l, g^l) in buffer l & 1
    float *wxg, *wyg;                   // [n], [m]: the published w of the last pass
    float *sx, *sy;                     // [n], [m]: per-point LSE seeds (owner only)
    double *part;                       // [2][G][2] per-CTA partials (double-buffered)
    unsigned *bar;                      // [2] barrier count, generation
    float *f, *g;                       // outputs
    GridResult *res;
};

__host__ __device__ inline int rup(int v, int a) { return (v + a - 1) / a * a; }

// Grid barrier (all CTAs co-resident: cooperative launch).  The CTA barrier orders the CTA's
// global writes before thread 0's device-scope fence; readers load published data with
// ld.global.cg (L2), never from a stale L1 line.
__device__ __forceinline__ void grid_barrier(unsigned *bar, unsigned G) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned *gen = bar + 1;
        const unsigned g0 = *gen;
        __threadfence();
        if (atomicAdd(bar, 1u) == G - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*gen == g0) {
            }
        }
        __threadfence();
    }
    __syncthreads();
}

// One pass over this CTA's output points [p0, p1) (P side coords pc [D][Pp] in smem) against
// all reduction points (qc [D][Qp], qw [Qp] in smem).  out(p, M, S) runs on warp 0, lane = p - pb.
template <int D, int EMU, typename Out>
__device__ __forceinline__ void grid_pass(const float *__restrict__ pc, int Pp, int p0, int p1,
                                          const float *__restrict__ qc, const float *__restrict__ qw, int Qp,
                                          float tk, float *seed, bool seeded, float2 *red, int *sflag, Out out) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int qs = rup((Qp + kGW - 1) / kGW, kChunk);
    const int q0 = w * qs, q1 = min(Qp, q0 + qs);
    for (int pb = p0; pb < p1; pb += 32) {
        const int p = pb + lane;
        const bool valid = p < p1;
        float2 pd[1][D];
#pragma unroll
        for (int k = 0; k < D; ++k) {
            const float v = valid ? pc[k * Pp + p] * tk : 0.f;
            pd[0][k] = make_float2(v, v);
        }
        bool sd = seeded;
        for (;;) {   // (at most twice: a seeded group whose sum left the safe range is redone exactly)
            float M[1];
            float2 S[1] = {make_float2(0.f, 0.f)};
            M[0] = sd ? (valid ? __ldcg(seed + p) + kGSeedMargin : 0.f) : -INFINITY;
            if (sd) {
                for (int q = q0; q < q1; q += kChunk) lse_chunk_seeded<D, 1, EMU>(qc, Qp, qw, q, pd, M, S);
            } else {
                for (int q = q0; q < q1; q += kChunk) lse_chunk<D, 1, EMU>(qc, Qp, qw, q, pd, M, S);
            }
            red[w * 32 + lane] = make_float2(M[0], S[0].x + S[0].y);
            __syncthreads();
            int fail = 0;
            float Mx = -INFINITY, Sx = 0.f;
            if (w == 0) {
                if (sd) {
                    Mx = red[lane].x;
                    for (int u = 0; u < kGW; ++u) Sx += red[u * 32 + lane].y;
                    fail = valid && !(Sx >= 0x1p-100f && Sx <= 0x1p100f);
                } else {
                    for (int u = 0; u < kGW; ++u) Mx = fmaxf(Mx, red[u * 32 + lane].x);
                    if (Mx > -INFINITY)
                        for (int u = 0; u < kGW; ++u) {
                            const float2 v = red[u * 32 + lane];
                            Sx += v.y * ex2(v.x - Mx);
                        }
                }
                fail = __any_sync(0xffffffffu, fail);
                if (lane == 0) *sflag = fail;
            }
            __syncthreads();   // (red is rewritten by the next round; sflag read below)
            if (*sflag) {      // CTA-uniform
                __syncthreads();
                sd = false;
                continue;
            }
            if (w == 0 && valid) {
                seed[p] = Mx + log2f(Sx);   // this sweep's LSE: the next sweep's seed
                out(p, Mx, Sx);
            }
            break;
        }
    }
}

template <int D, int EMU>
__global__ void __launch_bounds__(kGT, 1) k_grid_solve(GridArgs A) {
    extern __shared__ __align__(16) float sm[];
    __shared__ double s_red[2];
    __shared__ int s_flag;
    const int n = A.n, m = A.m, G = gridDim.x, c = blockIdx.x;
    const int Np = rup(n, kChunk), Mp = rup(m, kChunk);
    float *xq = sm;                 // [D][Np]
    float *yq = xq + D * Np;        // [D][Mp]
    float *wx = yq + D * Mp;        // [Np]
    float *wy = wx + Np;            // [Mp]
    float2 *red = reinterpret_cast<float2 *>(wy + Mp + ((Np + Mp) & 1));   // [32][32]
    const float eps = A.eps, kap = kLog2e / eps, tk = 2.f * kap, epsln2 = eps * kLn2;
    const float loga_u = (float)(-log((double)n)), logb_u = (float)(-log((double)m));
    // output ranges: ceil(P / G) points per CTA
    const int ci = (n + G - 1) / G, cj = (m + G - 1) / G;
    const int i0 = min(n, c * ci), i1 = min(n, i0 + ci);
    const int j0 = min(m, c * cj), j1 = min(m, j0 + cj);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;

    // ---- load (K1): both clouds, w of x from f^0; padding q's carry w = -inf
    for (int i = threadIdx.x; i < Np; i += kGT) {
        if (i < n) {
            float s = 0.f;
#pragma unroll
            for (int k = 0; k < D; ++k) {
                const float v = A.x[(size_t)i * D + k];
                xq[k * Np + i] = v;
                s = fmaf(v, v, s);
            }
            const float f0 = A.finit ? A.finit[i] : 0.f;
            wx[i] = fmaf(f0, kap, -s * kap);
            if (i >= i0 && i < i1) A.fbuf[i] = f0;
        } else {
#pragma unroll
            for (int k = 0; k < D; ++k) xq[k * Np + i] = 0.f;
            wx[i] = -INFINITY;
        }
    }
    for (int j = threadIdx.x; j < Mp; j += kGT) {
        if (j < m) {
#pragma unroll
            for (int k = 0; k < D; ++k) yq[k * Mp + j] = A.y[(size_t)j * D + k];
            if (j >= j0 && j < j1) A.gbuf[j] = 0.f;   // g^(0) = 0 (only f^(0) is needed)
        } else {
#pragma unroll
            for (int k = 0; k < D; ++k) yq[k * Mp + j] = 0.f;
            wy[j] = -INFINITY;
        }
    }
    __syncthreads();
    auto sqn = [&](const float *q, int stride, int p) {
        float s = 0.f;
#pragma unroll
        for (int k = 0; k < D; ++k) s = fmaf(q[k * stride + p], q[k * stride + p], s);
        return s;
    };
    // fixed-order sum of the G CTAs' partials (every CTA computes the same bits)
    auto grid_sum = [&](const double *pp) {
        if (w == 0) {
            double e = 0.0, bd = 0.0;
            for (int u = lane; u < G; u += 32) { e += __ldcg(pp + 2 * u); bd += __ldcg(pp + 2 * u + 1); }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                e += __shfl_xor_sync(0xffffffffu, e, o);
                bd += __shfl_xor_sync(0xffffffffu, bd, o);
            }
            if (lane == 0) { s_red[0] = e; s_red[1] = bd; }
        }
        __syncthreads();
    };
    auto warp_put = [&](double *pp, double e, double bd) {   // warp 0: this CTA's partial
        if (w == 0) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                e += __shfl_xor_sync(0xffffffffu, e, o);
                bd += __shfl_xor_sync(0xffffffffu, bd, o);
            }
            if (lane == 0) { pp[2 * c] = e; pp[2 * c + 1] = bd; }
        }
    };

    int l = 0, cur = 0, conv = 0, nonfin = 0, pass = 0;
    float err = INFINITY;
    for (;;) {
        const bool seeded = l >= 1;
        const bool check = l >= 1 && (l % A.check_every == 0 || l == A.max_iter);
        // ---- column pass: g^{l+1} (P = y, Q = x)
        const float *gold = A.gbuf + cur * m;
        float *gnew = A.gbuf + (cur ^ 1) * m;
        double e_loc = 0.0, bad = 0.0;
        grid_pass<D, EMU>(yq, Mp, j0, j1, xq, wx, Np, tk, A.sy, seeded, red, &s_flag, [&](int j, float Mv, float Sv) {
            const float s = sqn(yq, Mp, j);
            const float lb = A.b ? logf(A.b[j]) : logb_u;
            const float gsk = fmaf(eps, lb, s) - epsln2 * (Mv + log2f(Sv));
            gnew[j] = gsk;
            A.wyg[j] = fmaf(gsk, kap, -s * kap);
            bad += !isfinite(gsk) ? 1.0 : 0.0;
            if (check) {
                const double bj = A.b ? (double)A.b[j] : 1.0 / m;
                e_loc += bj * fabs((double)expm1f((__ldcg(gold + j) - gsk) / eps));
            }
        });
        double *pp = A.part + (size_t)(pass & 1) * 2 * G;
        warp_put(pp, e_loc, bad);
        ++pass;
        grid_barrier(A.bar, G);
        grid_sum(pp);
        if (s_red[1] != 0.0) { nonfin = 1; break; }
        if (check) {
            err = (float)s_red[0];
            if (err < A.tol) { conv = 1; break; }
        }
        if (l >= A.max_iter) break;
        // ---- row pass: f^{l+1} (P = x, Q = y); w of y from L2
        for (int j = threadIdx.x; j < m; j += kGT) wy[j] = __ldcg(A.wyg + j);
        __syncthreads();
        float *fnew = A.fbuf + (cur ^ 1) * n;
        bad = 0.0;
        grid_pass<D, EMU>(xq, Np, i0, i1, yq, wy, Mp, tk, A.sx, seeded, red, &s_flag, [&](int i, float Mv, float Sv) {
            const float s = sqn(xq, Np, i);
            const float la = A.a ? logf(A.a[i]) : loga_u;
            const float fsk = fmaf(eps, la, s) - epsln2 * (Mv + log2f(Sv));
            fnew[i] = fsk;
            A.wxg[i] = fmaf(fsk, kap, -s * kap);
            bad += !isfinite(fsk) ? 1.0 : 0.0;
        });
        pp = A.part + (size_t)(pass & 1) * 2 * G;
        warp_put(pp, 0.0, bad);
        ++pass;
        grid_barrier(A.bar, G);
        grid_sum(pp);
        if (s_red[1] != 0.0) { nonfin = 1; break; }
        for (int i = threadIdx.x; i < n; i += kGT) wx[i] = __ldcg(A.wxg + i);
        __syncthreads();
        cur ^= 1;
        ++l;
    }

    // ---- epilogue: (f^l, g^l) and E = <f,a> + <g,b> - eps sum(a) (Eq. 2 after an f-update)
    const float *fo = A.fbuf + cur * n, *go = A.gbuf + cur * m;
    double s = 0.0;
    for (int i = i0 + threadIdx.x; i < i1; i += kGT) {
        const float fv = __ldcg(fo + i);
        A.f[i] = fv;
        const double ai = A.a ? (double)A.a[i] : 1.0 / n;
        s += (double)fv * ai - (double)eps * ai;
    }
    for (int j = j0 + threadIdx.x; j < j1; j += kGT) {
        const float gv = __ldcg(go + j);
        A.g[j] = gv;
        s += (double)gv * (A.b ? (double)A.b[j] : 1.0 / m);
    }
    // fixed-shape CTA sum (warp sums, then warp 0 over the 32 warps in order)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    double *ws = reinterpret_cast<double *>(red);
    __syncthreads();
    if (lane == 0) ws[w] = s;
    __syncthreads();
    double *pp = A.part + (size_t)(pass & 1) * 2 * G;
    if (w == 0) {
        double t = lane < kGW ? ws[lane] : 0.0;
        warp_put(pp, t, 0.0);
    }
    grid_barrier(A.bar, G);
    grid_sum(pp);
    if (c == 0 && threadIdx.x == 0) {
        A.res->E = s_red[0];
        A.res->iterations = l;
        A.res->converged = conv;
        A.res->nonfinite = nonfin;
        A.res->err = err;
    }
}

template <int D>
size_t grid_smem(int n, int m) {
    const int Np = rup(n, kChunk), Mp = rup(m, kChunk);
    return sizeof(float) * ((size_t)(D + 1) * (Np + Mp) + 2) + sizeof(float2) * 32 * 32;
}

template <int D>
cudaError_t launch_grid_d(GridArgs A, int nsm, cudaStream_t st) {
    const size_t smem = grid_smem<D>(A.n, A.m);
    auto kern = k_grid_solve<D, 1>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kGT, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    void *args[] = {&A};
    return cudaLaunchCooperativeKernel((const void *)kern, dim3(nsm), dim3(kGT), args, smem, st);
}

}  // namespace

size_t grid_solver_smem(int d, int n, int m) {
    switch (d) {
        case 1: return grid_smem<1>(n, m);
        case 2: return grid_smem<2>(n, m);
        case 3: return grid_smem<3>(n, m);
        case 4: return grid_smem<4>(n, m);
        default: return ~(size_t)0;
    }
}

bool grid_solver_supported(int d, int n, int m) {
    return d >= 1 && d <= 4 && n >= 1 && m >= 1 && grid_solver_smem(d, n, m) <= 200 * 1024;
}

size_t grid_solver_workspace_bytes(int n, int m, int nsm) {
    return 64 + sizeof(double) * 4 * (size_t)nsm + sizeof(float) * 6 * ((size_t)n + m) + 64;
}

cudaError_t launch_grid_solver(const GridLaunch &L, cudaStream_t st) {
    if (!grid_solver_supported(L.d, L.n, L.m)) return cudaErrorInvalidValue;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    // workspace (grid_solver_workspace_bytes): result, barrier, partials, then the float arrays
    char *q = static_cast<char *>(L.work);
    GridArgs A;
    A.res = reinterpret_cast<GridResult *>(q);
    A.bar = reinterpret_cast<unsigned *>(q + 48);
    q += 64;
    A.part = reinterpret_cast<double *>(q); q += sizeof(double) * 4 * (size_t)nsm;
    float *fq = reinterpret_cast<float *>(q);
    A.fbuf = fq; fq += 2 * (size_t)L.n;
    A.gbuf = fq; fq += 2 * (size_t)L.m;
    A.wxg = fq; fq += L.n;
    A.wyg = fq; fq += L.m;
    A.sx = fq; fq += L.n;
    A.sy = fq;
    A.n = L.n; A.m = L.m;
    A.x = L.x; A.y = L.y; A.a = L.a; A.b = L.b; A.finit = L.finit;
    A.eps = L.eps; A.tol = L.tol; A.max_iter = L.max_iter; A.check_every = L.check_every;
    A.f = L.f; A.g = L.g;
    cudaError_t e = cudaMemsetAsync(A.bar, 0, 4 * sizeof(unsigned), st);
    if (e != cudaSuccess) return e;
    switch (L.d) {
        case 1: e = launch_grid_d<1>(A, nsm, st); break;
        case 2: e = launch_grid_d<2>(A, nsm, st); break;
        case 3: e = launch_grid_d<3>(A, nsm, st); break;
        case 4: e = launch_grid_d<4>(A, nsm, st); break;
        default: return cudaErrorInvalidValue;
    }
    if (e != cudaSuccess) return e;
    if (L.res_host) e = cudaMemcpyAsync(L.res_host, A.res, sizeof(GridResult), cudaMemcpyDeviceToHost, st);
    return e;
}

}  // namespace sk
