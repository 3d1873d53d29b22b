// sk_softsort.cu — K15: soft ranks and soft sort of batched 1D problems (Sec. 3.1, P:138-142;
// SURVEY.md NEXT-2), one extra weighted pass over the plan of a solved problem:
//     P_ij = exp((f_i + g_j - (x_i - y_j)^2) / eps)               (the plan of (f, g), Eq. (2))
//     rank_i = sum_j P_ij z_j / sum_j P_ij     ("n P z";   z_j = j + 1 by default)
//     sort_j = sum_i P_ij x_i / sum_i P_ij     ("n P^T x")
// (reading R-22: conditional means under the plan; equal to the paper's n P z and n P^T x
// whenever P has the uniform marginals, and insensitive to the marginal error of a finite-tol
// solve and to the last-bit noise of fp32 potentials, which 1/eps amplifies).
// One CTA per problem; x, y, f, g staged in shared memory; per output point two sweeps over the
// other side: the maximum exponent u = (f_i + g_j - d^2) log2(e)/eps (direct difference d, as
// the oracle's cost), then sum_j 2^(u - max) z_j and sum_j 2^(u - max): no overflow for any (f, g).
#include <algorithm>

#include "sk_internal.h"
#include "sk_common.cuh"

namespace sk {

constexpr int kSR = 512;

__global__ void __launch_bounds__(kSR) k_soft_rank_sort(const float *__restrict__ x, const float *__restrict__ y,
                                                        long long ys, const float *__restrict__ f,
                                                        const float *__restrict__ g, const float *__restrict__ z,
                                                        int n, int m, float eps, float *rank, float *sort) {
    extern __shared__ float sm[];
    float *xs = sm, *fs = xs + n, *ysm = fs + n, *gs = ysm + m, *zs = gs + m;
    const long long pr = blockIdx.x;
    const float kap = kLog2e / eps;
    for (int i = threadIdx.x; i < n; i += kSR) { xs[i] = x[pr * n + i]; fs[i] = f[pr * n + i]; }
    for (int j = threadIdx.x; j < m; j += kSR) {
        ysm[j] = y[pr * ys + j];
        gs[j] = g[pr * m + j];
        zs[j] = z ? z[j] : (float)(j + 1);
    }
    __syncthreads();
    if (rank) {
        for (int i = threadIdx.x; i < n; i += kSR) {
            const float xi = xs[i], fi = fs[i];
            float M = -INFINITY;
            for (int j = 0; j < m; ++j) {
                const float dd = xi - ysm[j];
                M = fmaxf(M, (fmaf(-dd, dd, fi + gs[j])) * kap);
            }
            float Sz = 0.f, S1 = 0.f;
            for (int j = 0; j < m; ++j) {
                const float dd = xi - ysm[j];
                const float e = ex2(fmaf(-dd, dd, fi + gs[j]) * kap - M);
                Sz = fmaf(e, zs[j], Sz);
                S1 += e;
            }
            rank[pr * n + i] = Sz / S1;
        }
    }
    if (sort) {
        for (int j = threadIdx.x; j < m; j += kSR) {
            const float yj = ysm[j], gj = gs[j];
            float M = -INFINITY;
            for (int i = 0; i < n; ++i) {
                const float dd = xs[i] - yj;
                M = fmaxf(M, (fmaf(-dd, dd, fs[i] + gj)) * kap);
            }
            float Sx = 0.f, S1 = 0.f;
            for (int i = 0; i < n; ++i) {
                const float dd = xs[i] - yj;
                const float e = ex2(fmaf(-dd, dd, fs[i] + gj) * kap - M);
                Sx = fmaf(e, xs[i], Sx);
                S1 += e;
            }
            sort[pr * m + j] = Sx / S1;
        }
    }
}

// Problems whose 2n + 3m floats exceed shared memory: the same two sweeps per output point with
// the other side read from global memory (every lane of a warp reads the same reduced point: one
// broadcast load per array), a grid of (output-point chunks, problems) per launch.
__global__ void __launch_bounds__(kSR) k_soft_rank_sort_g(const float *__restrict__ x, const float *__restrict__ y,
                                                          long long ys, const float *__restrict__ f,
                                                          const float *__restrict__ g, const float *__restrict__ z,
                                                          int n, int m, float eps, float *rank, float *sort) {
    const long long pr = blockIdx.y;
    const float kap = kLog2e / eps;
    const float *xr = x + pr * n, *fr = f + pr * n, *yr = y + pr * ys, *gr = g + pr * m;
    const int t = blockIdx.x * kSR + threadIdx.x;
    if (rank && t < n) {
        const float xi = xr[t], fi = fr[t];
        float M = -INFINITY;
        for (int j = 0; j < m; ++j) {
            const float dd = xi - __ldg(yr + j);
            M = fmaxf(M, (fmaf(-dd, dd, fi + __ldg(gr + j))) * kap);
        }
        float Sz = 0.f, S1 = 0.f;
        for (int j = 0; j < m; ++j) {
            const float dd = xi - __ldg(yr + j);
            const float e = ex2(fmaf(-dd, dd, fi + __ldg(gr + j)) * kap - M);
            Sz = fmaf(e, z ? __ldg(z + j) : (float)(j + 1), Sz);
            S1 += e;
        }
        rank[pr * n + t] = Sz / S1;
    }
    if (sort && t < m) {
        const float yj = yr[t], gj = gr[t];
        float M = -INFINITY;
        for (int i = 0; i < n; ++i) {
            const float dd = __ldg(xr + i) - yj;
            M = fmaxf(M, (fmaf(-dd, dd, __ldg(fr + i) + gj)) * kap);
        }
        float Sx = 0.f, S1 = 0.f;
        for (int i = 0; i < n; ++i) {
            const float xi = __ldg(xr + i);
            const float dd = xi - yj;
            const float e = ex2(fmaf(-dd, dd, __ldg(fr + i) + gj) * kap - M);
            Sx = fmaf(e, xi, Sx);
            S1 += e;
        }
        sort[pr * m + t] = Sx / S1;
    }
}

size_t soft_rank_sort_smem(int n, int m) { return sizeof(float) * (2 * (size_t)n + 3 * (size_t)m); }

cudaError_t launch_soft_rank_sort(long long B, int n, int m, const float *x, const float *y, long long ys,
                                  const float *f, const float *g, const float *z, float eps, float *rank,
                                  float *sort, cudaStream_t st) {
    const size_t smem = soft_rank_sort_smem(n, m);
    if (smem > 200 * 1024) {
        const int chunks = (std::max(n, m) + kSR - 1) / kSR;
        k_soft_rank_sort_g<<<dim3((unsigned)chunks, (unsigned)B), kSR, 0, st>>>(x, y, ys, f, g, z, n, m, eps, rank, sort);
        return cudaGetLastError();
    }
    cudaError_t e = cudaFuncSetAttribute(k_soft_rank_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_soft_rank_sort<<<(unsigned)B, kSR, smem, st>>>(x, y, ys, f, g, z, n, m, eps, rank, sort);
    return cudaGetLastError();
}

}  // namespace sk
