// sk_gauss.cu — K10 (Gaussian initializer) and K11 (GMM initializer).
//
// Gaussian (Sec. 3.2):
//   moments  m = sum_i w_i x_i,  S = sum_i w_i (x_i - m)(x_i - m)^T (+ ridge, R-11)
//            two passes, fp64 per-block partials, fixed-order final sums;
//   A = S_mu^{-1/2} (S_mu^{1/2} S_nu S_mu^{1/2})^{1/2} S_mu^{-1/2}
//            with fp64 coupled Newton-Schulz square roots (budget R-12)
//            in one CTA (d > 64: over the whole grid, one cooperative launch);
//   f*(x) = ||x||^2 - (x - m_mu)^T A (x - m_mu) - 2 m_nu^T x   (R-4).
// GMM (Sec. 3.3):
//   C~_kl = ||m_k - m'_l||^2 + tr(S_k + S'_l - 2 (S_k^{1/2} S'_l S_k^{1/2})^{1/2})  (Eq. 6)
//            one CTA per square root (batched NS);
//   f~ from the K x K entropic problem at the same eps (R-13), fp64, one CTA;
//   f^(0)(x) = sum_k f~_k p_k(x),  p_k = alpha_k N(x; m_k, S_k) / sum_l (...)  (Eq. 7),
//            log-domain with Cholesky factors, fp64.
//   d > 64: the per-component / per-pair matrices in global-memory slots (L2) instead of
//   shared memory.
#include <cooperative_groups.h>

#include <algorithm>

#include "sk_internal.h"
#include "sk_common.cuh"

namespace sk {

constexpr int kGT = 256;

// ------------------------------------------------------------- moments
// out[blk][E]: E = d (pass 1, mean == nullptr) or d*d (pass 2, centred by mean).  Pass 2: the
// 16 x 16 threads each own a TI x TI block of entries (rows br + 16 i, columns bc + 16 j, TI =
// ceil(d / 16): per chunk row, TI broadcast + TI conflict-free shared loads feed TI^2 FMAs).
template <int TI>
__global__ void __launch_bounds__(kGT) k_moment_partials(const float *__restrict__ x,
                                                         const float *__restrict__ w, long long n,
                                                         int d, const double *__restrict__ mean,
                                                         double *out) {
    constexpr int CH = 64;
    extern __shared__ double xs[];  // [CH][d] weighted/centred chunk, then [CH] weights
    double *ws = xs + CH * d;
    const long long per = (n + gridDim.x - 1) / gridDim.x;
    const long long lo = blockIdx.x * per, hi = min(n, lo + per);
    const int br = threadIdx.x >> 4, bc = threadIdx.x & 15;
    double acc[TI * TI];
#pragma unroll
    for (int t = 0; t < TI * TI; ++t) acc[t] = 0.0;
    for (long long c0 = lo; c0 < hi; c0 += CH) {
        const int cnt = (int)min((long long)CH, hi - c0);
        __syncthreads();
        for (int t = threadIdx.x; t < cnt * d; t += kGT) {
            const int r = t / d, k = t % d;
            const double v = x[(c0 + r) * d + k];
            xs[r * d + k] = mean ? v - mean[k] : v;
        }
        for (int r = threadIdx.x; r < cnt; r += kGT) ws[r] = w ? (double)w[c0 + r] : 1.0 / n;
        __syncthreads();
        if (mean) {
            for (int r = 0; r < cnt; ++r) {
                const double *xr = xs + r * d;
                const double wr = ws[r];
                double a[TI], b[TI];
#pragma unroll
                for (int i = 0; i < TI; ++i) a[i] = br + 16 * i < d ? wr * xr[br + 16 * i] : 0.0;
#pragma unroll
                for (int j = 0; j < TI; ++j) b[j] = bc + 16 * j < d ? xr[bc + 16 * j] : 0.0;
#pragma unroll
                for (int i = 0; i < TI; ++i)
#pragma unroll
                    for (int j = 0; j < TI; ++j) acc[TI * i + j] = fma(a[i], b[j], acc[TI * i + j]);
            }
        } else if (threadIdx.x < d) {
            double sm = 0.0;
            for (int r = 0; r < cnt; ++r) sm += ws[r] * xs[r * d + threadIdx.x];
            acc[0] += sm;
        }
    }
    if (mean) {
#pragma unroll
        for (int i = 0; i < TI; ++i)
#pragma unroll
            for (int j = 0; j < TI; ++j) {
                const int k = br + 16 * i, l = bc + 16 * j;
                if (k < d && l < d) out[(long long)blockIdx.x * d * d + k * d + l] = acc[TI * i + j];
            }
    } else if (threadIdx.x < d) {
        out[(long long)blockIdx.x * d + threadIdx.x] = acc[0];
    }
}

// Fixed-order sum over the nb block partials: 8 warps split the blocks (block b to warp b % 8, in
// order), then the 8 warp sums in warp order; 32 entries per CTA (lane = entry).
__global__ void __launch_bounds__(256) k_reduce_cols(const double *in, int nb, int E, double *out) {
    __shared__ double ps[8][32];
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    const int e = blockIdx.x * 32 + lane;
    double s = 0.0;
    if (e < E)
        for (int b = wp; b < nb; b += 8) s += in[(long long)b * E + e];
    ps[wp][lane] = s;
    __syncthreads();
    if (wp == 0 && e < E) {
        double t = 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) t += ps[u][lane];
        out[e] = t;
    }
}

// d in (64, 256]: the covariance partials per (64 x 64 output tile, row block): the tile's 64
// weighted centred columns and 64 centred columns of a 32-row chunk staged in shared memory;
// thread (br, bc) of 16 x 16 owns entries (i0 + br + 16 i, j0 + bc + 16 j), i, j < 4, each summed
// over the block's rows in order (as the d <= 64 kernel).
__global__ void __launch_bounds__(kGT) k_cov_partials_wide(const float *__restrict__ x, const float *__restrict__ w,
                                                           long long n, int d, const double *__restrict__ mean,
                                                           double *out) {
    constexpr int CH = 32;   // rows per chunk (64 columns per side: 33 KB of static shared memory)
    __shared__ double xa[CH][65], xb[CH][65], ws[CH];
    const int nt = (d + 63) / 64;
    const int i0 = (blockIdx.x / nt) * 64, j0 = (blockIdx.x % nt) * 64;
    const long long per = (n + gridDim.y - 1) / gridDim.y;
    const long long lo = blockIdx.y * per, hi = min(n, lo + per);
    const int br = threadIdx.x >> 4, bc = threadIdx.x & 15;
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    for (long long c0 = lo; c0 < hi; c0 += CH) {
        const int cnt = (int)min((long long)CH, hi - c0);
        __syncthreads();
        for (int t = threadIdx.x; t < cnt * 64; t += kGT) {
            const int r = t / 64, k = t % 64;
            const long long row = (c0 + r) * d;
            xa[r][k] = i0 + k < d ? (double)x[row + i0 + k] - mean[i0 + k] : 0.0;
            xb[r][k] = j0 + k < d ? (double)x[row + j0 + k] - mean[j0 + k] : 0.0;
        }
        for (int r = threadIdx.x; r < cnt; r += kGT) ws[r] = w ? (double)w[c0 + r] : 1.0 / n;
        __syncthreads();
        for (int r = 0; r < cnt; ++r) {
            const double wr = ws[r];
            double a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = wr * xa[r][br + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = xb[r][bc + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
    }
    double *o = out + (long long)blockIdx.y * d * d;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int k = i0 + br + 16 * i, l = j0 + bc + 16 * j;
            if (k < d && l < d) o[k * d + l] = acc[i][j];
        }
}

long long moments_blocks(int d) { return d <= 64 ? 296 : std::max(1, 592 / (((d + 63) / 64) * ((d + 63) / 64))); }

cudaError_t launch_moments(const float *x, const float *w, long long n, int d, double *mean,
                           double *cov, double *scratch, long long scratch_doubles, cudaStream_t st) {
    if (d > 256) return cudaErrorInvalidValue;
    if (d > 64) {
        long long nb = std::min((n + 63) / 64, moments_blocks(d));
        if (nb * d * d > scratch_doubles) nb = scratch_doubles / ((long long)d * d);
        if (nb < 1) return cudaErrorInvalidValue;
        const size_t smem = (64 * (size_t)d + 64) * sizeof(double);
        cudaError_t e = cudaFuncSetAttribute(k_moment_partials<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        k_moment_partials<1><<<(int)nb, kGT, smem, st>>>(x, w, n, d, nullptr, scratch);   // (pass 1: d <= 256 threads)
        k_reduce_cols<<<(d + 31) / 32, 256, 0, st>>>(scratch, (int)nb, d, mean);
        const int nt = (d + 63) / 64;
        k_cov_partials_wide<<<dim3((unsigned)(nt * nt), (unsigned)nb), kGT, 0, st>>>(x, w, n, d, mean, scratch);
        k_reduce_cols<<<(d * d + 31) / 32, 256, 0, st>>>(scratch, (int)nb, d * d, cov);
        return cudaGetLastError();
    }
    long long nb = (n + 63) / 64;   // one 64-point chunk per CTA up to 296 CTAs (a fixed partition of n)
    if (nb > 296) nb = 296;
    if (nb * d * d > scratch_doubles) nb = scratch_doubles / (d * d);
    if (nb < 1) return cudaErrorInvalidValue;
    const size_t smem = (64 * (size_t)d + 64) * sizeof(double);
    auto kern = d <= 16 ? k_moment_partials<1> : d <= 32 ? k_moment_partials<2>
              : d <= 48 ? k_moment_partials<3> : k_moment_partials<4>;
    kern<<<(int)nb, kGT, smem, st>>>(x, w, n, d, nullptr, scratch);
    k_reduce_cols<<<(d + 31) / 32, 256, 0, st>>>(scratch, (int)nb, d, mean);
    kern<<<(int)nb, kGT, smem, st>>>(x, w, n, d, mean, scratch);
    k_reduce_cols<<<(d * d + 31) / 32, 256, 0, st>>>(scratch, (int)nb, d * d, cov);
    return cudaGetLastError();
}

// ----------------------------------------------------- fp64 dense helpers
// C = A * B (d x d, smem, d <= 64), blockDim.x == 256; C must not alias A or B.  Thread (br, bc)
// of 16 x 16 owns C[br + 16 i][bc + 16 j], i, j < TI = ceil(d / 16): per k, TI broadcast loads
// of A and TI conflict-free loads of B feed TI^2 FMAs; each entry sums over k in order.
template <int TI>
__device__ __forceinline__ void mm_t(const double *A, const double *B, double *C, int d) {
    const int br = threadIdx.x >> 4, bc = threadIdx.x & 15;
    double acc[TI][TI];
#pragma unroll
    for (int i = 0; i < TI; ++i)
#pragma unroll
        for (int j = 0; j < TI; ++j) acc[i][j] = 0.0;
    if (br < d && bc < d) {
#pragma unroll 4
        for (int k = 0; k < d; ++k) {
            double a[TI], b[TI];
#pragma unroll
            for (int i = 0; i < TI; ++i) a[i] = br + 16 * i < d ? A[(br + 16 * i) * d + k] : 0.0;
#pragma unroll
            for (int j = 0; j < TI; ++j) b[j] = bc + 16 * j < d ? B[k * d + bc + 16 * j] : 0.0;
#pragma unroll
            for (int i = 0; i < TI; ++i)
#pragma unroll
                for (int j = 0; j < TI; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
#pragma unroll
        for (int i = 0; i < TI; ++i)
#pragma unroll
            for (int j = 0; j < TI; ++j)
                if (br + 16 * i < d && bc + 16 * j < d) C[(br + 16 * i) * d + bc + 16 * j] = acc[i][j];
    }
}

__device__ void mm(const double *A, const double *B, double *C, int d) {
    if (d <= 16) mm_t<1>(A, B, C, d);
    else if (d <= 32) mm_t<2>(A, B, C, d);
    else if (d <= 48) mm_t<3>(A, B, C, d);
    else mm_t<4>(A, B, C, d);
    __syncthreads();
}

__device__ double block_sum_any(double v, double *red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    __syncthreads();
    return s;
}

// Coupled Newton-Schulz: Y -> M^{1/2}, Z -> M^{-1/2} for SPD M (d x d, smem).
// Y_0 = M/||M||_F, Z_0 = I;  T = (3I - Z Y)/2;  Y <- Y T;  Z <- T Z.
// Stops when ||Z Y - I||_F < 1e-13 * d or the residual stagnates below 1e-7; max 100 sweeps
// (R-12).  Small eigenvalues lam of M/||M||_F need ~log(1/lam)/log(2.25) sweeps to enter the
// quadratic phase.
// Work: T, U (d x d).  Returns the final residual.
__device__ double ns_sqrt(const double *M, double *Y, double *Z, double *T, double *U, int d,
                          double *red) {
    double fr = 0.0;
    for (int e = threadIdx.x; e < d * d; e += blockDim.x) fr += M[e] * M[e];
    const double nrm = sqrt(block_sum_any(fr, red));
    for (int e = threadIdx.x; e < d * d; e += blockDim.x) {
        Y[e] = M[e] / nrm;
        Z[e] = (e / d == e % d) ? 1.0 : 0.0;
    }
    __syncthreads();
    double res = INFINITY, prev = INFINITY;
    for (int it = 0; it < 100; ++it) {
        mm(Z, Y, T, d);  // T = Z Y
        double r = 0.0;
        for (int e = threadIdx.x; e < d * d; e += blockDim.x) {
            const double v = T[e] - ((e / d == e % d) ? 1.0 : 0.0);
            r += v * v;
            T[e] = ((e / d == e % d) ? 1.5 : 0.0) - 0.5 * T[e];
        }
        res = sqrt(block_sum_any(r, red));
        // converged, or stagnated at the fp64 rounding floor (quadratic phase reached)
        if (res < 1e-13 * d || (res < 1e-7 && res > 0.5 * prev)) break;
        prev = res;
        mm(Y, T, U, d);  // U = Y T
        for (int e = threadIdx.x; e < d * d; e += blockDim.x) Y[e] = U[e];
        __syncthreads();
        mm(T, Z, U, d);  // U = T Z
        for (int e = threadIdx.x; e < d * d; e += blockDim.x) Z[e] = U[e];
        __syncthreads();
    }
    const double sq = sqrt(nrm);
    for (int e = threadIdx.x; e < d * d; e += blockDim.x) {
        Y[e] *= sq;
        Z[e] /= sq;
    }
    __syncthreads();
    return res;
}

__device__ void symmetrize(double *A, int d) {
    for (int e = threadIdx.x; e < d * d; e += blockDim.x) {
        const int i = e / d, j = e % d;
        if (i < j) {
            const double v = 0.5 * (A[i * d + j] + A[j * d + i]);
            A[i * d + j] = v;
            A[j * d + i] = v;
        }
    }
    __syncthreads();
}

// One CTA: ridge, NS square roots, A.  cov_* are modified in place (ridge added).
__global__ void __launch_bounds__(kGT) k_gauss_A(double *cov_mu, double *cov_nu, int d, float ridge_rel,
                                                  double *Aout, int *ns_fail) {
    extern __shared__ double sm[];
    __shared__ double red[kGT / 32];
    const int dd = d * d;
    double *Smu = sm, *Snu = sm + dd, *R = sm + 2 * dd, *Ri = sm + 3 * dd, *T = sm + 4 * dd,
           *U = sm + 5 * dd;
    double tr_mu = 0.0, tr_nu = 0.0;
    for (int k = 0; k < d; ++k) { tr_mu += cov_mu[k * d + k]; tr_nu += cov_nu[k * d + k]; }
    for (int e = threadIdx.x; e < dd; e += blockDim.x) {
        const bool diag = e / d == e % d;
        Smu[e] = cov_mu[e] + (diag ? ridge_rel * tr_mu / d : 0.0);
        Snu[e] = cov_nu[e] + (diag ? ridge_rel * tr_nu / d : 0.0);
    }
    __syncthreads();
    symmetrize(Smu, d);
    symmetrize(Snu, d);
    const double r1 = ns_sqrt(Smu, R, Ri, T, U, d, red);  // R = S_mu^{1/2}, Ri = S_mu^{-1/2}
    mm(R, Snu, T, d);                                     // T = R S_nu
    double *Mm = Smu;                                     // S_mu no longer needed
    mm(T, R, Mm, d);                                      // Mm = R S_nu R
    symmetrize(Mm, d);
    double *Q = Snu, *Qi = R;                             // S_nu, R no longer needed
    const double r2 = ns_sqrt(Mm, Q, Qi, T, U, d, red);  // Q = Mm^{1/2}
    mm(Ri, Q, T, d);
    mm(T, Ri, U, d);                                      // A = Ri Q Ri
    symmetrize(U, d);
    for (int e = threadIdx.x; e < dd; e += blockDim.x) Aout[e] = U[e];
    if (threadIdx.x == 0) *ns_fail = (r1 > 1e-6 || r2 > 1e-6 || !isfinite(r1) || !isfinite(r2));
}

// ---- d in (64, 256]: the same algorithm over the whole grid (one cooperative launch); the d x d
// fp64 matrices live in global memory (L2-resident: 6 x 512 KB at d = 256), read with ld.global.cg
// (written by other CTAs between grid barriers); products in 32 x 32 output tiles, one per CTA
// in turn, each entry summed over k in order; norms as fixed-order sums of the CTAs' partials.
namespace cgw {
namespace cg = cooperative_groups;
constexpr int kT = 32;

__device__ double grid_sum(double v, double *red, double *gpart, cg::grid_group &grid) {
    const double b = block_sum_any(v, red);
    if (threadIdx.x == 0) gpart[blockIdx.x] = b;
    grid.sync();
    double t = 0.0;
    for (unsigned k = 0; k < gridDim.x; ++k) t += __ldcg(gpart + k);
    grid.sync();   // (gpart is reused by the next sum)
    return t;
}

// C = A B (d x d); C must not alias A or B
__device__ void mm(const double *A, const double *B, double *C, int d, cg::grid_group &grid) {
    __shared__ double sa[kT][kT + 1], sb[kT][kT + 1];
    const int nt = (d + kT - 1) / kT;
    const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
    for (int t = blockIdx.x; t < nt * nt; t += gridDim.x) {
        const int i0 = (t / nt) * kT, j0 = (t % nt) * kT;
        double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
        for (int k0 = 0; k0 < d; k0 += kT) {
            __syncthreads();
            for (int e = threadIdx.x; e < kT * kT; e += blockDim.x) {
                const int r = e / kT, c = e % kT;
                sa[r][c] = (i0 + r < d && k0 + c < d) ? __ldcg(A + (long long)(i0 + r) * d + k0 + c) : 0.0;
                sb[r][c] = (k0 + r < d && j0 + c < d) ? __ldcg(B + (long long)(k0 + r) * d + j0 + c) : 0.0;
            }
            __syncthreads();
#pragma unroll 8
            for (int kk = 0; kk < kT; ++kk) {
                const double a0 = sa[ty][kk], a1 = sa[ty + 16][kk], b0 = sb[kk][tx], b1 = sb[kk][tx + 16];
                acc[0][0] = fma(a0, b0, acc[0][0]);
                acc[0][1] = fma(a0, b1, acc[0][1]);
                acc[1][0] = fma(a1, b0, acc[1][0]);
                acc[1][1] = fma(a1, b1, acc[1][1]);
            }
        }
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int r = i0 + ty + 16 * i, c = j0 + tx + 16 * j;
                if (r < d && c < d) C[(long long)r * d + c] = acc[i][j];
            }
    }
    grid.sync();
}

__device__ void copy(const double *S, double *D, int d, cg::grid_group &grid) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)d * d;
         e += (long long)gridDim.x * blockDim.x)
        D[e] = __ldcg(S + e);
    grid.sync();
}

__device__ void symmetrize(double *A, int d, cg::grid_group &grid) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)d * d;
         e += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(e / d), j = (int)(e % d);
        if (i < j) {
            const double v = 0.5 * (__ldcg(A + (long long)i * d + j) + __ldcg(A + (long long)j * d + i));
            A[(long long)i * d + j] = v;
            A[(long long)j * d + i] = v;
        }
    }
    grid.sync();
}

// coupled Newton-Schulz as ns_sqrt above (same iteration, stop rule and budget)
__device__ double ns_sqrt(const double *M, double *Y, double *Z, double *T, double *U, int d, double *red,
                          double *gpart, cg::grid_group &grid) {
    const long long dd = (long long)d * d, g0 = blockIdx.x * (long long)blockDim.x + threadIdx.x,
                    gs = (long long)gridDim.x * blockDim.x;
    double fr = 0.0;
    for (long long e = g0; e < dd; e += gs) { const double v = __ldcg(M + e); fr += v * v; }
    const double nrm = sqrt(grid_sum(fr, red, gpart, grid));
    for (long long e = g0; e < dd; e += gs) {
        Y[e] = __ldcg(M + e) / nrm;
        Z[e] = (e / d == e % d) ? 1.0 : 0.0;
    }
    grid.sync();
    double res = INFINITY, prev = INFINITY;
    for (int it = 0; it < 100; ++it) {
        mm(Z, Y, T, d, grid);  // T = Z Y
        double r = 0.0;
        for (long long e = g0; e < dd; e += gs) {
            const double t = __ldcg(T + e);
            const double v = t - ((e / d == e % d) ? 1.0 : 0.0);
            r += v * v;
            T[e] = ((e / d == e % d) ? 1.5 : 0.0) - 0.5 * t;
        }
        res = sqrt(grid_sum(r, red, gpart, grid));   // (its barriers publish T)
        if (res < 1e-13 * d || (res < 1e-7 && res > 0.5 * prev)) break;
        prev = res;
        mm(Y, T, U, d, grid);  // U = Y T
        copy(U, Y, d, grid);
        mm(T, Z, U, d, grid);  // U = T Z
        copy(U, Z, d, grid);
    }
    const double sq = sqrt(nrm);
    for (long long e = g0; e < dd; e += gs) {
        Y[e] = __ldcg(Y + e) * sq;
        Z[e] = __ldcg(Z + e) / sq;
    }
    grid.sync();
    return res;
}
}  // namespace cgw

// work: 4 d^2 + gridDim.x doubles
__global__ void __launch_bounds__(kGT) k_gauss_A_wide(double *cov_mu, double *cov_nu, int d, float ridge_rel,
                                                       double *Aout, int *ns_fail, double *work) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ double red[kGT / 32];
    const long long dd = (long long)d * d, g0 = blockIdx.x * (long long)blockDim.x + threadIdx.x,
                    gs = (long long)gridDim.x * blockDim.x;
    double *Smu = cov_mu, *Snu = cov_nu, *R = work, *Ri = work + dd, *T = work + 2 * dd, *U = work + 3 * dd,
           *gpart = work + 4 * dd;
    double tr_mu = 0.0, tr_nu = 0.0;
    for (int k = 0; k < d; ++k) { tr_mu += cov_mu[(long long)k * d + k]; tr_nu += cov_nu[(long long)k * d + k]; }
    grid.sync();   // (every thread has read the diagonals before they change)
    for (long long e = g0; e < dd; e += gs)
        if (e / d == e % d) {
            Smu[e] += ridge_rel * tr_mu / d;
            Snu[e] += ridge_rel * tr_nu / d;
        }
    grid.sync();
    cgw::symmetrize(Smu, d, grid);
    cgw::symmetrize(Snu, d, grid);
    const double r1 = cgw::ns_sqrt(Smu, R, Ri, T, U, d, red, gpart, grid);   // R = S_mu^{1/2}, Ri = S_mu^{-1/2}
    cgw::mm(R, Snu, T, d, grid);                                               // T = R S_nu
    double *Mm = Smu;
    cgw::mm(T, R, Mm, d, grid);                                                // Mm = R S_nu R
    cgw::symmetrize(Mm, d, grid);
    double *Q = Snu, *Qi = R;
    const double r2 = cgw::ns_sqrt(Mm, Q, Qi, T, U, d, red, gpart, grid);    // Q = Mm^{1/2}
    cgw::mm(Ri, Q, T, d, grid);
    cgw::mm(T, Ri, U, d, grid);                                                // A = Ri Q Ri
    cgw::symmetrize(U, d, grid);
    for (long long e = g0; e < dd; e += gs) Aout[e] = __ldcg(U + e);
    if (blockIdx.x == 0 && threadIdx.x == 0) *ns_fail = (r1 > 1e-6 || r2 > 1e-6 || !isfinite(r1) || !isfinite(r2));
}

size_t gauss_wide_work_doubles(int d) { return 4 * (size_t)d * d + 256; }

cudaError_t launch_gauss_A(const double *mean_mu, double *cov_mu, const double *mean_nu,
                           double *cov_nu, int d, float ridge_rel, double *A, int *ns_fail,
                           cudaStream_t st, double *work) {
    (void)mean_mu; (void)mean_nu;
    if (d > 64) {
        if (!work || d > 256) return cudaErrorInvalidValue;
        const int nt = (d + cgw::kT - 1) / cgw::kT;
        int dev = 0, nsm = 148, occ = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_gauss_A_wide, kGT, 0);
        if (e != cudaSuccess) return e;
        const int G = std::max(1, std::min({nt * nt, nsm * std::max(occ, 1), 256}));
        void *args[] = {&cov_mu, &cov_nu, &d, &ridge_rel, &A, &ns_fail, &work};
        return cudaLaunchCooperativeKernel((const void *)k_gauss_A_wide, dim3(G), dim3(kGT), args, 0, st);
    }
    const size_t smem = 6 * (size_t)d * d * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(k_gauss_A, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_gauss_A<<<1, kGT, smem, st>>>(cov_mu, cov_nu, d, ridge_rel, A, ns_fail);
    return cudaGetLastError();
}

// f*(x_i) in fp64 (d <= 64; A, means cached in shared memory), tiles of 64 points: the tile's
// centred coordinates staged by coalesced loads; thread (kq, p) forms rows k in [16 kq, 16 kq + 16)
// of A c_p (c_p 8 at a time in registers, A read as broadcast double2) and its part of
// c_p^T A c_p; the 4 parts summed in kq order.
constexpr int kPotTile = 64;

size_t gauss_pot_smem(int d) {
    const int dp = (d + 1) & ~1;
    return sizeof(double) * ((size_t)d * dp + 2 * d + (size_t)kPotTile * (d + 1) + 4 * kPotTile) +
           sizeof(float) * (size_t)kPotTile * d;
}

__global__ void __launch_bounds__(kGT) k_gauss_pot(const float *__restrict__ x, long long n, int d,
                                                    const double *__restrict__ mmu,
                                                    const double *__restrict__ mnu,
                                                    const double *__restrict__ A, float *pot) {
    extern __shared__ double s[];
    const int dp = (d + 1) & ~1, d1 = d + 1;
    double *sA = s;                       // [d][dp]
    double *smu = sA + d * dp, *snu = smu + d;
    double *cs = snu + d;                 // [64][d + 1] centred coordinates
    double *red = cs + kPotTile * d1;     // [4][64]
    float *xr = reinterpret_cast<float *>(red + 4 * kPotTile);   // [64][d] raw coordinates
    for (int e = threadIdx.x; e < d * dp; e += blockDim.x) {
        const int k = e / dp, l = e % dp;
        sA[e] = l < d ? A[k * d + l] : 0.0;
    }
    for (int k = threadIdx.x; k < d; k += blockDim.x) { smu[k] = mmu[k]; snu[k] = mnu[k]; }
    const int p = threadIdx.x & (kPotTile - 1), kq = threadIdx.x >> 6;
    const long long tiles = (n + kPotTile - 1) / kPotTile;
    for (long long tb = blockIdx.x; tb < tiles; tb += gridDim.x) {
        const long long i0 = tb * kPotTile;
        const int cnt = (int)min((long long)kPotTile, n - i0);
        __syncthreads();   // (the previous tile's readers are done; sA / means visible)
        for (int e = threadIdx.x; e < kPotTile * d; e += blockDim.x) {
            const int r = e / d, k = e % d;
            const float v = r < cnt ? x[(i0 + r) * d + k] : 0.f;
            xr[e] = v;
            cs[r * d1 + k] = (double)v - smu[k];
        }
        __syncthreads();
        const double *cp = cs + p * d1;
        double row[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) row[u] = 0.0;
        for (int l0 = 0; l0 < d; l0 += 8) {
            double c[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) c[u] = l0 + u < d ? cp[l0 + u] : 0.0;
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const int k = 16 * kq + u;
                if (k >= d) break;
                const double2 *ar = reinterpret_cast<const double2 *>(sA + k * dp + l0);
                double r = row[u];
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    if (l0 + 2 * v >= dp) break;
                    const double2 a2 = ar[v];
                    r = fma(a2.x, c[2 * v], r);
                    r = fma(a2.y, c[2 * v + 1], r);
                }
                row[u] = r;
            }
        }
        double q = 0.0;
#pragma unroll
        for (int u = 0; u < 16; ++u)
            if (16 * kq + u < d) q = fma(cp[16 * kq + u], row[u], q);
        red[kq * kPotTile + p] = q;
        __syncthreads();
        if (kq == 0 && p < cnt) {
            const double quad = ((red[p] + red[kPotTile + p]) + red[2 * kPotTile + p]) + red[3 * kPotTile + p];
            double nx = 0.0, lin = 0.0;
            for (int k = 0; k < d; ++k) {
                const double xk = xr[p * d + k];
                nx += xk * xk;
                lin += snu[k] * xk;
            }
            pot[i0 + p] = (float)(nx - quad - 2.0 * lin);
        }
    }
}

// d in (64, 256]: A (d x d fp64, 512 KB at d = 256) stays in global memory / L2; the tile's centred
// coordinates in shared memory ([64][d + 1]); thread (kq, p) forms the rows k = kq, kq + 4, .. of
// A c_p (a warp shares kq: A rows are broadcast loads) and its part of c_p^T A c_p; the 4 parts
// summed in kq order.
__global__ void __launch_bounds__(kGT) k_gauss_pot_wide(const float *__restrict__ x, long long n, int d,
                                                         const double *__restrict__ mmu,
                                                         const double *__restrict__ mnu,
                                                         const double *__restrict__ A, float *pot) {
    extern __shared__ double s[];
    const int d1 = d + 1;
    double *cs = s;                       // [64][d + 1]
    double *red = cs + kPotTile * d1;     // [4][64]
    const int p = threadIdx.x & (kPotTile - 1), kq = threadIdx.x >> 6;
    const long long tiles = (n + kPotTile - 1) / kPotTile;
    for (long long tb = blockIdx.x; tb < tiles; tb += gridDim.x) {
        const long long i0 = tb * kPotTile;
        const int cnt = (int)min((long long)kPotTile, n - i0);
        __syncthreads();
        for (int e = threadIdx.x; e < kPotTile * d; e += blockDim.x) {
            const int r = e / d, k = e % d;
            cs[r * d1 + k] = r < cnt ? (double)x[(i0 + r) * d + k] - mmu[k] : 0.0;
        }
        __syncthreads();
        const double *cp = cs + p * d1;
        double q = 0.0;
        for (int k = kq; k < d; k += 4) {
            const double *ar = A + (long long)k * d;
            double r0 = 0.0, r1 = 0.0;
            int l = 0;
            for (; l + 1 < d; l += 2) {
                r0 = fma(__ldg(ar + l), cp[l], r0);
                r1 = fma(__ldg(ar + l + 1), cp[l + 1], r1);
            }
            if (l < d) r0 = fma(__ldg(ar + l), cp[l], r0);
            q = fma(cp[k], r0 + r1, q);
        }
        red[kq * kPotTile + p] = q;
        __syncthreads();
        if (kq == 0 && p < cnt) {
            const double quad = ((red[p] + red[kPotTile + p]) + red[2 * kPotTile + p]) + red[3 * kPotTile + p];
            double nx = 0.0, lin = 0.0;
            for (int k = 0; k < d; ++k) {
                const double xk = x[(i0 + p) * d + k];
                nx += xk * xk;
                lin += mnu[k] * xk;
            }
            pot[i0 + p] = (float)(nx - quad - 2.0 * lin);
        }
    }
}

cudaError_t launch_gauss_potential(const float *x, long long n, int d, const double *m_mu,
                                   const double *m_nu, const double *A, float *pot, cudaStream_t st) {
    if (d > 64) {
        const size_t smem = sizeof(double) * ((size_t)kPotTile * (d + 1) + 4 * kPotTile);
        cudaError_t e = cudaFuncSetAttribute(k_gauss_pot_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        const long long tiles = (n + kPotTile - 1) / kPotTile;
        k_gauss_pot_wide<<<(int)(tiles > 148 ? 148 : tiles), kGT, smem, st>>>(x, n, d, m_mu, m_nu, A, pot);
        return cudaGetLastError();
    }
    const size_t smem = gauss_pot_smem(d);
    cudaError_t e = cudaFuncSetAttribute(k_gauss_pot, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const long long tiles = (n + kPotTile - 1) / kPotTile;
    k_gauss_pot<<<(int)(tiles > 148 * 2 ? 148 * 2 : tiles), kGT, smem, st>>>(x, n, d, m_mu, m_nu, A, pot);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ GMM
// work layout (doubles): R [Kx][d*d] (S_k^{1/2}), Linv [Kx][d*d], logdet [Kx], C [Kx*Ky], ft [Kx]
constexpr int kGmmWideSlots = 32;   // d > 64: CTAs (each with 5 d x d scratch matrices) of the NS kernels

size_t gmm_work_doubles(int d, int Kx, int Ky) {
    const size_t base = (size_t)2 * Kx * d * d + Kx + (size_t)Kx * Ky + Kx;
    return d > 64 ? base + (size_t)kGmmWideSlots * 5 * d * d : base;
}

__global__ void __launch_bounds__(kGT) k_gmm_sqrt(const float *covx, int d, double *R, int *flags) {
    extern __shared__ double sm[];
    __shared__ double red[kGT / 32];
    const int dd = d * d, k = blockIdx.x;
    double *M = sm, *Y = sm + dd, *Z = sm + 2 * dd, *T = sm + 3 * dd, *U = sm + 4 * dd;
    for (int e = threadIdx.x; e < dd; e += blockDim.x) M[e] = covx[(long long)k * dd + e];
    __syncthreads();
    symmetrize(M, d);
    const double r = ns_sqrt(M, Y, Z, T, U, d, red);
    for (int e = threadIdx.x; e < dd; e += blockDim.x) R[(long long)k * dd + e] = Y[e];
    if (threadIdx.x == 0 && (r > 1e-6 || !isfinite(r))) atomicOr(flags, 1);
}

__global__ void __launch_bounds__(kGT) k_gmm_bures(const float *mux, const float *covx, int Kx,
                                                    const float *muy, const float *covy, int Ky, int d,
                                                    const double *R, double *C, int *flags) {
    extern __shared__ double sm[];
    __shared__ double red[kGT / 32];
    const int dd = d * d, k = blockIdx.x / Ky, l = blockIdx.x % Ky;
    double *Sy = sm, *Rk = sm + dd, *M = sm + 2 * dd, *T = sm + 3 * dd, *U = sm + 4 * dd;
    for (int e = threadIdx.x; e < dd; e += blockDim.x) {
        Sy[e] = covy[(long long)l * dd + e];
        Rk[e] = R[(long long)k * dd + e];
    }
    __syncthreads();
    symmetrize(Sy, d);
    mm(Rk, Sy, T, d);
    mm(T, Rk, M, d);
    symmetrize(M, d);
    double *Y = Sy, *Z = Rk;  // free after M is formed
    const double r = ns_sqrt(M, Y, Z, T, U, d, red);
    if (threadIdx.x == 0) {
        double tr = 0.0, dm = 0.0;
        for (int i = 0; i < d; ++i) {
            tr += (double)covx[(long long)k * dd + i * d + i] + (double)covy[(long long)l * dd + i * d + i]
                  - 2.0 * Y[i * d + i];
            const double t = (double)mux[k * d + i] - (double)muy[l * d + i];
            dm += t * t;
        }
        C[k * Ky + l] = dm + tr;
        if (r > 1e-6 || !isfinite(r)) atomicOr(flags, 1);
    }
}

// K x K entropic OT (Alg. 1, g-then-f; R-13), one warp, in log2 units: F = f kappa,
// G = g kappa, Kc = -C kappa (kappa = log2(e)/eps, fp64).
// The K x K solve with Anderson acceleration (memory 5, reading R-29: the inner problem of the
// GMM initializer converges in thousands of plain sweeps at C3's eps; the paper only asks for
// its solution).  fp64 throughout (the mixing is sensitive to rounding near the solution).  Sweep
// l: G = g_sk(F), T = f_sk(G); err_l = sum_k a_k |expm1(ln2 (F_k - T_k))| (the row term of
// (f^l, g~), whose columns are exact); stop if err_l < tol (-> f~ = f^l) or at max_iter; else
// the ring slot gets (T, T - F) and F = sum_u alpha_u T_u with alpha from the regularised Gram
// system (lam = 1e-8 tr G / count) as in K13/K19.  Lane t owns outputs t and t + 32.
__device__ __forceinline__ void gmm_update_d(const double *__restrict__ Kc, int Kx, int Ky, bool cols,
                                             const double *in, double *out, const double *lw) {
    const int t = threadIdx.x;
    const int Kout = cols ? Ky : Kx, Kin = cols ? Kx : Ky;
    const int rs = cols ? Ky : 1, ks = cols ? 1 : Ky;
    double on[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int k = t + 32 * h;
        on[h] = 0.0;
        if (k >= Kout) continue;
        const double *kc = Kc + k * ks;
        double mx = -INFINITY;
        for (int r = 0; r < Kin; ++r) mx = fmax(mx, in[r] + kc[r * rs]);
        double sm = 0.0;
        for (int r = 0; r < Kin; ++r) sm += exp2(in[r] + kc[r * rs] - mx);
        on[h] = lw[k] - (mx + log2(sm));
    }
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h)
        if (t + 32 * h < Kout) out[t + 32 * h] = on[h];
    __syncwarp();
}

constexpr int kGmmAnd = 5;

__global__ void __launch_bounds__(32) k_gmm_sinkhorn_and(const double *C, int Kx, int Ky, const float *wx,
                                                          const float *wy, float eps_f, float tol, int max_iter,
                                                          double *ft, int *flags) {
    __shared__ double Kc[64 * 64], F[64], G[64], T[64], la[64], lb[64];
    __shared__ double Fh[kGmmAnd][64], Rh[kGmmAnd][64], Gm[kGmmAnd * kGmmAnd];
    const double eps = eps_f, kap = kLog2ed / eps;
    const int t = threadIdx.x;
    for (int e = t; e < Kx * Ky; e += 32) Kc[e] = -C[e] * kap;
    for (int i = t; i < 64; i += 32) {
        F[i] = 0.0;
        G[i] = 0.0;
        la[i] = i < Kx ? log2((double)wx[i]) : 0.0;
        lb[i] = i < Ky ? log2((double)wy[i]) : 0.0;
    }
    __syncwarp();
    int head = 0, cnt = 0;
    for (int l = 0;; ++l) {
        gmm_update_d(Kc, Kx, Ky, true, F, G, lb);
        gmm_update_d(Kc, Kx, Ky, false, G, T, la);
        double e = 0.0;
        for (int k = t; k < Kx; k += 32) e += (double)wx[k] * fabs(expm1(kLn2d * (F[k] - T[k])));
        for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
        if (!isfinite(e)) { if (t == 0) atomicOr(flags, 2); break; }
        if ((float)e < tol || l + 1 >= max_iter) break;
        const int cn = cnt < kGmmAnd ? cnt + 1 : kGmmAnd;
        double dv[kGmmAnd];
#pragma unroll
        for (int u = 0; u < kGmmAnd; ++u) dv[u] = 0.0;
        for (int k = t; k < Kx; k += 32) {
            const double r = T[k] - F[k];
#pragma unroll
            for (int u = 0; u < kGmmAnd; ++u)
                if (u < cn) dv[u] += r * (u == head ? r : Rh[u][k]);
            Fh[head][k] = T[k];
            Rh[head][k] = r;
        }
        double dl = 0.0;   // lane u: <r_new, r_u>
#pragma unroll
        for (int u = 0; u < kGmmAnd; ++u) {
            double v = dv[u];
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (t == u) dl = v;
        }
        __syncwarp();
        double row[kGmmAnd];
#pragma unroll
        for (int u = 0; u < kGmmAnd; ++u) {
            const double du = __shfl_sync(0xffffffffu, dl, u);
            double gv;
            if (t == head) gv = du;
            else if (u == head) gv = dl;
            else gv = t < kGmmAnd ? Gm[t * kGmmAnd + u] : 0.0;
            row[u] = (t < cn && u < cn) ? gv : (u == t ? 1.0 : 0.0);
        }
        __syncwarp();
        if (t < cn) { Gm[head * kGmmAnd + t] = dl; Gm[t * kGmmAnd + head] = dl; }
        double diag = 0.0;
#pragma unroll
        for (int u = 0; u < kGmmAnd; ++u)
            if (u == t) diag = row[u];
        double tr = t < cn ? diag : 0.0;
        for (int o = 16; o > 0; o >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, o);
        const double lam = tr > 0.0 ? 1e-8 * tr / cn : 1.0;
#pragma unroll
        for (int u = 0; u < kGmmAnd; ++u)
            if (u == t && t < cn) row[u] += lam;
        double rhs = t < cn ? 1.0 : 0.0;
        for (int c = 0; c < cn; ++c) {
            double piv[kGmmAnd], myc = 0.0;
#pragma unroll
            for (int u = 0; u < kGmmAnd; ++u) {
                piv[u] = __shfl_sync(0xffffffffu, row[u], c);
                if (u == c) myc = row[u];
            }
            const double prhs = __shfl_sync(0xffffffffu, rhs, c);
            const double pcc = __shfl_sync(0xffffffffu, myc, c);
            if (t != c) {
                const double q = myc / pcc;
#pragma unroll
                for (int u = 0; u < kGmmAnd; ++u) row[u] = fma(-q, piv[u], row[u]);
                rhs = fma(-q, prhs, rhs);
            }
        }
#pragma unroll
        for (int u = 0; u < kGmmAnd; ++u)
            if (u == t) diag = row[u];
        const double xl = t < cn ? rhs / diag : 0.0;
        double sx = xl;
        for (int o = 16; o > 0; o >>= 1) sx += __shfl_xor_sync(0xffffffffu, sx, o);
        double al[kGmmAnd];
#pragma unroll
        for (int u = 0; u < kGmmAnd; ++u) al[u] = __shfl_sync(0xffffffffu, xl / sx, u);
        __syncwarp();
        for (int k = t; k < Kx; k += 32) {
            double v = 0.0;
#pragma unroll
            for (int u = 0; u < kGmmAnd; ++u)
                if (u < cn) v = fma(al[u], Fh[u][k], v);
            F[k] = v;
        }
        head = (head + 1) % kGmmAnd;
        cnt = cn;
        __syncwarp();
    }
    // f~ is defined up to a constant and the mixing moves it along that line: return the
    // representative with sum_k a_k f~_k = 0 (R-29)
    double ma = 0.0, sa = 0.0;
    for (int k = t; k < Kx; k += 32) { ma += (double)wx[k] * F[k]; sa += (double)wx[k]; }
    for (int o = 16; o > 0; o >>= 1) {
        ma += __shfl_xor_sync(0xffffffffu, ma, o);
        sa += __shfl_xor_sync(0xffffffffu, sa, o);
    }
    for (int i = t; i < Kx; i += 32) ft[i] = (F[i] - ma / sa) / kap;
}

// Cholesky S_k = L L^T (fp64, one CTA, sequential columns), then Linv and log det L.
__global__ void __launch_bounds__(kGT) k_gmm_chol(const float *covx, int d, double *Linv, double *logdet,
                                                   int *flags) {
    extern __shared__ double sm[];
    const int dd = d * d, k = blockIdx.x;
    double *L = sm, *Li = sm + dd;
    for (int e = threadIdx.x; e < dd; e += blockDim.x) {
        const int i = e / d, j = e % d;
        L[e] = 0.5 * ((double)covx[(long long)k * dd + i * d + j] + (double)covx[(long long)k * dd + j * d + i]);
        Li[e] = 0.0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // textbook Cholesky-Banachiewicz, d <= 64
        int bad = 0;
        for (int j = 0; j < d; ++j) {
            double s = L[j * d + j];
            for (int t = 0; t < j; ++t) s -= L[j * d + t] * L[j * d + t];
            if (!(s > 0.0)) { bad = 1; s = 1e-300; }
            const double ljj = sqrt(s);
            L[j * d + j] = ljj;
            for (int i = j + 1; i < d; ++i) {
                double v = L[i * d + j];
                for (int t = 0; t < j; ++t) v -= L[i * d + t] * L[j * d + t];
                L[i * d + j] = v / ljj;
            }
            for (int t = j + 1; t < d; ++t) L[j * d + t] = 0.0;
        }
        double ld = 0.0;
        for (int j = 0; j < d; ++j) ld += log(L[j * d + j]);
        logdet[k] = ld;
        if (bad) atomicOr(flags, 4);
    }
    __syncthreads();
    // Linv: solve L * Li = I column by column (thread per column)
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
        for (int i = 0; i < d; ++i) {
            double v = (i == c) ? 1.0 : 0.0;
            for (int t = 0; t < i; ++t) v -= L[i * d + t] * Li[t * d + c];
            Li[i * d + c] = v / L[i * d + i];
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < dd; e += blockDim.x) Linv[(long long)k * dd + e] = Li[e];
}

// f^(0)(x_i) = sum_k f~_k p_k(x_i), log p_k = log a_k - 1/2 |Linv_k (x - m_k)|^2 - logdet_k - LSE.
__global__ void __launch_bounds__(kGT) k_gmm_pot(const float *__restrict__ x, long long n, int d, int K,
                                                  const float *__restrict__ wx, const float *__restrict__ mux,
                                                  const double *__restrict__ Linv,
                                                  const double *__restrict__ logdet,
                                                  const double *__restrict__ ft, float *pot) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const float *xi = x + i * d;
        double mx = -INFINITY, num = 0.0, den = 0.0;
        for (int k = 0; k < K; ++k) {
            const double *Li = Linv + (long long)k * d * d;
            const float *mk = mux + (long long)k * d;
            double q = 0.0;
            for (int r = 0; r < d; ++r) {
                double z = 0.0;
                for (int c = 0; c <= r; ++c) z += Li[r * d + c] * ((double)xi[c] - (double)mk[c]);
                q += z * z;
            }
            const double lp = log((double)wx[k]) - 0.5 * q - logdet[k];
            // streaming softmax-weighted mean of f~ (fixed k order)
            if (lp > mx) {
                const double sc = exp(mx - lp);
                num *= sc;
                den *= sc;
                mx = lp;
            }
            const double e = exp(lp - mx);
            num += e * ft[k];
            den += e;
        }
        pot[i] = (float)(num / den);
    }
}

// ---- d in (64, 256]: the same per-component / per-pair steps with each CTA's d x d matrices in
// global memory (its slot of 5 d^2 doubles, L2-resident) instead of shared memory: block-level
// products in 32 x 32 tiles (each entry summed over k in order), the same coupled Newton-Schulz
// iteration and stop rule as ns_sqrt, the Cholesky factorisation with the rows below the pivot
// updated in parallel.  Scratch written and read by the same CTA between __syncthreads.
namespace gwide {
constexpr int kT = 32;

__device__ void mm(const double *A, const double *B, double *C, int d) {
    __shared__ double sa[kT][kT + 1], sb[kT][kT + 1];
    const int nt = (d + kT - 1) / kT;
    const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
    for (int t = 0; t < nt * nt; ++t) {
        const int i0 = (t / nt) * kT, j0 = (t % nt) * kT;
        double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
        for (int k0 = 0; k0 < d; k0 += kT) {
            __syncthreads();
            for (int e = threadIdx.x; e < kT * kT; e += blockDim.x) {
                const int r = e / kT, c = e % kT;
                sa[r][c] = (i0 + r < d && k0 + c < d) ? __ldcg(A + (long long)(i0 + r) * d + k0 + c) : 0.0;
                sb[r][c] = (k0 + r < d && j0 + c < d) ? __ldcg(B + (long long)(k0 + r) * d + j0 + c) : 0.0;
            }
            __syncthreads();
#pragma unroll 8
            for (int kk = 0; kk < kT; ++kk) {
                const double a0 = sa[ty][kk], a1 = sa[ty + 16][kk], b0 = sb[kk][tx], b1 = sb[kk][tx + 16];
                acc[0][0] = fma(a0, b0, acc[0][0]);
                acc[0][1] = fma(a0, b1, acc[0][1]);
                acc[1][0] = fma(a1, b0, acc[1][0]);
                acc[1][1] = fma(a1, b1, acc[1][1]);
            }
        }
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int r = i0 + ty + 16 * i, c = j0 + tx + 16 * j;
                if (r < d && c < d) C[(long long)r * d + c] = acc[i][j];
            }
    }
    __syncthreads();
}

__device__ void symmetrize(double *A, int d) {
    for (int e = threadIdx.x; e < d * d; e += blockDim.x) {
        const int i = e / d, j = e % d;
        if (i < j) {
            const double v = 0.5 * (__ldcg(A + i * d + j) + __ldcg(A + j * d + i));
            A[i * d + j] = v;
            A[j * d + i] = v;
        }
    }
    __syncthreads();
}

__device__ double ns_sqrt(const double *M, double *Y, double *Z, double *T, double *U, int d, double *red) {
    const int dd = d * d;
    double fr = 0.0;
    for (int e = threadIdx.x; e < dd; e += blockDim.x) { const double v = __ldcg(M + e); fr += v * v; }
    const double nrm = sqrt(block_sum_any(fr, red));
    for (int e = threadIdx.x; e < dd; e += blockDim.x) {
        Y[e] = __ldcg(M + e) / nrm;
        Z[e] = (e / d == e % d) ? 1.0 : 0.0;
    }
    __syncthreads();
    double res = INFINITY, prev = INFINITY;
    for (int it = 0; it < 100; ++it) {
        mm(Z, Y, T, d);
        double r = 0.0;
        for (int e = threadIdx.x; e < dd; e += blockDim.x) {
            const double t = __ldcg(T + e);
            const double v = t - ((e / d == e % d) ? 1.0 : 0.0);
            r += v * v;
            T[e] = ((e / d == e % d) ? 1.5 : 0.0) - 0.5 * t;
        }
        res = sqrt(block_sum_any(r, red));
        if (res < 1e-13 * d || (res < 1e-7 && res > 0.5 * prev)) break;
        prev = res;
        mm(Y, T, U, d);
        for (int e = threadIdx.x; e < dd; e += blockDim.x) Y[e] = __ldcg(U + e);
        __syncthreads();
        mm(T, Z, U, d);
        for (int e = threadIdx.x; e < dd; e += blockDim.x) Z[e] = __ldcg(U + e);
        __syncthreads();
    }
    const double sq = sqrt(nrm);
    for (int e = threadIdx.x; e < dd; e += blockDim.x) {
        Y[e] = __ldcg(Y + e) * sq;
        Z[e] = __ldcg(Z + e) / sq;
    }
    __syncthreads();
    return res;
}
}  // namespace gwide

// R_k = S_k^{1/2} for every x component (CTA slot b takes components b, b + G, ..)
__global__ void __launch_bounds__(kGT) k_gmm_sqrt_wide(const float *covx, int d, int Kx, double *R, double *slots,
                                                        int *flags) {
    __shared__ double red[kGT / 32];
    const long long dd = (long long)d * d;
    double *M = slots + blockIdx.x * 5 * dd, *Y = M + dd, *Z = M + 2 * dd, *T = M + 3 * dd, *U = M + 4 * dd;
    for (int k = blockIdx.x; k < Kx; k += gridDim.x) {
        for (int e = threadIdx.x; e < dd; e += blockDim.x) M[e] = covx[k * dd + e];
        __syncthreads();
        gwide::symmetrize(M, d);
        const double r = gwide::ns_sqrt(M, Y, Z, T, U, d, red);
        for (int e = threadIdx.x; e < dd; e += blockDim.x) R[k * dd + e] = __ldcg(Y + e);
        if (threadIdx.x == 0 && (r > 1e-6 || !isfinite(r))) atomicOr(flags, 1);
        __syncthreads();
    }
}

// C_kl = |m_k - m'_l|^2 + tr(S_k + S'_l - 2 (R_k S'_l R_k)^{1/2}) for every pair (Eq. 6)
__global__ void __launch_bounds__(kGT) k_gmm_bures_wide(const float *mux, const float *covx, int Kx,
                                                         const float *muy, const float *covy, int Ky, int d,
                                                         const double *R, double *C, double *slots, int *flags) {
    __shared__ double red[kGT / 32];
    const long long dd = (long long)d * d;
    double *Sy = slots + blockIdx.x * 5 * dd, *Rk = Sy + dd, *M = Sy + 2 * dd, *T = Sy + 3 * dd, *U = Sy + 4 * dd;
    for (int pr = blockIdx.x; pr < Kx * Ky; pr += gridDim.x) {
        const int k = pr / Ky, l = pr % Ky;
        for (int e = threadIdx.x; e < dd; e += blockDim.x) {
            Sy[e] = covy[l * dd + e];
            Rk[e] = __ldcg(R + k * dd + e);
        }
        __syncthreads();
        gwide::symmetrize(Sy, d);
        gwide::mm(Rk, Sy, T, d);
        gwide::mm(T, Rk, M, d);
        gwide::symmetrize(M, d);
        double *Y = Sy, *Z = Rk;
        const double r = gwide::ns_sqrt(M, Y, Z, T, U, d, red);
        if (threadIdx.x == 0) {
            double tr = 0.0, dm = 0.0;
            for (int i = 0; i < d; ++i) {
                tr += (double)covx[k * dd + (long long)i * d + i] + (double)covy[l * dd + (long long)i * d + i]
                      - 2.0 * __ldcg(Y + (long long)i * d + i);
                const double t = (double)mux[k * d + i] - (double)muy[l * d + i];
                dm += t * t;
            }
            C[k * Ky + l] = dm + tr;
            if (r > 1e-6 || !isfinite(r)) atomicOr(flags, 1);
        }
        __syncthreads();
    }
}

// Cholesky-Banachiewicz per component (one CTA each, L in the slot): row j's pivot by thread 0,
// the rows below by the whole CTA; then L^{-1} a column per thread and log det L
__global__ void __launch_bounds__(kGT) k_gmm_chol_wide(const float *covx, int d, int Kx, double *Linv,
                                                        double *logdet, double *slots, int *flags) {
    __shared__ double s_ljj;
    const long long dd = (long long)d * d;
    double *L = slots + blockIdx.x * 5 * dd;
    for (int k = blockIdx.x; k < Kx; k += gridDim.x) {
        double *Li = Linv + k * dd;
        for (int e = threadIdx.x; e < dd; e += blockDim.x) {
            const int i = e / d, j = e % d;
            L[e] = 0.5 * ((double)covx[k * dd + (long long)i * d + j] + (double)covx[k * dd + (long long)j * d + i]);
        }
        __syncthreads();
        int bad = 0;
        for (int j = 0; j < d; ++j) {
            if (threadIdx.x == 0) {
                double s = __ldcg(L + (long long)j * d + j);
                for (int t = 0; t < j; ++t) { const double v = __ldcg(L + (long long)j * d + t); s -= v * v; }
                if (!(s > 0.0)) { bad = 1; s = 1e-300; }
                s_ljj = sqrt(s);
                L[(long long)j * d + j] = s_ljj;
            }
            __syncthreads();
            const double ljj = s_ljj;
            for (int i = j + 1 + threadIdx.x; i < d; i += blockDim.x) {
                double v = __ldcg(L + (long long)i * d + j);
                for (int t = 0; t < j; ++t) v -= __ldcg(L + (long long)i * d + t) * __ldcg(L + (long long)j * d + t);
                L[(long long)i * d + j] = v / ljj;
            }
            __syncthreads();
        }
        for (int e = threadIdx.x; e < dd; e += blockDim.x)
            if (e % d > e / d) L[e] = 0.0;
        __syncthreads();
        if (threadIdx.x == 0) {
            double ld = 0.0;
            for (int j = 0; j < d; ++j) ld += log(__ldcg(L + (long long)j * d + j));
            logdet[k] = ld;
            if (bad) atomicOr(flags, 4);
        }
        for (int c = threadIdx.x; c < d; c += blockDim.x) {
            for (int i = 0; i < d; ++i) {
                double v = (i == c) ? 1.0 : 0.0;
                for (int t = 0; t < i; ++t) v -= __ldcg(L + (long long)i * d + t) * __ldcg(Li + (long long)t * d + c);
                Li[(long long)i * d + c] = v / __ldcg(L + (long long)i * d + i);
            }
        }
        __syncthreads();
    }
}

cudaError_t launch_gmm_init(const float *x, long long n, int d, int Kx, const float *wx,
                            const float *mux, const float *covx, int Ky, const float *wy,
                            const float *muy, const float *covy, float eps, float inner_tol,
                            int inner_max_iter, float *pot, double *work, int *flags,
                            cudaStream_t st) {
    if (d > 256 || Kx > 64 || Ky > 64) return cudaErrorInvalidValue;
    const int dd = d * d;
    double *R = work, *Linv = R + (size_t)Kx * dd, *logdet = Linv + (size_t)Kx * dd,
           *C = logdet + Kx, *ft = C + (size_t)Kx * Ky;
    cudaError_t e;
    if (d > 64) {
        double *slots = ft + Kx;
        const int gs = std::min(Kx, kGmmWideSlots), gp = std::min(Kx * Ky, kGmmWideSlots);
        k_gmm_sqrt_wide<<<gs, kGT, 0, st>>>(covx, d, Kx, R, slots, flags);
        k_gmm_bures_wide<<<gp, kGT, 0, st>>>(mux, covx, Kx, muy, covy, Ky, d, R, C, slots, flags);
        k_gmm_sinkhorn_and<<<1, 32, 0, st>>>(C, Kx, Ky, wx, wy, eps, inner_tol, inner_max_iter, ft, flags);
        k_gmm_chol_wide<<<gs, kGT, 0, st>>>(covx, d, Kx, Linv, logdet, slots, flags);
        long long b = (n + kGT - 1) / kGT;
        k_gmm_pot<<<(int)(b > 148 * 8 ? 148 * 8 : b), kGT, 0, st>>>(x, n, d, Kx, wx, mux, Linv, logdet, ft, pot);
        return cudaGetLastError();
    }
    size_t s5 = 5 * (size_t)dd * sizeof(double), s2 = 2 * (size_t)dd * sizeof(double);
    if ((e = cudaFuncSetAttribute(k_gmm_sqrt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s5))) return e;
    if ((e = cudaFuncSetAttribute(k_gmm_bures, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s5))) return e;
    if ((e = cudaFuncSetAttribute(k_gmm_chol, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s2))) return e;
    k_gmm_sqrt<<<Kx, kGT, s5, st>>>(covx, d, R, flags);
    k_gmm_bures<<<Kx * Ky, kGT, s5, st>>>(mux, covx, Kx, muy, covy, Ky, d, R, C, flags);
    k_gmm_sinkhorn_and<<<1, 32, 0, st>>>(C, Kx, Ky, wx, wy, eps, inner_tol, inner_max_iter, ft, flags);
    k_gmm_chol<<<Kx, kGT, s2, st>>>(covx, d, Linv, logdet, flags);
    long long b = (n + kGT - 1) / kGT;
    k_gmm_pot<<<(int)(b > 148 * 8 ? 148 * 8 : b), kGT, 0, st>>>(x, n, d, Kx, wx, mux, Linv, logdet, ft, pot);
    return cudaGetLastError();
}

}  // namespace sk
