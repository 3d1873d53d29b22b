// sk_sort1d.cu — K8 (segmented stable sort / rank) and K9 (the 1D eps = 0 dual).
//
// K8: one CTA per row; keys packed as (order-preserving uint32 of the float,
//     original index) in one uint64 and bitonic-sorted in shared memory — unique
//     keys, so the result equals a stable sort with ties broken by index (R-16;
//     -0.0 is normalised to +0.0, NaN raises a flag).  Bit-exact.  Rows longer than 8192
//     keys: the same network over a global key array (long-distance stages one launch
//     each, the rest on 8192-key segments in shared memory).
// K9: for n = m, uniform weights and c(x, y) = (x - y)^2, the sorted identity
//     matching is optimal.  DualSort (Alg. 2, read as
//     f_i <- min_j (c_ij - c_jj + f_j), R-5) is a Bellman-Ford relaxation on the
//     graph with edges j -> i of weight c_ij - c_jj (appendix).  On sorted
//     supports with this submodular cost the shortest walks move between adjacent
//     indices only, so its fixed point from f = 0 (R-7) is, with
//        F_0 = 0,      F_{k+1} = F_k + (c_{k+1,k} - c_{k,k}),
//        B_{n-1} = 0,  B_k     = B_{k+1} + (c_{k,k+1} - c_{k+1,k+1}),
//        f~_k = min(0, F_k - max_{j<=k} F_j, B_k - max_{j>=k} B_j),
//     i.e. four fp64 block scans (prefix sum, suffix sum, prefix max, suffix max).
//     The oracle runs Alg. 2 itself to its fixed point; parity checks the two agree.
//     (n > 4096: the four n-vectors live in workspace instead of shared memory.)
//     Paper mode (iters = L > 0): exactly L Jacobi sweeps of Alg. 2, O(L n^2).
//     Then f^(0)_{sigma(k)} = f~_k.
#include <algorithm>

#include "sk_internal.h"
#include "sk_common.cuh"

namespace sk {

constexpr int kST = 512;

__device__ __forceinline__ uint32_t orderable(float v) {
    if (v == 0.f) v = 0.f;  // -0.0 -> +0.0
    uint32_t u = __float_as_uint(v);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__global__ void __launch_bounds__(kST) k_sort_rows(const float *__restrict__ x, int n, long long stride,
                                                   int *perm, int *rank, float *sorted, int *nanflag) {
    extern __shared__ unsigned long long key[];
    const int row = blockIdx.x;
    const float *xr = x + row * stride;
    int N2 = 1;
    while (N2 < n) N2 <<= 1;
    int bad = 0;
    for (int i = threadIdx.x; i < N2; i += kST) {
        if (i < n) {
            const float v = xr[i];
            bad |= isnan(v);
            key[i] = ((unsigned long long)orderable(v) << 32) | (unsigned)i;
        } else {
            key[i] = ~0ull;
        }
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(nanflag, 1);
    __syncthreads();
    for (int k = 2; k <= N2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < N2; i += kST) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const unsigned long long A = key[i], B = key[ixj];
                    const bool up = (i & k) == 0;
                    if ((A > B) == up) { key[i] = B; key[ixj] = A; }
                }
            }
            __syncthreads();
        }
    }
    for (int k = threadIdx.x; k < n; k += kST) {
        const int idx = (int)(key[k] & 0xffffffffu);
        if (perm) perm[(long long)row * n + k] = idx;
        if (rank) rank[(long long)row * n + idx] = k;
        if (sorted) sorted[(long long)row * n + k] = xr[idx];
    }
}

// ---- rows longer than 8192 keys: the same bitonic network over a global key array per row
// (B x N2 keys), compare distances j >= kSeg by one launch per (k, j) stage over all rows, and
// the stages j < kSeg of every k on 8192-key segments in shared memory.  The direction of a
// comparison is that of the global key index (i & k), so the result is the whole-row bitonic
// sort: keys (orderable value, index) are distinct, hence a stable sort by value.
constexpr int kSeg = 8192;

__global__ void k_keys_init(const float *__restrict__ x, int B, int n, long long stride, int N2,
                            unsigned long long *keys, int *nanflag) {
    const long long tot = (long long)B * N2;
    int bad = 0;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
        const long long row = e / N2;
        const int i = (int)(e % N2);
        if (i < n) {
            const float v = x[row * stride + i];
            bad |= isnan(v);
            keys[e] = ((unsigned long long)orderable(v) << 32) | (unsigned)i;
        } else {
            keys[e] = ~0ull;
        }
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(nanflag, 1);
}

// one global stage (k, j >= kSeg): every pair (i, i ^ j) with i < i ^ j once
__global__ void k_bitonic_global(unsigned long long *keys, int B, int N2, int k, int j) {
    const long long half = (long long)B * (N2 / 2);
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < half; t += (long long)gridDim.x * blockDim.x) {
        const long long row = t / (N2 / 2);
        const int q = (int)(t % (N2 / 2));
        const int i = ((q / j) * 2 * j) + (q % j);   // the lower index of the pair
        unsigned long long *kr = keys + row * N2;
        const unsigned long long A = kr[i], Bk = kr[i + j];
        const bool up = (i & k) == 0;
        if ((A > Bk) == up) { kr[i] = Bk; kr[i + j] = A; }
    }
}

// the stages (k, j) for j = jmax, .., 1 (jmax < kSeg; kmin..kmax: every k in [kmin, kmax] with all
// its j) on one kSeg segment in shared memory
__global__ void __launch_bounds__(kST) k_bitonic_seg(unsigned long long *keys, int N2, int kmin, int kmax) {
    extern __shared__ unsigned long long sk_[];
    const int segs = N2 / kSeg;
    const long long row = blockIdx.x / segs;
    const int base = (blockIdx.x % segs) * kSeg;
    unsigned long long *kr = keys + row * N2 + base;
    for (int i = threadIdx.x; i < kSeg; i += kST) sk_[i] = kr[i];
    __syncthreads();
    for (int k = kmin; k <= kmax; k <<= 1) {
        for (int j = min(k >> 1, kSeg >> 1); j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < kSeg; i += kST) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const unsigned long long A = sk_[i], Bk = sk_[ixj];
                    const bool up = ((base + i) & k) == 0;
                    if ((A > Bk) == up) { sk_[i] = Bk; sk_[ixj] = A; }
                }
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < kSeg; i += kST) kr[i] = sk_[i];
}

__global__ void k_keys_out(const unsigned long long *keys, const float *__restrict__ x, int B, int n, long long stride,
                           int N2, int *perm, int *rank, float *sorted) {
    const long long tot = (long long)B * n;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
        const long long row = e / n;
        const int k = (int)(e % n);
        const int idx = (int)(keys[row * N2 + k] & 0xffffffffu);
        if (perm) perm[row * n + k] = idx;
        if (rank) rank[row * n + idx] = k;
        if (sorted) sorted[row * n + k] = x[row * stride + idx];
    }
}

size_t sort_rows_scratch_keys(int B, int n) {
    if (n <= kSeg) return 0;
    long long N2 = 1;
    while (N2 < n) N2 <<= 1;
    return (size_t)B * N2;
}

cudaError_t launch_sort_rows(const float *x, int B, int n, long long stride, int *perm, int *rank,
                             float *sorted, int *nanflag, cudaStream_t st, unsigned long long *gkeys) {
    int N2 = 1;
    while (N2 < n) N2 <<= 1;
    if (n > kSeg) {
        if (!gkeys) return cudaErrorInvalidValue;
        const size_t smem = (size_t)kSeg * sizeof(unsigned long long);
        cudaError_t e = cudaFuncSetAttribute(k_bitonic_seg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        const long long tot = (long long)B * N2;
        const int g = (int)std::min<long long>((tot + 255) / 256, 148 * 16);
        k_keys_init<<<g, 256, 0, st>>>(x, B, n, stride, N2, gkeys, nanflag);
        const int nseg = B * (N2 / kSeg);
        k_bitonic_seg<<<nseg, kST, smem, st>>>(gkeys, N2, 2, kSeg);   // every segment sorted (alternating)
        for (int k = 2 * kSeg; k <= N2; k <<= 1) {
            for (int j = k >> 1; j >= kSeg; j >>= 1) k_bitonic_global<<<g, 256, 0, st>>>(gkeys, B, N2, k, j);
            k_bitonic_seg<<<nseg, kST, smem, st>>>(gkeys, N2, k, k);   // j = kSeg / 2 .. 1 of this k
        }
        const int go = (int)std::min<long long>(((long long)B * n + 255) / 256, 148 * 16);
        k_keys_out<<<go, 256, 0, st>>>(gkeys, x, B, n, stride, N2, perm, rank, sorted);
        return cudaGetLastError();
    }
    const size_t smem = (size_t)N2 * sizeof(unsigned long long);
    cudaError_t e = cudaFuncSetAttribute(k_sort_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_sort_rows<<<B, kST, smem, st>>>(x, n, stride, perm, rank, sorted, nanflag);
    return cudaGetLastError();
}

// Block-wide inclusive scan over n elements of per-thread contiguous chunks.
// op: 0 = sum, 1 = max.  reverse: scan from the end.  Fixed order (deterministic).
__device__ void block_scan(double *v, int n, int op, bool reverse, double *tmp /* kST */) {
    const int per = (n + kST - 1) / kST;
    const int lo = threadIdx.x * per, hi = min(n, lo + per);
    auto at = [&](int i) -> double & { return v[reverse ? n - 1 - i : i]; };
    double acc = op ? -INFINITY : 0.0;
    for (int i = lo; i < hi; ++i) { acc = op ? fmax(acc, at(i)) : acc + at(i); at(i) = acc; }
    tmp[threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {  // serial scan of kST chunk totals (fixed order)
        double run = op ? -INFINITY : 0.0;
        for (int t = 0; t < kST; ++t) {
            const double c = tmp[t];
            tmp[t] = run;  // exclusive prefix
            run = op ? fmax(run, c) : run + c;
        }
    }
    __syncthreads();
    const double pre = tmp[threadIdx.x];
    for (int i = lo; i < hi; ++i) at(i) = op ? fmax(pre, at(i)) : pre + at(i);
    __syncthreads();
}

// (gscr != nullptr: n > 4096, the four n-vectors of problem b in gscr + 4 n b instead of shared
// memory; the same scans in the same order)
__global__ void __launch_bounds__(kST) k_dual_closed(const float *__restrict__ xs_all,
                                                     const int *__restrict__ perm,
                                                     const float *__restrict__ ys_all, int y_shared,
                                                     int n, float *pot, double *gscr) {
    extern __shared__ double sd[];
    __shared__ double tmp_g[kST];
    double *base = gscr ? gscr + 4LL * n * blockIdx.x : sd;
    double *F = base, *Bv = base + n, *Fm = base + 2 * n, *Bm = base + 3 * n, *tmp = gscr ? tmp_g : sd + 4 * n;
    const int prob = blockIdx.x;
    const float *xs = xs_all + (long long)prob * n;
    const float *ys = ys_all + (y_shared ? 0 : (long long)prob * n);
    // increments: F_{k+1} - F_k and B_k - B_{k+1}
    for (int k = threadIdx.x; k < n; k += kST) {
        double df = 0.0, db = 0.0;
        if (k >= 1) {
            const double xk = xs[k], xk1 = xs[k - 1], yk1 = ys[k - 1];
            df = (xk - yk1) * (xk - yk1) - (xk1 - yk1) * (xk1 - yk1);  // c_{k,k-1} - c_{k-1,k-1}
        }
        if (k + 1 < n) {
            const double xk = xs[k], yk = ys[k + 1], xk1 = xs[k + 1];
            db = (xk - yk) * (xk - yk) - (xk1 - yk) * (xk1 - yk);       // c_{k,k+1} - c_{k+1,k+1}
        }
        F[k] = df;
        Bv[k] = db;  // B_k = sum_{t >= k} db_t  (db_{n-1} = 0)
    }
    __syncthreads();
    block_scan(F, n, 0, false, tmp);
    block_scan(Bv, n, 0, true, tmp);
    for (int k = threadIdx.x; k < n; k += kST) { Fm[k] = F[k]; Bm[k] = Bv[k]; }
    __syncthreads();
    block_scan(Fm, n, 1, false, tmp);
    block_scan(Bm, n, 1, true, tmp);
    for (int k = threadIdx.x; k < n; k += kST) {
        const double fk = fmin(0.0, fmin(F[k] - Fm[k], Bv[k] - Bm[k]));
        pot[(long long)prob * n + perm[(long long)prob * n + k]] = (float)fk;
    }
}

// Paper mode: exactly L Jacobi sweeps f_i <- min_j (c_ij - c_jj + f_j) from f = 0 (fp64).
__global__ void __launch_bounds__(kST) k_dual_jacobi(const float *__restrict__ xs_all,
                                                     const int *__restrict__ perm,
                                                     const float *__restrict__ ys_all, int y_shared,
                                                     int n, int iters, float *pot) {
    extern __shared__ double sd[];
    double *xs = sd, *ys = sd + n, *cjj = sd + 2 * n, *f = sd + 3 * n, *fn = sd + 4 * n;
    const int prob = blockIdx.x;
    for (int k = threadIdx.x; k < n; k += kST) {
        xs[k] = xs_all[(long long)prob * n + k];
        ys[k] = ys_all[(y_shared ? 0 : (long long)prob * n) + k];
        cjj[k] = (xs[k] - ys[k]) * (xs[k] - ys[k]);
        f[k] = 0.0;
    }
    __syncthreads();
    for (int s = 0; s < iters; ++s) {
        for (int i = threadIdx.x; i < n; i += kST) {
            double best = INFINITY;
            const double xi = xs[i];
            for (int j = 0; j < n; ++j) {
                const double c = (xi - ys[j]) * (xi - ys[j]);
                best = fmin(best, c - cjj[j] + f[j]);
            }
            fn[i] = best;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < n; i += kST) f[i] = fn[i];
        __syncthreads();
    }
    for (int k = threadIdx.x; k < n; k += kST)
        pot[(long long)prob * n + perm[(long long)prob * n + k]] = (float)f[k];
}

cudaError_t launch_sort1d_dual(const float *xs_sorted, const int *perm, const float *ys_sorted,
                               int y_shared, int B, int n, int iters, float *pot, cudaStream_t st, double *gscr) {
    if (iters <= 0) {
        const bool glob = n > 4096;
        if (glob && !gscr) return cudaErrorInvalidValue;
        const size_t smem = glob ? 0 : (4 * (size_t)n + kST) * sizeof(double);
        cudaError_t e = cudaFuncSetAttribute(k_dual_closed, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        k_dual_closed<<<B, kST, smem, st>>>(xs_sorted, perm, ys_sorted, y_shared, n, pot, glob ? gscr : nullptr);
    } else {
        const size_t smem = 5 * (size_t)n * sizeof(double);
        cudaError_t e = cudaFuncSetAttribute(k_dual_jacobi, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        k_dual_jacobi<<<B, kST, smem, st>>>(xs_sorted, perm, ys_sorted, y_shared, n, iters, pot);
    }
    return cudaGetLastError();
}

}  // namespace sk

namespace sk {

// ------------------------------------------------------------------- K18
// General 1D initializer (Sec. 3.1 for any n, m and weights; reading R-26):
// on the sorted supports, the north-west corner plan — a staircase of edges whose
// cumulative-mass ties split it into trees — and its eps = 0 dual by Alg. 3/4
// (P:429-455): f = 0, UpdateTree for every tree, then rounds of
//     f_{s(k)} <- min_{i in T_k, j} c_ij - c_{iota(j),j} + f_{iota(j)} - (f_i - f_{s(k)})   (Jacobi, all trees)
//     UpdateTree(k) for every tree
// until f is unchanged.  One CTA per problem; the NW walk by one thread (exact ties: integers
// for uniform weights, fp64 cumulative sums otherwise), the tree walks one thread per tree, the
// root minimum over all (i, j) pairs by all threads (fp64, order-free min: deterministic).
constexpr int kNW = 512;

__device__ __forceinline__ unsigned long long ord_dbl(double v) {   // order-preserving key
    const unsigned long long u = __double_as_longlong(v);
    return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double dbl_ord(unsigned long long k) {
    return __longlong_as_double((k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k);
}

__global__ void __launch_bounds__(kNW) k_nw1d(const float *__restrict__ xs_all, const int *__restrict__ xperm_all,
                                              const float *__restrict__ ys_all, const int *__restrict__ yperm_all,
                                              int y_shared, const float *__restrict__ a, const float *__restrict__ b,
                                              int n, int m, int max_rounds, float *pot, int *rounds_out,
                                              char *gscr, long long gstride) {
    extern __shared__ double smd_[];
    const long long pr = blockIdx.x;
    // (gscr: problems beyond shared memory keep the same arrays in a global slot per problem)
    double *smd = gscr ? reinterpret_cast<double *>(gscr + pr * gstride) : smd_;
    double *X = smd, *Y = X + n, *f = Y + m, *g = f + n, *fold = g + m, *base = fold + n;
    int *ei = reinterpret_cast<int *>(base + m);   // edges (n + m - 1 at most)
    int *ej = ei + (n + m);
    int *tel = ej + (n + m);                        // tree t: edges [tel[t], tel[t + 1])
    int *iota = tel + (n + m + 1);                  // smallest source of sink j
    int *tof = iota + m;                            // tree of source i
    unsigned long long *slot = reinterpret_cast<unsigned long long *>(tof + n + 1);  // [K] (4(n+m)+1 ints + 1 pad)
    __shared__ int sK, sE, schanged;
    const float *xs = xs_all + pr * n;
    const int *xperm = xperm_all + pr * n;
    const float *ys = ys_all + (y_shared ? 0 : pr * m);
    const int *yperm = yperm_all + (y_shared ? 0 : pr * m);
    for (int i = threadIdx.x; i < n; i += kNW) X[i] = (double)xs[i];
    for (int j = threadIdx.x; j < m; j += kNW) { Y[j] = (double)ys[j]; iota[j] = -1; }
    __syncthreads();
    if (threadIdx.x == 0) {   // the NW walk: edges in staircase order, trees at the ties
        const bool uni = !a && !b;
        const float *ar = a ? a + pr * n : nullptr, *br = b ? b + (y_shared ? 0 : pr * m) : nullptr;
        double A = 0.0, Bc = 0.0;
        int k = 0, l = 0, t = 0, e = 0;
        if (!uni) {
            A = ar ? (double)ar[xperm[0]] : 1.0 / n;
            Bc = br ? (double)br[yperm[0]] : 1.0 / m;
        }
        tel[0] = 0;
        for (;;) {
            ei[e] = k; ej[e] = l; ++e;
            if (iota[l] < 0) iota[l] = k;
            tof[k] = t;
            if (k == n - 1 && l == m - 1) break;
            int step;   // 1: source, 2: sink, 3: both (a tie: a new tree)
            if (uni) {
                const long long ak = (long long)(k + 1) * m, bl = (long long)(l + 1) * n;
                step = ak < bl ? 1 : (bl < ak ? 2 : 3);
            } else {
                step = A < Bc ? 1 : (Bc < A ? 2 : 3);
            }
            if (step & 1) { ++k; if (!uni) A += ar ? (double)ar[xperm[k]] : 1.0 / n; }
            if (step & 2) { ++l; if (!uni) Bc += br ? (double)br[yperm[l]] : 1.0 / m; }
            if (step == 3) tel[++t] = e;
        }
        tel[t + 1] = e;
        sK = t + 1;
        sE = e;
    }
    __syncthreads();
    const int K = sK;
    for (int i = threadIdx.x; i < n; i += kNW) f[i] = 0.0;
    __syncthreads();
    auto cost = [&](int i, int j) { const double d = X[i] - Y[j]; return d * d; };
    auto update_trees = [&]() {   // Alg. 4 for every tree (one thread per tree)
        for (int t = threadIdx.x; t < K; t += kNW) {
            int pi = -1, pj = -1;
            for (int e = tel[t]; e < tel[t + 1]; ++e) {
                const int i = ei[e], j = ej[e];
                if (i != pi && j != pj) g[j] = cost(i, j) - f[i];        // the root's first edge
                else if (i == pi) g[j] = cost(i, j) - f[i];              // a new sink
                else f[i] = cost(i, j) - g[j];                            // a new source
                pi = i; pj = j;
            }
        }
        __syncthreads();
    };
    update_trees();
    // R-26: a root moves only if its bound is below it by more than tol (its own tight edges
    // give the root value itself up to fp64 rounding); max |C| is at a corner of the sorted cost
    const double cmax = fmax(fmax(cost(0, 0), cost(0, m - 1)), fmax(cost(n - 1, 0), cost(n - 1, m - 1)));
    const double tol = 1e-12 * fmax(1.0, cmax);
    int rounds = 0;
    for (; rounds < max_rounds;) {
        ++rounds;
        for (int i = threadIdx.x; i < n; i += kNW) fold[i] = f[i];
        for (int t = threadIdx.x; t < K; t += kNW) slot[t] = ~0ull;
        if (threadIdx.x == 0) schanged = 0;
        __syncthreads();
        for (int j = threadIdx.x; j < m; j += kNW) base[j] = -cost(iota[j], j) + fold[iota[j]];
        __syncthreads();
        // per source i: min_j c_ij + base_j - (f_i - f_root) -> its tree's slot (order-free min)
        for (int i = threadIdx.x; i < n; i += kNW) {
            const int t = tof[i];
            const int root = ei[tel[t]];
            double v = INFINITY;
            for (int j = 0; j < m; ++j) v = fmin(v, cost(i, j) + base[j] - (fold[i] - fold[root]));
            atomicMin(&slot[t], ord_dbl(v));
        }
        __syncthreads();
        for (int t = threadIdx.x; t < K; t += kNW) {
            const int root = ei[tel[t]];
            const double v = dbl_ord(slot[t]);
            if (v < fold[root] - tol) { f[root] = v; schanged = 1; }
        }
        __syncthreads();
        if (!schanged) break;
        update_trees();
    }
    for (int i = threadIdx.x; i < n; i += kNW) pot[pr * n + xperm[i]] = (float)f[i];
    if (threadIdx.x == 0 && rounds_out) rounds_out[pr] = rounds;
}

size_t nw1d_smem_bytes(int n, int m) {
    return sizeof(double) * (3 * (size_t)n + 3 * (size_t)m) + sizeof(int) * (4 * (size_t)(n + m) + 2) +
           sizeof(unsigned long long) * (size_t)(n < m ? n : m);
}

size_t nw1d_slot_bytes(int n, int m) { return (nw1d_smem_bytes(n, m) + 255) / 256 * 256; }

cudaError_t launch_nw1d(const float *xs, const int *xperm, const float *ys, const int *yperm, int y_shared,
                        const float *a, const float *b, int B, int n, int m, int max_rounds, float *pot, int *rounds,
                        cudaStream_t st, char *gscr) {
    const size_t bytes = nw1d_smem_bytes(n, m);
    if (bytes > 220 * 1024) {
        if (!gscr) return cudaErrorInvalidValue;
        k_nw1d<<<B, kNW, 0, st>>>(xs, xperm, ys, yperm, y_shared, a, b, n, m, max_rounds, pot, rounds, gscr,
                                  (long long)nw1d_slot_bytes(n, m));
        return cudaGetLastError();
    }
    cudaError_t e = cudaFuncSetAttribute(k_nw1d, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
    k_nw1d<<<B, kNW, bytes, st>>>(xs, xperm, ys, yperm, y_shared, a, b, n, m, max_rounds, pot, rounds, nullptr, 0);
    return cudaGetLastError();
}

}  // namespace sk
