// sk_gmmfit.cu — K16: fitting the K-component GMMs of the GMM initializer on the device
// (SURVEY.md NEXT-3).  P:209: "Given two empirical measures mu, nu, we fit first two
// K-component GMMs"; the paper fits them with sklearn on the CPU, which dominates its GMM
// initializer's cost.  Here: expectation-maximisation for full-covariance
// mixtures, fp64 state, from a caller-given start (reading R-23):
//     weights 1/K, means = x[idx_k], covariances = the biased covariance of x + reg I;
//   E-step  log p_ik = log w_k - 1/2 |L_k^{-1}(x_i - m_k)|^2 - log det L_k   (S_k = L_k L_k^T),
//           r_ik = exp(log p_ik - LSE_k log p_ik),  ll = mean_i LSE_k log p_ik - d/2 log 2 pi;
//   M-step  n_k = sum_i r_ik,  w_k = n_k / n,  m_k = sum_i r_ik x_i / n_k,
//           S_k = sum_i r_ik x_i x_i^T / n_k - m_k m_k^T + reg I.
// k-means start (kmeans_iters > 0, reading R-28 = sklearn's init_params="kmeans"): Lloyd from
// centers x[idx] (assign to the nearest center, ties to the lowest k; non-empty clusters move
// to their mean), a final assignment, and the M-step of those one-hot responsibilities.  The
// hard assignment reuses the E-step kernel (HARD: r_ik one-hot) and its statistics.
// Kernels per iteration: k_em_chol (one CTA per component: Cholesky, L^-1, log det),
// k_em_estep (fixed point chunks per CTA: responsibilities, then the sufficient statistics
// (n_k, sum r x, sum r x x^T upper triangle) accumulated per thread-owned statistic in fp64 and
// written as per-CTA partials), k_em_mstep (one CTA: fixed-order reduction of the partials and
// the parameter update).  Deterministic (fixed partition and reduction order).  d > 32: the
// E-step split into per-point responsibilities and tiled x x^T statistics (the *_wide kernels).
#include <algorithm>
#include <cfloat>

#include "sk_internal.h"
#include "sk_common.cuh"

namespace sk {

constexpr int kEmT = 256;
constexpr int kEmTile = 64;      // points staged per E-step tile
constexpr int kEmBlocks = 296;   // fixed point partition (2 CTAs per SM)

__host__ __device__ inline int em_stats(int K, int d) { return K * (1 + d + d * (d + 1) / 2); }
__host__ __device__ inline int em_xs(int d) { return d + 2 - (d & 1); }   // padded row stride of x tiles

// state (doubles): W[K] | MU[K d] | COV[K d d] | LINV[K d d] | LOGDET[K] | LL[1]
struct EmState {
    double *W, *MU, *COV, *LINV, *LOGDET, *LL;
};
__host__ __device__ inline EmState em_state(double *base, int K, int d) {
    EmState s;
    s.W = base;
    s.MU = s.W + K;
    s.COV = s.MU + (long long)K * d;
    s.LINV = s.COV + (long long)K * d * d;
    s.LOGDET = s.LINV + (long long)K * d * d;
    s.LL = s.LOGDET + K;
    return s;
}
// d > 32 (the wide path): a row partition of at most 48 blocks, fewer when the statistics are many
// (the partials stay <= 2^24 doubles)
inline int em_nb(int K, int d) {
    if (d <= 32) return kEmBlocks;
    const long long S1 = em_stats(K, d) + 1;
    return (int)std::max(1LL, std::min(48LL, (1LL << 24) / S1));
}
size_t em_state_doubles(int K, int d) { return (size_t)K * (1 + d + 2 * d * d + 1) + 1; }
size_t em_partial_doubles(int K, int d) { return (size_t)em_nb(K, d) * (em_stats(K, d) + 1); }   // + S + 1 reduced (em_work_doubles)
size_t em_wide_doubles(long long n, int K, int d) { return d > 32 ? (size_t)n * K + (size_t)K * d * d : 0; }
size_t em_work_doubles(int K, int d) { return em_partial_doubles(K, d) + em_stats(K, d) + 1; }

// start: w = 1/K, m_k = x[idx_k], S_k = cov0 + reg I (cov0: biased covariance of x)
__global__ void k_em_init(const float *__restrict__ x, int d, int K, const int *__restrict__ idx,
                          const double *__restrict__ cov0, double reg, double *base) {
    const EmState s = em_state(base, K, d);
    for (int e = threadIdx.x; e < K * d * d; e += blockDim.x) {
        const int r = (e / d) % d, c = e % d;
        s.COV[e] = cov0[r * d + c] + (r == c ? reg : 0.0);
    }
    for (int e = threadIdx.x; e < K * d; e += blockDim.x)
        s.MU[e] = (double)x[(long long)idx[e / d] * d + e % d];
    for (int k = threadIdx.x; k < K; k += blockDim.x) s.W[k] = 1.0 / K;
    if (threadIdx.x == 0) *s.LL = -INFINITY;   // (no previous log-likelihood)
}

// Cholesky S_k = L L^T (fp64), L^{-1}, log det L: one warp per component, lane i holding row i
// in registers.  Right-looking: step j takes the pivot from lane j, scales column j, and updates
// the trailing lower triangle with column j broadcast by shuffles.  Then lane c forward-solves
// column c of L^{-1} (L broadcast from shared memory).  DM >= d (compile-time register rows).
template <int DM>
__global__ void __launch_bounds__(32) k_em_chol(double *base, int K, int d, int *flags, const int *skip) {
    __shared__ double sL[DM * DM];
    if (skip && *(volatile const int *)skip) return;
    const EmState s = em_state(base, K, d);
    const int dd = d * d, k = blockIdx.x, lane = threadIdx.x;
    double a[DM];
#pragma unroll
    for (int c = 0; c < DM; ++c)
        a[c] = (lane < d && c < d) ? 0.5 * (s.COV[(long long)k * dd + lane * d + c] + s.COV[(long long)k * dd + c * d + lane])
                                    : 0.0;
    int bad = 0;
#pragma unroll
    for (int j = 0; j < DM; ++j) {
        if (j >= d) break;
        double v = __shfl_sync(0xffffffffu, a[j], j);   // the pivot a_jj (lane j's current value)
        if (!(v > 0.0)) { bad = 1; v = 1e-300; }
        const double ljj = sqrt(v), rj = 1.0 / ljj;
        const double lij = lane == j ? ljj : (lane > j ? a[j] * rj : 0.0);
        a[j] = lij;
#pragma unroll
        for (int c = j + 1; c < DM; ++c) {   // a_ic -= l_ij l_cj for j < c <= i
            const double lcj = __shfl_sync(0xffffffffu, lij, c);
            if (c <= lane) a[c] = fma(-lij, lcj, a[c]);
        }
    }
#pragma unroll
    for (int c = 0; c < DM; ++c)
        if (c > lane) a[c] = 0.0;
    double ld = 0.0;
#pragma unroll
    for (int c = 0; c < DM; ++c)
        if (c == lane && lane < d) ld = log(a[c]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ld += __shfl_xor_sync(0xffffffffu, ld, o);
    if (lane < d) {
#pragma unroll
        for (int c = 0; c < DM; ++c) sL[lane * DM + c] = a[c];
    }
    __syncwarp();
    if (lane == 0) {
        s.LOGDET[k] = ld;
        if (bad) atomicOr(flags, 1);
    }
    if (lane < d) {   // column `lane` of L^{-1}: Li[i] = (delta_ic - sum_{t<i} L_it Li[t]) / L_ii
        double col[DM], rd[DM];
#pragma unroll
        for (int i = 0; i < DM; ++i) rd[i] = i < d ? 1.0 / sL[i * DM + i] : 0.0;   // (independent)
#pragma unroll
        for (int i = 0; i < DM; ++i) {
            double v = i == lane ? 1.0 : 0.0;
#pragma unroll
            for (int t = 0; t < i; ++t) v = fma(-sL[i * DM + t], col[t], v);
            col[i] = v * rd[i];
        }
#pragma unroll
        for (int i = 0; i < DM; ++i)
            if (i < d) s.LINV[(long long)k * dd + i * d + lane] = col[i];
    }
}

// E-step + sufficient statistics over this CTA's fixed chunk of points.  Statistic s of
// component k (base k (1 + d + T)): 0 = n_k, 1..d = sum r x, then sum r x_a x_b for a <= b.
// OWN (K d <= kEmT): thread t = (k, a) owns n_k (a = 0), sum r x_a and the row sum r x_a x_b
// (all b in registers, the b >= a half stored): one broadcast row of x per point instead of
// three loads per statistic.  Otherwise each thread owns up to MAXS statistics.
template <int MAXS, int DM, bool HARD, bool OWN>
__global__ void __launch_bounds__(kEmT) k_em_estep(const float *__restrict__ x, long long n, int d, int K,
                                                    const double *__restrict__ base, double *part,
                                                    const int *skip) {
    extern __shared__ double sm[];
    if (skip && *(volatile const int *)skip) return;
    // row strides padded by 16 bytes: the lanes of a warp read the rows of different points /
    // components at once, and unpadded 128-byte multiples would put them all in the same banks
    const int XS = em_xs(d);
    constexpr int LS = DM * DM + 2, MS = DM + 2;
    double *xs = sm;                          // [kEmTile][XS]
    double *rs = xs + kEmTile * XS;           // [kEmTile][K]
    double *lls = rs + kEmTile * K;           // [kEmTile]
    double *sL = lls + kEmTile;               // [K][LS] L^{-1} rows (lower triangle used)
    double *sM = sL + K * LS;                 // [K][MS] means
    double *sC = sM + K * MS;                 // [K] log w_k - log det L_k
    const EmState s = em_state(const_cast<double *>(base), K, d);
    if (!HARD)
        for (int e = threadIdx.x; e < K * DM * DM; e += kEmT) {
            const int k = e / (DM * DM), r = (e / DM) % DM, c = e % DM;
            sL[k * LS + r * DM + c] = (r < d && c < d) ? s.LINV[(long long)k * d * d + r * d + c] : 0.0;
        }
    for (int e = threadIdx.x; e < K * DM; e += kEmT) {
        const int k = e / DM, c = e % DM;
        sM[k * MS + c] = c < d ? s.MU[(long long)k * d + c] : 0.0;
    }
    if (!HARD)
        for (int k = threadIdx.x; k < K; k += kEmT) sC[k] = log(s.W[k]) - s.LOGDET[k];
    const int T = d * (d + 1) / 2, per = 1 + d + T, S = K * per;
    const long long chunk = (n + gridDim.x - 1) / gridDim.x;
    const long long p0 = blockIdx.x * chunk, p1 = min(n, p0 + chunk);
    // this thread's statistics: (k, kind, a, b) decoded once
    double acc[MAXS];
    short sk_[MAXS], sa[MAXS], sb[MAXS];
#pragma unroll
    for (int u = 0; u < MAXS; ++u) {
        acc[u] = 0.0;
        const int st = threadIdx.x + u * kEmT;
        sk_[u] = -1;
        if (st < S) {
            const int k = st / per, o = st % per;
            sk_[u] = (short)k;
            if (o == 0) { sa[u] = -1; sb[u] = -1; }
            else if (o <= d) { sa[u] = (short)(o - 1); sb[u] = -1; }
            else {   // packed upper triangle, row-major: (a, b), a <= b
                int q = o - 1 - d, a = 0;
                while (q >= d - a) { q -= d - a; ++a; }
                sa[u] = (short)a; sb[u] = (short)(a + q);
            }
        }
    }
    double ll = 0.0;
    const int ok = threadIdx.x / d, oa = threadIdx.x % d;   // OWN: this thread's (k, a)
    const bool owner = OWN && (int)threadIdx.x < K * d;
    double on = 0.0, osum = 0.0, oxx[OWN ? DM : 1];
#pragma unroll
    for (int b = 0; b < (OWN ? DM : 1); ++b) oxx[b] = 0.0;
    for (long long t0 = p0; t0 < p1; t0 += kEmTile) {
        const int np = (int)min((long long)kEmTile, p1 - t0);
        for (int e = threadIdx.x; e < np * d; e += kEmT) xs[(e / d) * XS + e % d] = (double)x[(t0 + e / d) * d + e % d];
        __syncthreads();
        // log p of (point, component) pairs.  K <= 32: groups of G = pow2 >= K consecutive lanes
        // per point, so the normalisation (max, sum of exps / the nearest center) is a group
        // shuffle reduction with one exponential per lane; otherwise one thread per point.
        auto logp = [&](int pp, int k) {
            const double *xi = xs + pp * XS;
            const double *Li = sL + k * LS;
            const double *mk = sM + k * MS;
            double dx[DM];
#pragma unroll
            for (int c = 0; c < DM; ++c) dx[c] = c < d ? xi[c] - mk[c] : 0.0;
            double q = 0.0;
            if (HARD) {   // k-means: minus the squared distance (summed in coordinate order)
#pragma unroll
                for (int c = 0; c < DM; ++c) q += dx[c] * dx[c];
                return -q;
            }
#pragma unroll
            for (int r = 0; r < DM; ++r) {
                double z = 0.0;
#pragma unroll
                for (int c = 0; c <= r; ++c) z = fma(Li[r * DM + c], dx[c], z);
                q = fma(z, z, q);   // (rows r >= d are zero)
            }
            return sC[k] - 0.5 * q;
        };
        if (K <= 32) {
            const int G = K <= 1 ? 1 : 1 << (32 - __clz(K - 1));
            for (int b0 = 0; b0 < np; b0 += kEmT / G) {
                const int pp = b0 + (int)threadIdx.x / G, k = (int)threadIdx.x % G;
                const bool live = pp < np && k < K;
                const double lp = live ? logp(pp, k) : -INFINITY;
                double mx = lp;
                int kb = live ? k : 1 << 30;
                for (int o = G / 2; o > 0; o >>= 1) {   // max; HARD: the first maximum's k
                    const double om = __shfl_xor_sync(0xffffffffu, mx, o);
                    const int okb = __shfl_xor_sync(0xffffffffu, kb, o);
                    if (om > mx || (om == mx && okb < kb)) { mx = om; kb = okb; }
                }
                if (HARD) {
                    if (live) rs[pp * K + k] = k == kb ? 1.0 : 0.0;
                    if (live && k == 0) lls[pp] = -mx;   // (inertia)
                } else {
                    double den = live ? exp(lp - mx) : 0.0;
                    for (int o = G / 2; o > 0; o >>= 1) den += __shfl_xor_sync(0xffffffffu, den, o);
                    const double lse = mx + log(den);
                    if (live) rs[pp * K + k] = exp(lp - lse);
                    if (live && k == 0) lls[pp] = lse;
                }
            }
        } else {
            for (int e = threadIdx.x; e < np * K; e += kEmT) rs[e] = logp(e / K, e % K);
            __syncthreads();
            if (HARD && threadIdx.x < np) {   // nearest center, ties to the lowest k: one-hot
                double *ri = rs + threadIdx.x * K;
                int kb = 0;
                for (int k = 1; k < K; ++k)
                    if (ri[k] > ri[kb]) kb = k;
                lls[threadIdx.x] = -ri[kb];   // (inertia)
                for (int k = 0; k < K; ++k) ri[k] = k == kb ? 1.0 : 0.0;
            } else if (threadIdx.x < np) {   // normalise point t0 + threadIdx.x (fixed k order)
                double *ri = rs + threadIdx.x * K;
                double mx = -INFINITY;
                for (int k = 0; k < K; ++k) mx = fmax(mx, ri[k]);
                double den = 0.0;
                for (int k = 0; k < K; ++k) den += exp(ri[k] - mx);
                const double lse = mx + log(den);
                for (int k = 0; k < K; ++k) ri[k] = exp(ri[k] - lse);
                lls[threadIdx.x] = lse;
            }
        }
        __syncthreads();
        if constexpr (OWN) {
            if (owner) {
                for (int p = 0; p < np; ++p) {
                    const double r = rs[p * K + ok];
                    const double *xp = xs + p * XS;
                    const double ra = r * xp[oa];
                    on += r;
                    osum += ra;
#pragma unroll
                    for (int b = 0; b < DM; ++b)
                        if (b < d) oxx[b] = fma(ra, xp[b], oxx[b]);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < (OWN ? 0 : MAXS); ++u) {
            if (sk_[u] < 0) continue;
            const int k = sk_[u], a = sa[u], b = sb[u];
            double v = acc[u];
            for (int p = 0; p < np; ++p) {
                const double r = rs[p * K + k];
                const double f = a < 0 ? 1.0 : (b < 0 ? xs[p * XS + a] : xs[p * XS + a] * xs[p * XS + b]);
                v = fma(r, f, v);
            }
            acc[u] = v;
        }
        if (threadIdx.x == 0)
            for (int p = 0; p < np; ++p) ll += lls[p];
        __syncthreads();
    }
    double *out = part + (long long)blockIdx.x * (S + 1);
    if constexpr (OWN) {
        if (owner) {
            double *ok_out = out + ok * per;
            if (oa == 0) ok_out[0] = on;
            ok_out[1 + oa] = osum;
            const int o0 = 1 + d + oa * d - oa * (oa - 1) / 2;   // packed (a, a)
#pragma unroll
            for (int b = 0; b < DM; ++b)
                if (b >= oa && b < d) ok_out[o0 + (b - oa)] = oxx[b];
        }
    }
#pragma unroll
    for (int u = 0; u < (OWN ? 0 : MAXS); ++u) {
        const int st = threadIdx.x + u * kEmT;
        if (st < S) out[st] = acc[u];
    }
    if (threadIdx.x == 0) out[S] = ll;
}

// Reduction of the per-CTA partials, one warp per statistic: lane l sums CTAs l, l + 32, ... in
// order, then a fixed shuffle tree (deterministic).  out[S + 1].
__global__ void __launch_bounds__(kEmT) k_em_reduce(const double *part, int nb, int S1, double *out, const int *skip) {
    if (skip && *(volatile const int *)skip) return;
    const int st = (blockIdx.x * kEmT + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (st >= S1) return;
    double v = 0.0;
    for (int b = lane; b < nb; b += 32) v += part[(long long)b * S1 + st];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) out[st] = v;
}

// M-step from the reduced statistics: w, m, S (+ reg I) and the mean log-likelihood of the E-step
// that produced them.
// mode 0: EM step (tracks convergence: *LL holds the previous E-step's log-likelihood; flags[1]
// = converged (|ll - ll_prev| < tol, the later EM kernels then return at once), flags[2] = EM
// steps done); mode 1: the k-means start's one-hot M-step (LL reset to -inf); mode 2: the
// evaluation pass into the scratch state (LL only matters).
__global__ void __launch_bounds__(kEmT) k_em_mstep(const double *tot, long long n, int d, int K, double reg,
                                                    double *base, int mode, double tol, int *flags) {
    if (mode == 0 && *(volatile const int *)&flags[1]) return;
    const EmState s = em_state(base, K, d);
    const double ll_prev = *s.LL;
    __syncthreads();
    const int T = d * (d + 1) / 2, per = 1 + d + T, S = K * per;
    const double eps10 = 10.0 * DBL_EPSILON;   // (as sklearn: n_k + 10 eps guards empty components)
    for (int e = threadIdx.x; e < K * d; e += blockDim.x) {
        const int k = e / d, a = e % d;
        s.MU[e] = tot[k * per + 1 + a] / (tot[k * per] + eps10);
    }
    for (int k = threadIdx.x; k < K; k += blockDim.x) s.W[k] = (tot[k * per] + eps10) / (double)n;
    __syncthreads();
    for (int e = threadIdx.x; e < K * d * d; e += blockDim.x) {
        const int k = e / (d * d), r = (e / d) % d, c = e % d;
        const int a = min(r, c), b = max(r, c);
        const int o = 1 + d + a * d - a * (a - 1) / 2 + (b - a);   // packed (a, b), a <= b
        const double nk = tot[k * per] + eps10;
        s.COV[e] = tot[k * per + o] / nk - s.MU[k * d + r] * s.MU[k * d + c] + (r == c ? reg : 0.0);
    }
    if (threadIdx.x == 0) {
        const double ll = tot[S] / (double)n - 0.5 * d * log(2.0 * 3.14159265358979323846);
        *s.LL = mode == 1 ? -INFINITY : ll;
        if (mode == 0) {
            flags[2] += 1;
            if (tol > 0.0 && fabs(ll - ll_prev) < tol) flags[1] = 1;
        }
    }
}

// Lloyd's center update from the hard statistics: a non-empty cluster moves to its mean.
__global__ void k_km_update(const double *tot, int d, int K, double *base) {
    const EmState s = em_state(base, K, d);
    const int per = 1 + d + d * (d + 1) / 2;
    for (int e = threadIdx.x; e < K * d; e += blockDim.x) {
        const int k = e / d, a = e % d;
        const double nk = tot[k * per];
        if (nk > 0.0) s.MU[e] = tot[k * per + 1 + a] / nk;
    }
}

__global__ void k_em_out(const double *base, int K, int d, float *w, float *mu, float *cov, double *ll_out) {
    const EmState s = em_state(const_cast<double *>(base), K, d);
    for (int e = threadIdx.x; e < K * d * d; e += blockDim.x) cov[e] = (float)s.COV[e];
    for (int e = threadIdx.x; e < K * d; e += blockDim.x) mu[e] = (float)s.MU[e];
    for (int k = threadIdx.x; k < K; k += blockDim.x) w[k] = (float)s.W[k];
    if (threadIdx.x == 0 && ll_out) *ll_out = *s.LL;
}

// ---------------------------------------------------------------- d in (32, 256]
// The same EM with the per-component work split differently: Cholesky one CTA per component (L in
// a scratch slot, rows below each pivot in parallel); responsibilities one thread per point
// (log p_ik for all k from L^-1 rows read as broadcasts, normalised in k order, written to
// resp [n][K]); the statistics of each (row block, component, 64 x 64 tile of x x^T) by one CTA
// (rows in order, as the fused E-step), n_k and sum r x by the tile-(0, 0) CTA.  Same partials
// layout, reduction, M-step and stopping rule as d <= 32.
__global__ void __launch_bounds__(kEmT) k_em_chol_wide(double *base, int K, int d, int *flags, const int *skip,
                                                        double *Lscr) {
    __shared__ double s_ljj;
    if (skip && *(volatile const int *)skip) return;
    const EmState s = em_state(base, K, d);
    const long long dd = (long long)d * d;
    const int k = blockIdx.x;
    double *L = Lscr + k * dd, *Li = s.LINV + k * dd;
    for (long long e = threadIdx.x; e < dd; e += blockDim.x) {
        const int i = (int)(e / d), j = (int)(e % d);
        L[e] = 0.5 * (s.COV[k * dd + (long long)i * d + j] + s.COV[k * dd + (long long)j * d + i]);
    }
    __syncthreads();
    int bad = 0;
    for (int j = 0; j < d; ++j) {
        if (threadIdx.x == 0) {
            double v = __ldcg(L + (long long)j * d + j);
            for (int t = 0; t < j; ++t) { const double a = __ldcg(L + (long long)j * d + t); v -= a * a; }
            if (!(v > 0.0)) { bad = 1; v = 1e-300; }
            s_ljj = sqrt(v);
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
    if (threadIdx.x == 0) {
        double ld = 0.0;
        for (int j = 0; j < d; ++j) ld += log(__ldcg(L + (long long)j * d + j));
        s.LOGDET[k] = ld;
        if (bad) atomicOr(flags, 1);
    }
    for (int c = threadIdx.x; c < d; c += blockDim.x)
        for (int i = 0; i < d; ++i) {
            double v = (i == c) ? 1.0 : 0.0;
            for (int t = c; t < i; ++t) v -= __ldcg(L + (long long)i * d + t) * __ldcg(Li + (long long)t * d + c);
            Li[(long long)i * d + c] = i < c ? 0.0 : v / __ldcg(L + (long long)i * d + i);
        }
}

template <bool HARD>
__global__ void __launch_bounds__(kEmT) k_em_resp_wide(const float *__restrict__ x, long long n, int d, int K,
                                                        const double *__restrict__ base, double *resp, double *part,
                                                        const int *skip) {
    __shared__ double lls[kEmT];
    if (skip && *(volatile const int *)skip) return;
    const EmState s = em_state(const_cast<double *>(base), K, d);
    const int S = em_stats(K, d);
    const long long chunk = (n + gridDim.x - 1) / gridDim.x;
    const long long p0 = blockIdx.x * chunk, p1 = min(n, p0 + chunk);
    double ll = 0.0;
    for (long long t0 = p0; t0 < p1; t0 += kEmT) {
        const long long i = t0 + threadIdx.x;
        if (i < p1) {
            const float *xi = x + i * d;
            double *ri = resp + i * K;
            double mx = -INFINITY;
            int kb = 0;
            for (int k = 0; k < K; ++k) {
                const double *mk = s.MU + (long long)k * d;
                double q = 0.0;
                if (HARD) {
                    for (int c = 0; c < d; ++c) { const double t = (double)xi[c] - mk[c]; q += t * t; }
                    q = -q;
                    if (q > mx) { mx = q; kb = k; }
                } else {
                    const double *Lk = s.LINV + (long long)k * d * d;
                    double qq = 0.0;
                    for (int r = 0; r < d; ++r) {
                        double z = 0.0;
                        for (int c = 0; c <= r; ++c) z = fma(Lk[(long long)r * d + c], (double)xi[c] - mk[c], z);
                        qq = fma(z, z, qq);
                    }
                    q = log(s.W[k]) - s.LOGDET[k] - 0.5 * qq;
                    mx = fmax(mx, q);
                }
                ri[k] = q;
            }
            if (HARD) {
                for (int k = 0; k < K; ++k) ri[k] = k == kb ? 1.0 : 0.0;
                lls[threadIdx.x] = -mx;   // (inertia)
            } else {
                double den = 0.0;
                for (int k = 0; k < K; ++k) den += exp(ri[k] - mx);
                const double lse = mx + log(den);
                for (int k = 0; k < K; ++k) ri[k] = exp(ri[k] - lse);
                lls[threadIdx.x] = lse;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            const int np = (int)min((long long)kEmT, p1 - t0);
            for (int p = 0; p < np; ++p) ll += lls[p];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) part[(long long)blockIdx.x * (S + 1) + S] = ll;
}

__global__ void __launch_bounds__(kEmT) k_em_stats_wide(const float *__restrict__ x, long long n, int d, int K,
                                                         const double *__restrict__ resp, double *part,
                                                         const int *skip) {
    constexpr int CH = 32;
    __shared__ double xa[CH][65], xb[CH][65], rr[CH];
    if (skip && *(volatile const int *)skip) return;
    const int nt = (d + 63) / 64, ti = blockIdx.x / nt, tj = blockIdx.x % nt;
    if (ti > tj) return;   // (the packed upper triangle only)
    const int k = blockIdx.y, b = blockIdx.z;
    const int i0 = ti * 64, j0 = tj * 64;
    const int T = d * (d + 1) / 2, per = 1 + d + T, S = K * per;
    const long long chunk = (n + gridDim.z - 1) / gridDim.z;
    const long long p0 = b * chunk, p1 = min(n, p0 + chunk);
    const int br = threadIdx.x >> 4, bc = threadIdx.x & 15;
    double acc[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
    double nk = 0.0, sx = 0.0;   // tile (0, 0): n_k (thread 0) and sum r x_a (thread a < d)
    const bool first = blockIdx.x == 0;
    for (long long c0 = p0; c0 < p1; c0 += CH) {
        const int cnt = (int)min((long long)CH, p1 - c0);
        __syncthreads();
        for (int t = threadIdx.x; t < cnt * 64; t += kEmT) {
            const int r = t / 64, c = t % 64;
            const long long row = (c0 + r) * d;
            xa[r][c] = i0 + c < d ? (double)x[row + i0 + c] : 0.0;
            xb[r][c] = j0 + c < d ? (double)x[row + j0 + c] : 0.0;
        }
        for (int r = threadIdx.x; r < cnt; r += kEmT) rr[r] = resp[(c0 + r) * K + k];
        __syncthreads();
        for (int r = 0; r < cnt; ++r) {
            const double w = rr[r];
            double a[4], bb[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) a[u] = w * xa[r][br + 16 * u];
#pragma unroll
            for (int v = 0; v < 4; ++v) bb[v] = xb[r][bc + 16 * v];
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], bb[v], acc[u][v]);
        }
        if (first) {
            for (int r = 0; r < cnt; ++r) {
                const double w = rr[r];
                if (threadIdx.x == 0) nk += w;
                if ((int)threadIdx.x < d) sx = fma(w, (double)x[(c0 + r) * d + threadIdx.x], sx);
            }
        }
    }
    double *out = part + (long long)b * (S + 1) + (long long)k * per;
    if (first) {
        if (threadIdx.x == 0) out[0] = nk;
        if ((int)threadIdx.x < d) out[1 + threadIdx.x] = sx;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int a = i0 + br + 16 * u, c = j0 + bc + 16 * v;
            if (a < d && c < d && c >= a) out[1 + d + a * d - a * (a - 1) / 2 + (c - a)] = acc[u][v];
        }
}

template <bool HARD>
static cudaError_t launch_estep_wide(const float *x, long long n, int d, int K, const double *base, double *part,
                                     double *resp, const int *skip, cudaStream_t st) {
    const int nb = em_nb(K, d), nt = (d + 63) / 64;
    k_em_resp_wide<HARD><<<nb, kEmT, 0, st>>>(x, n, d, K, base, resp, part, skip);
    k_em_stats_wide<<<dim3((unsigned)(nt * nt), (unsigned)K, (unsigned)nb), kEmT, 0, st>>>(x, n, d, K, resp, part, skip);
    return cudaGetLastError();
}

template <int MAXS, int DM, bool HARD, bool OWN>
static cudaError_t launch_estep_d(const float *x, long long n, int d, int K, const double *base, double *part,
                                  const int *skip, cudaStream_t st) {
    const size_t smem = sizeof(double) * ((size_t)kEmTile * (em_xs(d) + K) + kEmTile + (size_t)K * (DM * DM + DM + 5));
    cudaError_t e = cudaFuncSetAttribute(k_em_estep<MAXS, DM, HARD, OWN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    k_em_estep<MAXS, DM, HARD, OWN><<<kEmBlocks, kEmT, smem, st>>>(x, n, d, K, base, part, skip);
    return cudaGetLastError();
}
template <int MAXS, bool HARD, bool OWN>
static cudaError_t launch_estep_m(const float *x, long long n, int d, int K, const double *base, double *part,
                                  const int *skip, cudaStream_t st) {
    if (d <= 8) return launch_estep_d<MAXS, 8, HARD, OWN>(x, n, d, K, base, part, skip, st);
    if (d <= 16) return launch_estep_d<MAXS, 16, HARD, OWN>(x, n, d, K, base, part, skip, st);
    return launch_estep_d<MAXS, 32, HARD, OWN>(x, n, d, K, base, part, skip, st);
}
template <bool HARD>
static cudaError_t launch_estep(int maxs, const float *x, long long n, int d, int K, const double *base,
                                double *part, const int *skip, cudaStream_t st) {
    if (K * d <= kEmT) return launch_estep_m<1, HARD, true>(x, n, d, K, base, part, skip, st);
    if (maxs <= 8) return launch_estep_m<8, HARD, false>(x, n, d, K, base, part, skip, st);
    if (maxs <= 20) return launch_estep_m<20, HARD, false>(x, n, d, K, base, part, skip, st);
    return launch_estep_m<40, HARD, false>(x, n, d, K, base, part, skip, st);
}

// iters EM steps from the start above; the state (em_state_doubles) and partials
// (em_partial_doubles) are caller workspace; cov0 = biased covariance of x (d x d).  A final
// E-step evaluates the mean log-likelihood of the returned parameters.
cudaError_t launch_gmm_fit(const float *x, long long n, int d, int K, const int *idx, const double *cov0,
                           int kmeans_iters, int iters, double tol, double reg, double *state, double *part,
                           int *flags, float *w, float *mu, float *cov, double *ll_out, int *h_conv,
                           cudaStream_t st, double *wide) {
    const int S = em_stats(K, d);
    const int maxs = (S + kEmT - 1) / kEmT;
    const bool wd = d > 32;
    if (d < 1 || d > 256 || K < 1 || K > 64 || (!wd && maxs > 40) || (wd && !wide)) return cudaErrorInvalidValue;
    const int nb = em_nb(K, d);
    double *resp = wide, *Lscr = wide ? wide + n * K : nullptr;
    auto estep = [&](bool hard, const int *sk) {
        if (wd) return hard ? launch_estep_wide<true>(x, n, d, K, state, part, resp, sk, st)
                            : launch_estep_wide<false>(x, n, d, K, state, part, resp, sk, st);
        return hard ? launch_estep<true>(maxs, x, n, d, K, state, part, sk, st)
                    : launch_estep<false>(maxs, x, n, d, K, state, part, sk, st);
    };
    k_em_init<<<1, kEmT, 0, st>>>(x, d, K, idx, cov0, reg, state);
    double *tot = part + em_partial_doubles(K, d);   // [S + 1] after the partials
    const int rblocks = (32 * (S + 1) + kEmT - 1) / kEmT;
    cudaError_t e = cudaSuccess;
    for (int t = 0; t <= kmeans_iters && kmeans_iters > 0; ++t) {   // Lloyd, then the one-hot M-step
        e = estep(true, nullptr);
        if (e != cudaSuccess) return e;
        k_em_reduce<<<rblocks, kEmT, 0, st>>>(part, nb, S + 1, tot, nullptr);
        if (t < kmeans_iters) k_km_update<<<1, kEmT, 0, st>>>(tot, d, K, state);
        else k_em_mstep<<<1, kEmT, 0, st>>>(tot, n, d, K, reg, state, 1, 0.0, flags);
    }
    const int *skip = flags + 1;   // set once EM has converged (tol > 0): the rest are no-ops
    int poll = 2, next_poll = 2;   // tol > 0: the host reads the flag after 2, 4, 8, ... steps
    for (int it = 0; it <= iters; ++it) {
        if (tol > 0.0 && h_conv && it == next_poll && it < iters) {
            e = cudaMemcpyAsync(h_conv, flags + 1, sizeof(int), cudaMemcpyDeviceToHost, st);
            if (e == cudaSuccess) e = cudaStreamSynchronize(st);
            if (e != cudaSuccess) return e;
            if (*h_conv) it = iters;   // straight to the evaluation pass
            poll *= 2;
            next_poll = it + poll;
        }
        const bool eval = it == iters;   // evaluation only: the log-likelihood of the returned parameters
        const int *sk = eval ? nullptr : skip;
        if (wd) k_em_chol_wide<<<K, kEmT, 0, st>>>(state, K, d, flags, sk, Lscr);
        else if (d <= 8) k_em_chol<8><<<K, 32, 0, st>>>(state, K, d, flags, sk);
        else if (d <= 16) k_em_chol<16><<<K, 32, 0, st>>>(state, K, d, flags, sk);
        else k_em_chol<32><<<K, 32, 0, st>>>(state, K, d, flags, sk);
        e = estep(false, sk);
        if (e != cudaSuccess) return e;
        k_em_reduce<<<rblocks, kEmT, 0, st>>>(part, nb, S + 1, tot, sk);
        if (eval) {
            k_em_mstep<<<1, kEmT, 0, st>>>(tot, n, d, K, reg, state + em_state_doubles(K, d), 2, 0.0, flags);
            break;
        }
        k_em_mstep<<<1, kEmT, 0, st>>>(tot, n, d, K, reg, state, 0, tol, flags);
    }
    // the evaluation pass wrote a scratch state; its LL is the returned parameters' likelihood
    const EmState scratch = em_state(state + em_state_doubles(K, d), K, d);
    e = cudaMemcpyAsync(em_state(state, K, d).LL, scratch.LL, sizeof(double), cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return e;
    k_em_out<<<1, kEmT, 0, st>>>(state, K, d, w, mu, cov, ll_out);
    return cudaGetLastError();
}

int gmm_fit_blocks() { return kEmBlocks; }

}  // namespace sk
