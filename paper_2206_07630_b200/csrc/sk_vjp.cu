// sk_vjp.cu — K17: implicit differentiation of the Sinkhorn potentials.
//
// With H(f, g) = [grad_1 E; grad_2 E] = [a - P 1; b - P^T 1] (Eq. 2), P_ij = exp((f_i + g_j - C_ij)/eps),
// H = 0 at the optimum (f*, g*) and the implicit function theorem gives, for a cotangent z on
// (f*, g*):   J_F^T z = - J_H,.^T (J_H,(f,g)^T)^{-1} z.   Here J_H,(f,g) = -(1/eps) M with
//     M = [[diag(r), P], [P^T, diag(c)]],   r = P 1,  c = P^T 1,
// symmetric positive semi-definite with the null vector e = (1_n, -1_m) (the shift of (f, g)).
// The VJP is eps J_H,.^T w with w = M^+ z (z projected on e^perp; min-norm w), and for the
// squared-Euclidean cost (C_ij = |x_i - y_j|^2):
//     grad_x_i = 2 sum_j P_ij (w_f,i + w_g,j)(x_i - y_j),   grad_y_j = 2 sum_i P_ij (w_f,i + w_g,j)(y_j - x_i),
//     grad_a = eps w_f,   grad_b = eps w_g.
// w solves M w = z by conjugate gradients preconditioned with diag(r, c) (fp64 vectors, the two
// plan products per iteration are K17a passes); deterministic (fixed reduction orders).
#include <cmath>

#include "sk_internal.h"
#include "sk_common.cuh"

namespace sk {

constexpr int kVT = 128;       // output points per CTA of the plan pass
constexpr int kVTile = 128;    // reduced points staged per tile
constexpr int kVecT = 1024;    // the single-CTA vector kernels

// K17a: for each output point p (coordinates ps, potential hp) over the reduced side (qs, hq):
//   A[p]    = sum_q P_pq v_q                                   (v == nullptr: v = 1)
//   G[p][k] = sum_q P_pq (s_p + v_q)(p_k - q_k)                (if G != nullptr; s == nullptr: 0)
// P_pq = exp((hp_p + hq_q - |p - q|^2)/eps) with the direct difference (fp32 terms, fp64 sums).
template <int DM>
__global__ void __launch_bounds__(kVT) k_plan_pass(const float *__restrict__ ps, const float *__restrict__ hp, int P,
                                                   const float *__restrict__ qs, const float *__restrict__ hq, int Q,
                                                   int d, float eps, const double *__restrict__ s,
                                                   const double *__restrict__ v, double *A, double *G) {
    __shared__ float qc[DM][kVTile];
    __shared__ float qh[kVTile];
    __shared__ double qv[kVTile];
    const int p = blockIdx.x * kVT + threadIdx.x;
    const float kap = kLog2e / eps;
    float pc[DM];
#pragma unroll
    for (int k = 0; k < DM; ++k) pc[k] = (p < P && k < d) ? ps[(long long)p * d + k] : 0.f;
    const float hpp = p < P ? hp[p] : 0.f;
    const double sp = (s && p < P) ? s[p] : 0.0;
    double a = 0.0, gk[DM];
#pragma unroll
    for (int k = 0; k < DM; ++k) gk[k] = 0.0;
    for (int q0 = 0; q0 < Q; q0 += kVTile) {
        const int nq = min(kVTile, Q - q0);
        __syncthreads();
        for (int e = threadIdx.x; e < kVTile; e += kVT) {
            const bool ok = e < nq;
#pragma unroll
            for (int k = 0; k < DM; ++k) qc[k][e] = (ok && k < d) ? qs[(long long)(q0 + e) * d + k] : 0.f;
            qh[e] = ok ? hq[q0 + e] : 0.f;
            qv[e] = ok ? (v ? v[q0 + e] : 1.0) : 0.0;
        }
        __syncthreads();
        for (int j = 0; j < nq; ++j) {
            float c = 0.f;
#pragma unroll
            for (int k = 0; k < DM; ++k) {
                const float df = pc[k] - qc[k][j];
                c = fmaf(df, df, c);
            }
            const double pw = (double)ex2((hpp + qh[j] - c) * kap);
            a = fma(pw, qv[j], a);
            if (G) {
                const double wt = pw * (sp + qv[j]);
#pragma unroll
                for (int k = 0; k < DM; ++k) gk[k] = fma(wt, (double)(pc[k] - qc[k][j]), gk[k]);
            }
        }
    }
    if (p >= P) return;
    if (A) A[p] = a;
    if (G)
#pragma unroll
        for (int k = 0; k < DM; ++k)
            if (k < d) G[(long long)p * d + k] = gk[k];
}

static int dm_of(int d) { return d <= 4 ? 4 : (d <= 16 ? 16 : (d <= 32 ? 32 : (d <= 64 ? 64 : (d <= 256 ? 256 : 0)))); }

// K17a for d in (64, 256]: 32 output points per CTA, 256 threads.  Per 32-point reduced tile:
// phase 1, thread (p, u) forms P_pq for q = u, u + 8, .. (the cost in k order with direct fp32
// differences, as above) into shared memory; phase 2, thread p sums A[p] over the tile in q order
// and threads (p, u) accumulate G[p][k] for k = u, u + 8, .. (32 doubles each) in q order.
constexpr int kVWP = 32, kVWQ = 32, kVWT = 256;
__global__ void __launch_bounds__(kVWT) k_plan_pass_wide(const float *__restrict__ ps, const float *__restrict__ hp,
                                                         int P, const float *__restrict__ qs,
                                                         const float *__restrict__ hq, int Q, int d, float eps,
                                                         const double *__restrict__ s, const double *__restrict__ v,
                                                         double *A, double *G) {
    extern __shared__ float wsm[];
    const int d1 = d + 1;
    float *sp = wsm;                        // [kVWP][d + 1]
    float *sq = sp + kVWP * d1;             // [kVWQ][d + 1]
    double *pw = reinterpret_cast<double *>(sq + kVWQ * d1 + ((kVWP + kVWQ) * d1 & 1));   // [kVWP][kVWQ]
    double *qv = pw + kVWP * kVWQ;          // [kVWQ]
    float *qh = reinterpret_cast<float *>(qv + kVWQ);   // [kVWQ]
    const int p0 = blockIdx.x * kVWP;
    const int pl = threadIdx.x >> 3, u = threadIdx.x & 7;
    const int p = p0 + pl;
    const float kap = kLog2e / eps;
    for (int e = threadIdx.x; e < kVWP * d; e += kVWT) {
        const int r = e / d, k = e % d;
        sp[r * d1 + k] = p0 + r < P ? ps[(long long)(p0 + r) * d + k] : 0.f;
    }
    const float hpp = p < P ? hp[p] : 0.f;
    const double spp = (s && p < P) ? s[p] : 0.0;
    double a = 0.0, gk[32];
#pragma unroll
    for (int t = 0; t < 32; ++t) gk[t] = 0.0;
    for (int q0 = 0; q0 < Q; q0 += kVWQ) {
        const int nq = min(kVWQ, Q - q0);
        __syncthreads();
        for (int e = threadIdx.x; e < kVWQ * d; e += kVWT) {
            const int r = e / d, k = e % d;
            sq[r * d1 + k] = r < nq ? qs[(long long)(q0 + r) * d + k] : 0.f;
        }
        for (int e = threadIdx.x; e < kVWQ; e += kVWT) {
            qh[e] = e < nq ? hq[q0 + e] : 0.f;
            qv[e] = e < nq ? (v ? v[q0 + e] : 1.0) : 0.0;
        }
        __syncthreads();
        for (int j = u; j < nq; j += 8) {
            const float *pp = sp + pl * d1, *qq = sq + j * d1;
            float c = 0.f;
            for (int k = 0; k < d; ++k) {
                const float df = pp[k] - qq[k];
                c = fmaf(df, df, c);
            }
            pw[pl * kVWQ + j] = (double)ex2((hpp + qh[j] - c) * kap);
        }
        __syncthreads();
        if (u == 0)
            for (int j = 0; j < nq; ++j) a = fma(pw[pl * kVWQ + j], qv[j], a);
        if (G) {
            const float *pp = sp + pl * d1;
            for (int j = 0; j < nq; ++j) {
                const double wt = pw[pl * kVWQ + j] * (spp + qv[j]);
                const float *qq = sq + j * d1;
#pragma unroll
                for (int t = 0; t < 32; ++t) {
                    const int k = u + 8 * t;
                    if (k < d) gk[t] = fma(wt, (double)(pp[k] - qq[k]), gk[t]);
                }
            }
        }
    }
    if (p >= P) return;
    if (A && u == 0) A[p] = a;
    if (G)
#pragma unroll
        for (int t = 0; t < 32; ++t) {
            const int k = u + 8 * t;
            if (k < d) G[(long long)p * d + k] = gk[t];
        }
}

cudaError_t launch_plan_pass(const float *ps, const float *hp, int P, const float *qs, const float *hq, int Q, int d,
                             float eps, const double *s, const double *v, double *A, double *G, cudaStream_t st) {
    const int grid = (P + kVT - 1) / kVT;
    switch (dm_of(d)) {
        case 4: k_plan_pass<4><<<grid, kVT, 0, st>>>(ps, hp, P, qs, hq, Q, d, eps, s, v, A, G); break;
        case 16: k_plan_pass<16><<<grid, kVT, 0, st>>>(ps, hp, P, qs, hq, Q, d, eps, s, v, A, G); break;
        case 32: k_plan_pass<32><<<grid, kVT, 0, st>>>(ps, hp, P, qs, hq, Q, d, eps, s, v, A, G); break;
        case 64: k_plan_pass<64><<<grid, kVT, 0, st>>>(ps, hp, P, qs, hq, Q, d, eps, s, v, A, G); break;
        case 256: {
            const size_t smem = sizeof(float) * ((size_t)(kVWP + kVWQ) * (d + 1) + 1) +
                                sizeof(double) * ((size_t)kVWP * kVWQ + kVWQ) + sizeof(float) * kVWQ + 16;
            cudaError_t e = cudaFuncSetAttribute(k_plan_pass_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return e;
            k_plan_pass_wide<<<(P + kVWP - 1) / kVWP, kVWT, smem, st>>>(ps, hp, P, qs, hq, Q, d, eps, s, v, A, G);
            break;
        }
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

// ---------------------------------------------------------------- PCG (single CTA, fp64)
// Workspace layout (doubles), N = n + m:  r_c = [r | c] (diag of M), w, res, zp, pp, Ap, z,
// and scalars sc[8]: 0 rz, 1 pAp, 2 alpha, 3 beta, 4 |res|^2, 5 |z|^2.
__device__ __forceinline__ double cta_sum(double v, double *red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    for (int i = 0; i < kVecT / 32; ++i) t += red[i];
    return t;
}

// start: z' = z - (z.e / e.e) e (e = (1_n, -1_m)); w = 0; res = z'; zp = res / D; pp = zp; rz = res.zp
__global__ void __launch_bounds__(kVecT) k_cg_start(int n, int m, const float *zf, const float *zg, const double *dg,
                                                    double *w, double *res, double *zp, double *pp, double *z,
                                                    double *sc) {
    __shared__ double red[kVecT / 32];
    const int N = n + m;
    double ze = 0.0;
    for (int i = threadIdx.x; i < N; i += kVecT) ze += i < n ? (double)zf[i] : -(double)zg[i - n];
    ze = cta_sum(ze, red) / N;
    double rz = 0.0, zz = 0.0;
    for (int i = threadIdx.x; i < N; i += kVecT) {
        const double zi = i < n ? (double)zf[i] - ze : (double)zg[i - n] + ze;
        z[i] = zi;
        w[i] = 0.0;
        res[i] = zi;
        const double q = zi / dg[i];
        zp[i] = q;
        pp[i] = q;
        rz += zi * q;
        zz += zi * zi;
    }
    rz = cta_sum(rz, red);
    zz = cta_sum(zz, red);
    if (threadIdx.x == 0) { sc[0] = rz; sc[4] = zz; sc[5] = zz; }
}

// Ap = M pp from the two plan products: Ap_f = r pp_f + (P pp_g), Ap_g = (P^T pp_f) + c pp_g
// (prod holds [P pp_g | P^T pp_f]); then alpha = rz / pp.Ap, w += alpha pp, res -= alpha Ap,
// zp = res / D, rz' = res.zp, beta = rz'/rz, pp = zp + beta pp.
__global__ void __launch_bounds__(kVecT) k_cg_step(int n, int m, const double *dg, const double *prod, double *w,
                                                   double *res, double *zp, double *pp, double *Ap, double *sc) {
    __shared__ double red[kVecT / 32];
    const int N = n + m;
    double pap = 0.0;
    for (int i = threadIdx.x; i < N; i += kVecT) {
        const double a = dg[i] * pp[i] + prod[i];
        Ap[i] = a;
        pap += pp[i] * a;
    }
    pap = cta_sum(pap, red);
    const double rz = sc[0];
    const double alpha = pap > 0.0 ? rz / pap : 0.0;
    double rzn = 0.0, rr = 0.0;
    for (int i = threadIdx.x; i < N; i += kVecT) {
        w[i] += alpha * pp[i];
        const double ri = res[i] - alpha * Ap[i];
        res[i] = ri;
        const double q = ri / dg[i];
        zp[i] = q;
        rzn += ri * q;
        rr += ri * ri;
    }
    rzn = cta_sum(rzn, red);
    rr = cta_sum(rr, red);
    const double beta = rz > 0.0 ? rzn / rz : 0.0;
    for (int i = threadIdx.x; i < N; i += kVecT) pp[i] = zp[i] + beta * pp[i];
    if (threadIdx.x == 0) { sc[0] = rzn; sc[1] = pap; sc[2] = alpha; sc[3] = beta; sc[4] = rr; }
}

// min-norm w: remove the e component; grad_a = eps w_f, grad_b = eps w_g
__global__ void __launch_bounds__(kVecT) k_cg_finish(int n, int m, float eps, double *w, float *ga, float *gb) {
    __shared__ double red[kVecT / 32];
    const int N = n + m;
    double we = 0.0;
    for (int i = threadIdx.x; i < N; i += kVecT) we += i < n ? w[i] : -w[i];
    we = cta_sum(we, red) / N;
    __syncthreads();
    for (int i = threadIdx.x; i < N; i += kVecT) {
        const double v = i < n ? w[i] - we : w[i] + we;
        w[i] = v;
        if (i < n) { if (ga) ga[i] = (float)(eps * v); }
        else if (gb) gb[i - n] = (float)(eps * v);
    }
}

__global__ void k_scale_out(const double *G, long long cnt, double s, float *out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < cnt; i += (long long)gridDim.x * blockDim.x)
        out[i] = (float)(s * G[i]);
}

size_t vjp_work_doubles(long long n, long long m, int d) { return 8 * (size_t)(n + m) + 16 + (size_t)(n + m) * d; }

// The whole VJP: r, c, PCG to |res| <= tol |z'| (checked every 8 iterations; at most max_iter),
// then the gradients.  work: vjp_work_doubles(n, m, d).  Returns the iterations in *iters and the
// final relative residual in *relres (host).
cudaError_t launch_vjp(long long n, long long m, int d, const float *x, const float *y, float eps, const float *f,
                       const float *g, const float *zf, const float *zg, double tol, int max_iter, double *work,
                       float *gx, float *gy, float *ga, float *gb, int *iters, double *relres, cudaStream_t st) {
    if (dm_of(d) == 0) return cudaErrorInvalidValue;
    const long long N = n + m;
    double *dg = work, *w = dg + N, *res = w + N, *zp = res + N, *pp = zp + N, *Ap = pp + N, *z = Ap + N,
           *prod = z + N, *sc = prod + N, *G = sc + 16;
    cudaError_t e;
    // diag(M): r = P 1 (rows), c = P^T 1 (columns)
    if ((e = launch_plan_pass(x, f, (int)n, y, g, (int)m, d, eps, nullptr, nullptr, dg, nullptr, st))) return e;
    if ((e = launch_plan_pass(y, g, (int)m, x, f, (int)n, d, eps, nullptr, nullptr, dg + n, nullptr, st))) return e;
    k_cg_start<<<1, kVecT, 0, st>>>((int)n, (int)m, zf, zg, dg, w, res, zp, pp, z, sc);
    int it = 0;
    double hsc[8] = {0};
    for (; it < max_iter;) {
        for (int k = 0; k < 8 && it < max_iter; ++k, ++it) {
            // prod = [P pp_g | P^T pp_f]
            if ((e = launch_plan_pass(x, f, (int)n, y, g, (int)m, d, eps, nullptr, pp + n, prod, nullptr, st))) return e;
            if ((e = launch_plan_pass(y, g, (int)m, x, f, (int)n, d, eps, nullptr, pp, prod + n, nullptr, st))) return e;
            k_cg_step<<<1, kVecT, 0, st>>>((int)n, (int)m, dg, prod, w, res, zp, pp, Ap, sc);
        }
        if ((e = cudaMemcpyAsync(hsc, sc, sizeof(hsc), cudaMemcpyDeviceToHost, st))) return e;
        if ((e = cudaStreamSynchronize(st))) return e;
        if (!(hsc[5] > 0.0) || std::sqrt(hsc[4]) <= tol * std::sqrt(hsc[5])) break;
    }
    if ((e = cudaMemcpyAsync(hsc, sc, sizeof(hsc), cudaMemcpyDeviceToHost, st))) return e;
    if ((e = cudaStreamSynchronize(st))) return e;
    *iters = it;
    *relres = hsc[5] > 0.0 ? std::sqrt(hsc[4] / hsc[5]) : 0.0;
    k_cg_finish<<<1, kVecT, 0, st>>>((int)n, (int)m, eps, w, ga, gb);
    // gradients: grad_x_i = 2 sum_j P_ij (w_f,i + w_g,j)(x_i - y_j), grad_y_j likewise
    if (gx) {
        if ((e = launch_plan_pass(x, f, (int)n, y, g, (int)m, d, eps, w, w + n, nullptr, G, st))) return e;
        k_scale_out<<<296, 256, 0, st>>>(G, n * d, 2.0, gx);
    }
    if (gy) {
        if ((e = launch_plan_pass(y, g, (int)m, x, f, (int)n, d, eps, w + n, w, nullptr, G, st))) return e;
        k_scale_out<<<296, 256, 0, st>>>(G, m * d, 2.0, gy);
    }
    return cudaGetLastError();
}

}  // namespace sk
