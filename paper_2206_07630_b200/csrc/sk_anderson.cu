// sk_anderson.cu — K19: Anderson acceleration ("Anderson
// acceleration (And = 5)"; R-27) on the multi-kernel solver (K2 / K3 / K4 passes).
// Sweep l evaluates g~ = g_sk(f^l) (column pass + merge) and T(f^l) = f_sk(g~) (row pass +
// merge, which also sums this slice's err_l term sum_i a_i |expm1((f^l_i - T(f^l)_i)/eps)|
// into vec[8]); then per slice (row shard):
//   k_and_dots  : r = T(f^l) - f^l into the ring slot `head` with T(f^l), and per-block fp64
//                 partials of <r, R_u> for the filled slots (fixed grid: deterministic);
//   k_and_rowsum: one warp: the slice's dots summed over the blocks in order -> vec[0..8);
// (sharded: ncclAllReduce(sum) of vec over the ranks), then once:
//   k_and_decide: one warp: vec summed over the slices in order -> err_l and the stop decision
//                 (checked at (l + 1) % k == 0 and l + 1 = max_iter); unless stopped, the Gram
//                 row/column of the slot, alpha from (G + lam I) x = 1 (lam = 1e-8 tr G / count,
//                 1 if tr G = 0), alpha = x / sum x (Gauss-Jordan, lane r holds row r), the ring
//                 advances and the sweep counter moves to l + 1;
// and per slice:
//   k_and_mix   : f^{l+1} = sum_u alpha_u T(f_u) over the filled slots, written over T(f^l) in
//                 the potential buffer with its packed w (and the K3 image's w columns).
// Every kernel returns at once when the stop flag is set.  State lives on the device (no host
// round trip per sweep).
#include "sk_internal.h"
#include "sk_common.cuh"

namespace sk {

constexpr int kAT = 256;
constexpr int kAndBlocks = 296;
constexpr int kAndM = 8;   // largest memory

struct AndState {
    int head, cnt;
    double G[kAndM * kAndM];
    double alpha[kAndM];
};

size_t anderson_state_bytes() { return sizeof(AndState); }
size_t anderson_blk_doubles() { return (size_t)kAndBlocks * kAndM; }
size_t anderson_vec_doubles() { return 16; }

// F, R: [mem][n] fp32 ring; blk: [kAndBlocks][kAndM]
__global__ void __launch_bounds__(kAT) k_and_dots(Side X, const DevStatus *st, const AndState *as, int mem,
                                                   float *F, float *R, double *blk) {
    __shared__ double red[kAT / 32][kAndM];
    if (*(volatile const int *)&st->stop) return;
    const int l = st->iter;   // (the decision has not advanced it yet)
    const float *f = (l & 1) ? X.pot[1] : X.pot[0];   // f^l    = pot[l & 1]
    const float *T = (l & 1) ? X.pot[0] : X.pot[1];   // T(f^l) = pot[(l + 1) & 1]
    const int head = as->head, cn = as->cnt < mem ? as->cnt + 1 : mem;
    const long long n = X.P;
    double acc[kAndM];
#pragma unroll
    for (int u = 0; u < kAndM; ++u) acc[u] = 0.0;
    for (long long i = blockIdx.x * (long long)kAT + threadIdx.x; i < n; i += (long long)gridDim.x * kAT) {
        const float t = T[i], r = t - f[i];
        F[(long long)head * n + i] = t;
#pragma unroll
        for (int u = 0; u < kAndM; ++u)
            if (u < cn) acc[u] = fma((double)r, (double)(u == head ? r : R[(long long)u * n + i]), acc[u]);
        R[(long long)head * n + i] = r;
    }
    const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
#pragma unroll
    for (int u = 0; u < kAndM; ++u) {
        double v = acc[u];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (ln == 0) red[w][u] = v;
    }
    __syncthreads();
    if (threadIdx.x < kAndM) {
        double v = 0.0;
        for (int k = 0; k < kAT / 32; ++k) v += red[k][threadIdx.x];
        blk[(long long)blockIdx.x * kAndM + threadIdx.x] = v;
    }
}

__global__ void __launch_bounds__(32) k_and_rowsum(const DevStatus *st, const double *blk, int nblk, double *vec) {
    if (*(volatile const int *)&st->stop) return;
    const int lane = threadIdx.x;
    if (lane < kAndM) {
        double v = 0.0;
        for (int b = 0; b < nblk; ++b) v += blk[(long long)b * kAndM + lane];
        vec[lane] = v;
    }
}

__global__ void __launch_bounds__(32) k_and_decide(DevStatus *st, AndState *as, int mem, const double *vec, int ns) {
    if (*(volatile const int *)&st->stop) return;
    const int lane = threadIdx.x, head = as->head, cn = as->cnt < mem ? as->cnt + 1 : mem;
    double dl = 0.0, et = 0.0;   // <r_new, r_lane> and err_l, summed over the slices in order
    for (int i = 0; i < ns; ++i) {
        if (lane < kAndM) dl += vec[i * 16 + lane];
        et += vec[i * 16 + kAndM];
    }
    if (lane >= cn) dl = 0.0;
    // the stop decision (every lane computes it; lane 0 writes)
    const int l = st->iter, l1 = l + 1;
    if (!isfinite(et)) {
        // T(f^l) became non-finite on some slice (rank): (f^l, g~ = g_sk(f^l)) is the last finite
        // pair (a sharded row merge does not stop on its own slice's non-finite rows)
        if (lane == 0) { st->err = (float)et; st->nonfinite = 1; st->final_iter = l; __threadfence(); st->stop = 1; }
        return;
    }
    bool stop = false;
    if (l1 % st->check_every == 0 || l1 >= st->max_iter) {
        if (lane == 0) st->err = (float)et;
        if ((float)et < st->tol) {
            stop = true;
            if (lane == 0) st->converged = 1;
        }
    }
    if (l1 >= st->max_iter) stop = true;
    if (stop) {
        if (lane == 0) { st->final_iter = l; __threadfence(); st->stop = 1; }
        return;
    }
    double row[kAndM];
#pragma unroll
    for (int u = 0; u < kAndM; ++u) {
        const double du = __shfl_sync(0xffffffffu, dl, u);   // <r_new, r_u>
        double gv;
        if (lane == head) gv = du;
        else if (u == head) gv = dl;
        else gv = lane < kAndM ? as->G[lane * kAndM + u] : 0.0;
        row[u] = (lane < cn && u < cn) ? gv : (u == lane ? 1.0 : 0.0);
    }
    __syncwarp();
    if (lane < cn) {   // the Gram row/column of the new slot, for later sweeps
        as->G[head * kAndM + lane] = dl;
        as->G[lane * kAndM + head] = dl;
    }
    double diag = 0.0;
#pragma unroll
    for (int u = 0; u < kAndM; ++u)
        if (u == lane) diag = row[u];
    double tr = lane < cn ? diag : 0.0;
    for (int o = 16; o > 0; o >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, o);
    const double lam = tr > 0.0 ? 1e-8 * tr / cn : 1.0;
#pragma unroll
    for (int u = 0; u < kAndM; ++u)
        if (u == lane && lane < cn) row[u] += lam;
    double rhs = lane < cn ? 1.0 : 0.0;
    for (int c = 0; c < cn; ++c) {   // Gauss-Jordan, pivots in order
        double piv[kAndM], myc = 0.0;
#pragma unroll
        for (int u = 0; u < kAndM; ++u) {
            piv[u] = __shfl_sync(0xffffffffu, row[u], c);
            if (u == c) myc = row[u];
        }
        const double prhs = __shfl_sync(0xffffffffu, rhs, c);
        const double pcc = __shfl_sync(0xffffffffu, myc, c);
        if (lane != c) {
            const double q = myc / pcc;
#pragma unroll
            for (int u = 0; u < kAndM; ++u) row[u] = fma(-q, piv[u], row[u]);
            rhs = fma(-q, prhs, rhs);
        }
    }
#pragma unroll
    for (int u = 0; u < kAndM; ++u)
        if (u == lane) diag = row[u];
    const double xl = lane < cn ? rhs / diag : 0.0;
    double sx = xl;
    for (int o = 16; o > 0; o >>= 1) sx += __shfl_xor_sync(0xffffffffu, sx, o);
    // degenerate least squares (R-30): a non-finite or zero sum x, or a non-finite alpha, falls
    // back to the plain update f^{l+1} = T(f^l) for this sweep (the history is kept)
    double al = xl / sx;
    const bool degen = !isfinite(sx) || sx == 0.0 || __any_sync(0xffffffffu, lane < cn && !isfinite(al));
    if (degen) al = lane == head ? 1.0 : 0.0;
    if (lane < kAndM) as->alpha[lane] = lane < cn ? al : 0.0;
    if (lane == 0) {
        as->head = (head + 1) % mem;
        as->cnt = cn;
        st->iter = l1;
    }
}

__global__ void __launch_bounds__(kAT) k_and_mix(Side X, const DevStatus *st, const AndState *as, const float *F,
                                                  float eps) {
    if (*(volatile const int *)&st->stop) return;
    const int l1 = st->iter;
    float *fn = (l1 & 1) ? X.pot[1] : X.pot[0];   // the slot holding T(f^l) -> f^{l+1}
    const int cn = as->cnt;   // (advanced by k_and_decide)
    double al[kAndM];
#pragma unroll
    for (int u = 0; u < kAndM; ++u) al[u] = as->alpha[u];
    const float kap = kLog2e / eps;
    const long long n = X.P;
    for (long long i = blockIdx.x * (long long)kAT + threadIdx.x; i < n; i += (long long)gridDim.x * kAT) {
        double v = 0.0;
#pragma unroll
        for (int u = 0; u < kAndM; ++u)
            if (u < cn) v = fma(al[u], (double)F[(long long)u * n + i], v);
        const float h = (float)v;
        fn[i] = h;
        const float wn = fmaf(h, kap, -X.nk[i]);
        const long long t = i / X.tq, o = i % X.tq;
        X.pack[t * (long long)(X.D + 1) * X.tq + (long long)X.D * X.tq + o] = wn;
        if (X.tcimg) tc_put_w(X.tcimg, X.P, i, wn, X.tc_c, X.tc_rb);
    }
}

cudaError_t launch_anderson_dots(const Side &X, const DevStatus *st, const void *state, int mem, float *F,
                                 float *R, double *blk, double *vec, cudaStream_t s) {
    if (mem < 2 || mem > kAndM) return cudaErrorInvalidValue;
    k_and_dots<<<kAndBlocks, kAT, 0, s>>>(X, st, (const AndState *)state, mem, F, R, blk);
    k_and_rowsum<<<1, 32, 0, s>>>(st, blk, kAndBlocks, vec);
    return cudaGetLastError();
}

cudaError_t launch_anderson_decide(DevStatus *st, void *state, int mem, const double *vec, int ns, cudaStream_t s) {
    k_and_decide<<<1, 32, 0, s>>>(st, (AndState *)state, mem, vec, ns);
    return cudaGetLastError();
}

cudaError_t launch_anderson_mix(const Side &X, const DevStatus *st, const void *state, const float *F, float eps,
                                cudaStream_t s) {
    k_and_mix<<<kAndBlocks, kAT, 0, s>>>(X, st, (const AndState *)state, F, eps);
    return cudaGetLastError();
}

}  // namespace sk
