// sk_api.cu — the C ABI (include/sinkhorn_b200.h): context, argument checks,
// host/device staging, dispatch to the kernels and the device-driven solve loop.
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/sinkhorn_b200.h"
#include "sk_internal.h"

using namespace sk;

// ----------------------------------------------------------------- NCCL (dlopen)
namespace {
typedef struct { char internal[128]; } nccl_id_t;
typedef void *nccl_comm_t;
typedef int (*fn_get_id)(nccl_id_t *);
typedef int (*fn_init_rank)(nccl_comm_t *, int, nccl_id_t, int);
typedef int (*fn_allgather)(const void *, void *, size_t, int, nccl_comm_t, cudaStream_t);
typedef int (*fn_allreduce)(const void *, void *, size_t, int, int, nccl_comm_t, cudaStream_t);
typedef int (*fn_destroy)(nccl_comm_t);
typedef const char *(*fn_errstr)(int);
constexpr int kNcclFloat32 = 7, kNcclFloat64 = 8, kNcclSum = 0, kNcclMax = 2;

struct Nccl {
    void *h = nullptr;
    fn_get_id get_id = nullptr;
    fn_init_rank init_rank = nullptr;
    fn_allgather allgather = nullptr;
    fn_allreduce allreduce = nullptr;
    fn_destroy destroy = nullptr;
    fn_errstr errstr = nullptr;
    bool load() {
        if (h) return true;
        const char *names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char *nm : names) {
            h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
            if (h) break;
        }
        if (!h) return false;
        get_id = (fn_get_id)dlsym(h, "ncclGetUniqueId");
        init_rank = (fn_init_rank)dlsym(h, "ncclCommInitRank");
        allgather = (fn_allgather)dlsym(h, "ncclAllGather");
        allreduce = (fn_allreduce)dlsym(h, "ncclAllReduce");
        destroy = (fn_destroy)dlsym(h, "ncclCommDestroy");
        errstr = (fn_errstr)dlsym(h, "ncclGetErrorString");
        return get_id && init_rank && allgather && allreduce && destroy;
    }
};
Nccl g_nccl;

struct Buf {
    void *p = nullptr;
    size_t cap = 0;
};
}  // namespace

struct sk_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::string err;
    std::vector<Buf> bufs;
    int timing = 0;
    sk_counters cnt{};
    nccl_comm_t comm = nullptr;
    int rank = 0, world = 1;
    int *h_flag = nullptr;  // pinned host scratch
    DevStatus *h_status = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    std::vector<cudaEvent_t> tev;   // per-launch timing events of the dominant kernel (pool)
    float omega = 1.f;              // Alg. 1's relaxation for the following solves
    float decay_init = 0.f, decay_rate = 1.f;   // eps-decay for the following solves (R-25)
    int anderson = 0;               // Anderson memory for the following solves (R-27; 0: off)
    int adapt = 0;                  // adaptive momentum window (R-31; 0: off)
    int force_nccl = 0;             // sk_set_force_nccl: a 1-rank communicator takes the NCCL path
    // diagnostics / tuning (sk_set_tuning): kernel variants and balances measured in DESIGN.md
    struct Tuning {
        int tc = 1;             // tensor-core cross term for d in [tc_min_d, 64] (0: FFMA kernel K2)
        int tc_min_d = 17;      // the smallest d on the tensor-core kernel K3 (BJ.ns: FFMA below) ...
        int tc_small_d = 1;     // ... except for large problems (max(n, m) > 16384): K3 at every d
        int fused = 1;          // stored mode: the fused single-read sweep K5
        int seeded = 1;         // max-free (seeded) passes (from sweep seed_from on)
        int seed_from = 1;      // the first seeded sweep (0-based, >= 1: sweep 0 has no previous LSEs)
        float tc_margin = 4.f;  // K3 seeded shift above the previous LSE (log2 units)
        float lse_margin = 4.f; // K2 seeded shift above the previous LSE (log2 units)
        int lse_emu8 = 1;       // K2 seeded D <= 4: exponential pairs of 8 on the FMA pipe
        int tc_emu = 2;         // K3: exponential pairs of 8 on the FMA pipe
        int tc_epi = 16;        // K3 epilogue organisation (16 or 162)
        int tc_pipe = 0;        // K3 seeded epilogue with software-pipelined TMEM loads
        int batched_shape = 1;  // K13: 512 x 2 points for 512 < P <= 1024 (0: 1024 x 1)
        int batched_cl = 0;     // K13: 0 auto, 1 one CTA, 2 a CTA pair per problem
        int batched_park = 12;  // K13 batches: sweeps per turn of the park / resume scheduler (0: off)
        int grid_solver = 1;    // the subsample initializer's inner solve on K20 (0: solve_impl)
    } tune;
};

namespace {
enum BufId {
    B_STAGE0 = 0, B_STAGE_END = 16,   // staging of host arrays
    B_FLAG = 16, B_XPACK, B_XC, B_XNK, B_XPOT, B_YPACK, B_YC, B_YNK, B_YPOT, B_PART, B_BLKE, B_BLKB,
    B_STATUS, B_COST, B_REP, B_SORT, B_PERM, B_YSORT, B_GAUSS, B_GAUSS2, B_GMM, B_EMWIDE, B_SORTKEYS, B_DUALSCR, B_SUBW, B_SUBZ,
    B_SUBF, B_SUBG, B_IDX, B_OUT, B_FA, B_QUEUE, B_XIMG, B_YIMG, B_XLSE, B_YLSE, B_TCMAX, B_EMST, B_EMPART, B_EMIDX, B_VJP, B_ANDFR, B_ANDBLK, B_ANDVEC, B_ANDST, B_XCHG, B_PARK, B_XCNT, B_XROW, B_XCNT2, B_GRID, B_NBUF
};

sk_status fail(sk_ctx *c, sk_status s, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) c->err = buf;
    return s;
}

#define CU(call)                                                                                  \
    do {                                                                                          \
        cudaError_t _e = (call);                                                                  \
        if (_e != cudaSuccess)                                                                    \
            return fail(ctx, _e == cudaErrorMemoryAllocation ? SK_ENOMEM : SK_ECUDA, "%s: %s (%s:%d)", \
                        #call, cudaGetErrorString(_e), __FILE__, __LINE__);                       \
    } while (0)

#define CK(call)                              \
    do {                                      \
        sk_status _s = (call);                \
        if (_s != SK_OK) return _s;           \
    } while (0)

void *ensure(sk_ctx *ctx, int id, size_t bytes, cudaError_t *e) {
    Buf &b = ctx->bufs[id];
    *e = cudaSuccess;
    if (bytes == 0) bytes = 16;
    if (b.cap >= bytes) return b.p;
    if (b.p) {
        cudaStreamSynchronize(ctx->stream);
        cudaFree(b.p);
        b.p = nullptr;
        b.cap = 0;
    }
    size_t cap = std::max(bytes, (size_t)256);
    *e = cudaMalloc(&b.p, cap);
    if (*e != cudaSuccess) { cudaGetLastError(); b.p = nullptr; return nullptr; }
    b.cap = cap;
    return b.p;
}

#define ENSURE(ptr, type, id, count)                                                              \
    type *ptr = nullptr;                                                                          \
    do {                                                                                          \
        cudaError_t _e;                                                                           \
        ptr = (type *)ensure(ctx, id, sizeof(type) * (size_t)(count), &_e);                       \
        if (!ptr) return fail(ctx, SK_ENOMEM, "workspace allocation of %zu bytes failed: %s",     \
                              sizeof(type) * (size_t)(count), cudaGetErrorString(_e));             \
    } while (0)

bool is_device_ptr(const void *p) {
    if (!p) return true;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// Staging of caller arrays that may live in host memory.
struct Stager {
    sk_ctx *ctx;
    int next = B_STAGE0;
    struct Out { void *host; void *dev; size_t bytes; };
    std::vector<Out> outs;
    explicit Stager(sk_ctx *c) : ctx(c) {}
    sk_status in(const void *p, size_t bytes, const void **dev) {
        if (!p || is_device_ptr(p)) { *dev = p; return SK_OK; }
        if (next >= B_STAGE_END) return fail(ctx, SK_EINVAL, "too many host arrays");
        cudaError_t e;
        void *d = ensure(ctx, next++, bytes, &e);
        if (!d) return fail(ctx, SK_ENOMEM, "staging allocation failed");
        CU(cudaMemcpyAsync(d, p, bytes, cudaMemcpyHostToDevice, ctx->stream));
        *dev = d;
        return SK_OK;
    }
    template <class T> sk_status in_t(const T *p, size_t count, const T **dev) {
        const void *d;
        sk_status s = in(p, count * sizeof(T), &d);
        *dev = (const T *)d;
        return s;
    }
    template <class T> sk_status out_t(T *p, size_t count, T **dev) {
        if (!p || is_device_ptr(p)) { *dev = p; return SK_OK; }
        if (next >= B_STAGE_END) return fail(ctx, SK_EINVAL, "too many host arrays");
        cudaError_t e;
        void *d = ensure(ctx, next++, count * sizeof(T), &e);
        if (!d) return fail(ctx, SK_ENOMEM, "staging allocation failed");
        outs.push_back({p, d, count * sizeof(T)});
        *dev = (T *)d;
        return SK_OK;
    }
    sk_status flush() {
        for (auto &o : outs) CU(cudaMemcpyAsync(o.host, o.dev, o.bytes, cudaMemcpyDeviceToHost, ctx->stream));
        outs.clear();
        return SK_OK;
    }
};

// Device-side validation of arrays; one D2H read of a flag.
sk_status check_arrays(sk_ctx *ctx, std::initializer_list<std::pair<const float *, long long>> finite,
                       std::initializer_list<std::pair<const float *, long long>> positive,
                       const char *what) {
    ENSURE(flag, int, B_FLAG, 4);
    CU(cudaMemsetAsync(flag, 0, sizeof(int), ctx->stream));
    CheckList L{};
    auto flush = [&]() -> sk_status {
        if (L.cnt) { CU(launch_check_multi(L, flag, ctx->stream)); ctx->cnt.kernel_launches++; }
        L = CheckList{};
        return SK_OK;
    };
    auto add = [&](const float *p, long long n, int pos) -> sk_status {
        if (!p || n <= 0) return SK_OK;
        if (L.cnt == 8) CK(flush());
        L.p[L.cnt] = p; L.n[L.cnt] = n; L.positive[L.cnt] = pos; ++L.cnt;
        L.total += n;
        return SK_OK;
    };
    for (auto &p : finite) CK(add(p.first, p.second, 0));
    for (auto &p : positive) CK(add(p.first, p.second, 1));
    CK(flush());
    CU(cudaMemcpyAsync(ctx->h_flag, flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    if (*ctx->h_flag) return fail(ctx, SK_EINVAL, "%s: non-finite input or non-positive weight", what);
    return SK_OK;
}

bool bad_scalar(float v) { return !std::isfinite(v); }

// Occupancy-aware split count: smallest waste of the last wave, at least ~2 waves.
int choose_split(long long ptiles, long long qtiles_per_unit, int occ, int max_split) {
    const long long slots = 148LL * std::max(occ, 1);
    int best = 1;
    double best_cost = 1e30;
    for (int s = 1; s <= max_split && s <= std::max<long long>(1, qtiles_per_unit); ++s) {
        const long long ctas = ptiles * s;
        const double waves = (double)ctas / slots;
        const double cost = std::ceil(waves) / waves * (1.0 + 0.002 * s) + (waves < 1.0 ? 1.0 / waves : 0.0);
        if (cost < best_cost - 1e-9) { best_cost = cost; best = s; }
    }
    return best;
}

long long shard_block_rows(long long n) {
    long long per = (n + SK_SHARD_BLOCKS - 1) / SK_SHARD_BLOCKS;
    return (per + 255) / 256 * 256;
}

// ------------------------------------------------------------ the solve core
// One problem: all m columns, and the rows of one or more "rank slices".  The
// real sharded path has one slice per process and an ncclAllGather of the column
// partials; the unsharded path has one slice covering all rows; the emulated
// path (testing) has `world` slices in one process whose column partials land in
// their slots directly.  The partition of rows into SK_SHARD_BLOCKS fixed blocks
// and of each block into split_q sub-splits depends on (n_total, m, d) only, so all
// three produce bit-identical results.
struct Slice {
    long long row0, n;
    const float *x, *a, *f_init;
    float *f;               // device output (n)
    int rank;
};

struct Problem {
    long long n_total, m;
    int d;
    const float *y, *b;
    float eps, tol;
    int max_iter, check_every;
    sk_cost_mode mode;
    float *g;               // device output (m)
    int world;              // ranks of the partition (1 = unsharded)
    bool nccl;              // partials exchanged with ncclAllGather (one local slice; world >= 1)
    bool partitioned = false;  // sharded entries: results must not depend on the world size
    float omega = 1.f;         // Alg. 1's relaxation (sk_set_relaxation)
};

// Per-launch CUDA-event timing of the dominant kernel (only while ctx->timing is set).  Each
// launch is tagged with its sweep and kind so that launches that returned at entry (enqueued
// ahead of the host poll, after the stop flag was set) are excluded once L is known.
struct LaunchTimer {
    enum Kind { COL = 0, ROW = 1, FUSED = 2 };
    struct Rec { int a, b, sweep, kind; double entries, bytes; };
    sk_ctx *ctx;
    bool on;
    std::vector<Rec> recs;
    int next = 0;
    LaunchTimer(sk_ctx *c) : ctx(c), on(c->timing != 0) {}
    int ev() {
        if (next >= (int)ctx->tev.size()) {
            cudaEvent_t e;
            if (cudaEventCreate(&e) != cudaSuccess) { cudaGetLastError(); return -1; }
            ctx->tev.push_back(e);
        }
        return next++;
    }
    int start() {
        if (!on) return -1;
        const int a = ev();
        if (a >= 0) cudaEventRecord(ctx->tev[a], ctx->stream);
        return a;
    }
    void stop(int a, int sweep, int kind, double entries, double bytes) {
        if (!on || a < 0) return;
        const int b = ev();
        if (b < 0) return;
        cudaEventRecord(ctx->tev[b], ctx->stream);
        recs.push_back({a, b, sweep, kind, entries, bytes});
    }
    // after the stream has been synchronised; L = sweeps of the solve
    void collect(int L) {
        for (const Rec &r : recs) {
            const bool ran = r.kind == COL ? r.sweep <= L : r.sweep < L;
            if (!ran) continue;
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, ctx->tev[r.a], ctx->tev[r.b]) != cudaSuccess) { cudaGetLastError(); continue; }
            ctx->cnt.dom_launches++;
            ctx->cnt.dom_ms += ms;
            ctx->cnt.dom_entries += r.entries;
            ctx->cnt.dom_bytes += r.bytes;
        }
        recs.clear();
        next = 0;
    }
};

sk_status solve_core(sk_ctx *ctx, const Problem &P, std::vector<Slice> &slices, sk_report *rep) {
    cudaStream_t st = ctx->stream;
    LaunchTimer tm(ctx);
    // sharded: the rank partition of the rows (SK_SHARD_BLOCKS / world blocks per rank); a 1-rank
    // communicator (sk_set_force_nccl) takes the same path with its 8 blocks
    const bool sharded = P.world > 1 || P.nccl;
    const auto &T = ctx->tune;
    // Anderson (R-27, K19): omega = 1; the stored path runs the separate row/column passes; rows
    // may be sharded (the Gram dots and the error are summed over the slices / ranks)
    const int amem = ctx->anderson >= 2 ? ctx->anderson : 0;
    if (amem && P.omega != 1.f)
        return fail(ctx, SK_EUNSUPPORTED, "Anderson acceleration needs omega = 1");
    // adaptive momentum (R-31): starts plain, the merges read omega from the device status
    const int adapt = ctx->adapt;
    if (adapt && (amem || P.omega != 1.f))
        return fail(ctx, SK_EUNSUPPORTED, "adaptive momentum combines with neither Anderson nor a fixed omega");
    const bool rterms = adapt || P.omega != 1.f;   // relaxed row terms of err and E
    const long long m = P.m, n_glob = P.n_total;
    const int ns = (int)slices.size();
    long long n_max = 0, n_sum = 0;
    for (auto &sl : slices) { n_max = std::max(n_max, sl.n); n_sum += sl.n; }
    const bool stored_ok = P.d >= 1 && (m % 4 == 0);
    bool stored = P.mode == SK_COST_STORED;
    if (P.mode == SK_COST_AUTO) {
        stored = stored_ok && P.d >= 8 && P.d < 32 && 4.0 * n_sum * m <= 8.0e9;
        if (stored) {   // AUTO falls back to the online cost when C does not fit
            const size_t need = sizeof(float) * (size_t)n_sum * m;
            size_t fr = 0, tot = 0;
            if (ctx->bufs[B_COST].cap < need &&
                (cudaMemGetInfo(&fr, &tot) != cudaSuccess || fr + ctx->bufs[B_COST].cap < need + ((size_t)512 << 20)))
                stored = false;
        }
    }
    if (stored && !stored_ok) return fail(ctx, SK_EUNSUPPORTED, "stored-cost mode needs m %% 4 == 0");
    // tensor-core cross term for d in (16, 64] (BJ.ns "only when d >= 32"; d in (16, 32] pads to
    // K = 32); sk_set_tuning("tc", 0) forces the FFMA kernel (comparison knob)
    // large problems run the tensor-core cross term at every d (T.tc_small_d): at small d it is not
    // the cross term's flops that matter but the FMA pipe it occupies next to the FMA-pipe
    // exponentials (C4, d = 3: 1162 -> 1104 ms); small problems keep K2 below tc_min_d
    const bool large_p = std::max(n_glob, m) > 16384;
    bool tc = !stored && P.d <= 256 && T.tc != 0 && (P.d >= T.tc_min_d || (large_p && T.tc_small_d));
    unsigned *amax = nullptr;
    if (tc) {
        // per-side max |coordinate| (global over the ranks) -> the fold scales; a problem whose
        // scaled coordinates would leave the fp16 range runs on the FFMA kernel instead
        cudaError_t e1;
        amax = (unsigned *)ensure(ctx, B_TCMAX, 2 * sizeof(unsigned), &e1);
        if (!amax) return fail(ctx, SK_ENOMEM, "tensor-core scales");
        CU(cudaMemsetAsync(amax, 0, 2 * sizeof(unsigned), st));
        for (auto &sl : slices) CU(launch_absmax(sl.x, sl.n * P.d, amax, st));
        CU(launch_absmax(P.y, m * P.d, amax + 1, st));
        if (P.nccl && sharded) {
            int r = g_nccl.allreduce(amax, amax, 1, kNcclFloat32, kNcclMax, ctx->comm, st);
            if (r != 0) return fail(ctx, SK_ENCCL, "ncclAllReduce(max) failed");
        }
        unsigned h[2];
        CU(cudaMemcpyAsync(h, amax, sizeof h, cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        float hx, hy;
        memcpy(&hx, &h[0], 4);
        memcpy(&hy, &h[1], 4);
        tc = tc_fold_ok(hx, hy, P.eps);
        ctx->cnt.kernel_launches += ns + 1;
    }
    const int ksteps = (P.d + 15) / 16;
    const int D = (stored || tc) ? 0 : lse_dpad(P.d);
    if (!stored && !tc && D == 0) return fail(ctx, SK_EUNSUPPORTED, "online path supports d <= 256");
    const int tq = stored ? 256 : (tc ? tc_points_per_tile() : lse_tq(D));
    const long long yt = lse_tiles(m, tq);
    const int pmode = stored ? PACK_STORED : (tc ? PACK_TC : PACK_ONLINE);

    // per-slice X sides, carved from one allocation per array
    std::vector<long long> off(ns + 1, 0), offp(ns + 1, 0);
    for (int i = 0; i < ns; ++i) {
        off[i + 1] = off[i] + slices[i].n;
        offp[i + 1] = offp[i] + lse_tiles(slices[i].n, tq) * (D + 1) * tq;
    }
    ENSURE(xpack, float, B_XPACK, offp[ns]);
    ENSURE(xc, float, B_XC, off[ns]);
    ENSURE(xnk, float, B_XNK, off[ns]);
    ENSURE(xpot, float, B_XPOT, 2 * off[ns]);
    ENSURE(ypack, float, B_YPACK, yt * (D + 1) * tq);
    ENSURE(yc, float, B_YC, m);
    ENSURE(ynk, float, B_YNK, m);
    ENSURE(ypot, float, B_YPOT, 2 * m);
    ENSURE(status, DevStatus, B_STATUS, 1);
    char *ximg = nullptr, *yimg = nullptr;
    std::vector<long long> offi(ns + 1, 0);
    // d <= 16 (one K = 16 step): compact SW32 operand images, a quarter of the K = 64 bytes;
    // d > 64: K chunks of 64
    const int tc_rb = tc_row_bytes(P.d);
    if (tc) {
        for (int i = 0; i < ns; ++i) offi[i + 1] = offi[i] + (long long)tc_image_bytes(slices[i].n, tc_rb);
        cudaError_t e1, e2;
        ximg = (char *)ensure(ctx, B_XIMG, (size_t)offi[ns], &e1);
        yimg = (char *)ensure(ctx, B_YIMG, tc_image_bytes(m, tc_rb), &e2);
        if (!ximg || !yimg) return fail(ctx, SK_ENOMEM, "tensor-core operand images");
        for (int i = 0; i < ns; ++i)
            CU(launch_pack_tc(slices[i].x, slices[i].n, P.d, amax, 0, P.eps, ximg + offi[i], st, tc_rb));
        CU(launch_pack_tc(P.y, m, P.d, amax, 1, P.eps, yimg, st, tc_rb));
        ctx->cnt.kernel_launches += ns + 1;
    }
    std::vector<Side> X(ns);
    for (int i = 0; i < ns; ++i) {
        const long long n = slices[i].n;
        X[i] = Side{(int)n, P.d, D, tq, xpack + offp[i], xc + off[i], xnk + off[i],
                    {xpot + 2 * off[i], xpot + 2 * off[i] + n}};
    }
    Side Y{(int)m, P.d, D, tq, ypack, yc, ynk, {ypot, ypot + m}};
    // online paths: per-point LSE seeds for the max-free (seeded) passes from sweep seed_from on
    // stored mode with the fused sweep (one persistent CTA per SM): 8 blocks x split_q = one wave
    const bool fused = stored && T.fused != 0 && stored_fused_supported(m) && P.omega == 1.f && !amem && !adapt;
    const bool seedable = !stored;
    if (tc) {   // the seeded passes' exact fallback reads the caller's coordinates
        for (int i = 0; i < ns; ++i) {
            X[i].raw = slices[i].x; X[i].tcimg = (unsigned char *)ximg + offi[i]; X[i].tc_c = tc_fold_c(); X[i].tc_rb = tc_rb;
        }
        Y.tc_rb = tc_rb;
        Y.raw = P.y;
        Y.tcimg = (unsigned char *)yimg;
        Y.tc_c = tc_fold_c();
    }
    if (seedable || fused) {   // (the fused stored sweep seeds its row shifts the same way)
        ENSURE(xlse, float, B_XLSE, off[ns]);
        ENSURE(ylse, float, B_YLSE, m);
        for (int i = 0; i < ns; ++i) X[i].lse = xlse + off[i];
        Y.lse = ylse;
    }
    // seeded passes from sweep seed_from (the second).  Rows: a point whose seeded sum leaves the safe range is
    // recomputed exactly in the merge (the reduced side, all columns, is on every rank).  Columns:
    // the exact fallback would need every rank's rows, so a failing column makes the merge set
    // st->colfail and the whole column pass is redone exactly (gated on the flag) - the same path
    // for every entry, so the unsharded, emulated and sharded solves are bit-identical.
    const bool col_seed = seedable && T.seeded;
    const bool row_seed = seedable && T.seeded;
    const int seed_from = T.seed_from;   // the first seeded sweep (0-based; its seeds are the previous sweep's LSEs)

    // column-pass partition (a function of n_total, m, d only): SK_SHARD_BLOCKS fixed row
    // blocks, each cut into split_q sub-splits sized for the 8-rank launch; empty blocks
    // write (-inf, 0) partials.
    const long long bs_rows = shard_block_rows(n_glob);
    const int nblk_glob = (int)((n_glob + bs_rows - 1) / bs_rows);
    const int blk_per_rank = sharded ? SK_SHARD_BLOCKS / P.world : nblk_glob;
    // small online problems (d <= 4): one output point per thread, so their few P tiles still fill
    // the SMs (a function of the global sizes: the split structure stays partition-invariant)
    const bool r1 = !stored && !tc && D <= 4 && std::max(n_glob, m) <= 16384;
    const int occ = stored ? 8 : (tc ? 1 : lse_occupancy_ctas(D, r1 ? 1 : 0));
    const int Rr = tc ? 1 : (r1 ? 1 : (D <= 4 ? 4 : (D <= 16 ? 2 : 1)));
    const long long pcta = tc ? tc_points_per_tile() : 128LL * Rr;   // output points per CTA (pair)
    const long long ptiles_col = stored ? (m + 511) / 512 : (m + pcta - 1) / pcta;
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->device);
    const int split_q = fused ? std::max(1, nsm / SK_SHARD_BLOCKS)
                              : choose_split(ptiles_col, stored ? bs_rows / 64 : bs_rows / tq, occ, 64);
    const int nsplit_col = (sharded ? SK_SHARD_BLOCKS : nblk_glob) * split_q;
    int split_row = 1;
    if (!stored) {
        // from n_total, not the local slice: the row-pass split (and so the summation order of
        // every row's LSE) is the same for every partition of the rows; sized for the 8-rank
        // launch (one block of rows per GPU), so that every rank's launch fills the GPU - fewer
        // ranks run the same split structure in more waves
        const long long ptiles_row = (bs_rows + pcta - 1) / pcta;
        split_row = choose_split(ptiles_row, yt, occ, 64);
    }
    const long long part_elems = std::max((long long)nsplit_col * m, (long long)split_row * n_max);
    ENSURE(part, float2, B_PART, part_elems);
    // the column partials are pre-merged per fixed row block (K6a) into the exchange buffer
    // [nblk_x][m] - the allgather payload (8 B per column per block) - and the blocks merged in
    // block order: the same merge tree for every partition of the rows (and a 8-way merge instead
    // of a nblk x split_q one: the stored path's 144-split merge took 31 us per sweep)
    const int nblk_x = sharded ? SK_SHARD_BLOCKS : nblk_glob;
    float2 *xchg = nullptr;
    int *xcnt = nullptr;   // K2: arrival counters of the fused premerge [8 blocks][P tiles]
    {
        ENSURE(xc2, float2, B_XCHG, (long long)nblk_x * m);
        xchg = xc2;
        if (!tc && !stored) {
            ENSURE(xc3, int, B_XCNT, (long long)SK_SHARD_BLOCKS * ptiles_col);
            xcnt = xc3;
            CU(cudaMemsetAsync(xcnt, 0, sizeof(int) * (size_t)SK_SHARD_BLOCKS * ptiles_col, st));
        }
    }
    // K2 row pass: its split_row partials merged per P tile the same way into one (M, S) per row
    // (xrow), which the row merge then reads as a single split
    float2 *xrow = nullptr;
    int *xcnt2 = nullptr;
    if (!stored && !tc) {
        const long long ptiles_rmax = (n_max + pcta - 1) / pcta;
        ENSURE(xr2, float2, B_XROW, n_max);
        ENSURE(xr3, int, B_XCNT2, ptiles_rmax);
        xrow = xr2;
        xcnt2 = xr3;
        CU(cudaMemsetAsync(xcnt2, 0, sizeof(int) * (size_t)ptiles_rmax, st));
    }
    ENSURE(blke, double, B_BLKE, 2 * kMergeMaxBlocks);
    ENSURE(blkb, int, B_BLKB, 2048);

    const float loga_u = (float)(-std::log((double)n_glob)), logb_u = (float)(-std::log((double)m));
    for (int i = 0; i < ns; ++i)
        CU(pack_side(X[i], slices[i].x, slices[i].a, loga_u, slices[i].f_init, P.eps, st, pmode));
    CU(pack_side(Y, P.y, P.b, logb_u, nullptr, P.eps, st, pmode));
    if (tc) {   // extra columns: w from the packed sides, zero shifts
        for (int i = 0; i < ns; ++i) CU(launch_pack_tc_ext(slices[i].n, X[i].pack, X[i].tcimg, st, tc_rb));
        CU(launch_pack_tc_ext(m, Y.pack, Y.tcimg, st, tc_rb));
        ctx->cnt.kernel_launches += ns + 1;
    }
    const float tc_margin = T.tc_margin;
    CU(launch_status_init(status, P.max_iter, P.check_every, P.tol, st, amem ? 1 : 0, adapt ? 1.f : P.omega));
    ctx->cnt.kernel_launches += ns + 2;
    float *andfr = nullptr;     // per slice i: F at 2 mem off[i], R at F + mem n_i
    double *andblk = nullptr, *andvec = nullptr;
    void *andst = nullptr;
    if (amem) {
        ENSURE(afr, float, B_ANDFR, 2 * (size_t)amem * off[ns]);
        ENSURE(ablk, double, B_ANDBLK, anderson_blk_doubles());
        ENSURE(avec, double, B_ANDVEC, anderson_vec_doubles() * ns);
        ENSURE(ast, char, B_ANDST, anderson_state_bytes());
        andfr = afr;
        andblk = ablk;
        andvec = avec;
        andst = ast;
        CU(cudaMemsetAsync(andst, 0, anderson_state_bytes(), st));
        CU(cudaMemsetAsync(andvec, 0, sizeof(double) * anderson_vec_doubles() * ns, st));
    }
    auto andF = [&](int i) { return andfr + 2 * (size_t)amem * off[i]; };
    auto andR = [&](int i) { return andfr + 2 * (size_t)amem * off[i] + (size_t)amem * slices[i].n; };

    std::vector<float *> C(ns, nullptr);
    double build_ms = 0.0;
    if (stored) {
        cudaError_t e;
        float *Call = (float *)ensure(ctx, B_COST, sizeof(float) * (size_t)n_sum * m, &e);
        if (!Call) return fail(ctx, SK_ENOMEM, "stored cost needs %.2f GiB", 4.0 * n_sum * m / (1 << 30));
        CU(cudaEventRecord(ctx->ev0, st));
        for (int i = 0; i < ns; ++i) {
            C[i] = Call + off[i] * m;
            CU(launch_build_cost(slices[i].x, P.y, slices[i].n, m, P.d, C[i], st));
            ctx->cnt.kernel_launches++;
        }
        CU(cudaEventRecord(ctx->ev1, st));
        CU(cudaEventSynchronize(ctx->ev1));
        float ms = 0.f;
        CU(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
        build_ms = ms;
    }

    const long long slot = (long long)blk_per_rank * split_q * m;   // one rank's partial slots
    auto col_part = [&](int i) { return part + (sharded ? (long long)slices[i].rank * slot : 0); };
    MergePass mcol{MERGE_COL, &Y, xchg, nblk_x, P.eps, P.b, status, blke,
                   blkb, nullptr, 0.f, sharded ? 1 : 0, 0};
    mcol.omega = P.omega;
    mcol.adapt = adapt;
    mcol.anderson = amem ? 1 : 0;
    int sweep = 0;   // sweeps enqueued so far (seeded passes from seed_from on)

    // stored mode: one HBM read of C per sweep (fused row + column passes, H4s) when m fits
    bool first = true;

    // column pass of every slice (+ its per-block premerge into the exchange buffer); seeded:
    // max-free (shift = previous LSE + margin); only_if: the gated exact redo (not timed)
    auto col_stage = [&](const int *only_if, bool seeded) -> sk_status {
        const int nb = sharded ? blk_per_rank : nblk_glob;
        for (int i = 0; i < ns; ++i) {
            const double ent = (double)slices[i].n * m;
            const int t0 = (fused || only_if) ? -1 : tm.start();   // fused: the dominant kernel is the sweep
            if (stored) {
                StoredPass scol{C[i], slices[i].n, m, P.eps, X[i].pack, col_part(i), bs_rows, nb, split_q,
                                &status->stop, only_if};
                CU(launch_stored_cols(scol, st));
            } else if (tc) {
                TcPass colp{yimg, ximg + offi[i], (int)m, slices[i].n, ksteps, nb, (int)(bs_rows / tq), split_q,
                            col_part(i), P.eps, &status->stop};
                colp.seeded = seeded;
                colp.only_if = only_if;
                colp.emu = T.tc_emu;
                colp.epi = T.tc_epi;
                colp.pipe = T.tc_pipe;
                colp.rb = tc_rb;
                CU(launch_lse_tc(colp, st));
            } else {
                LsePass colp{&Y, &X[i], nb, (int)(bs_rows / tq), split_q, col_part(i), P.eps, &status->stop};
                colp.seeded = seeded;
                colp.only_if = only_if;
                colp.emu8 = T.lse_emu8;
                colp.margin = T.lse_margin;
                colp.R = r1 ? 1 : 0;
                // the block partials straight into the exchange buffer (fused K6a)
                const long long b0 = sharded ? (long long)slices[i].rank * blk_per_rank : 0;
                colp.xchg = xchg + b0 * m;
                colp.cnt = xcnt + b0 * ptiles_col;
                CU(launch_lse(colp, st));
            }
            if (t0 >= 0) tm.stop(t0, sweep, LaunchTimer::COL, ent, stored ? 4.0 * ent : 0.0);
            if (tc || stored) {   // (K2 merges its blocks itself)
                const long long xoff = sharded ? (long long)slices[i].rank * blk_per_rank * m : 0;
                CU(launch_premerge(col_part(i), nb, split_q, m, xchg + xoff, &status->stop, only_if, st));
            }
        }
        return SK_OK;
    };
    // the fused stored sweep's column partials are scaled sums (merge mode `scaled`); a column
    // outside the safe range sets status->colfail and the column pass is redone exactly
    MergePass mcol_scaled = mcol, mcol_redo = mcol;
    mcol_scaled.scaled = 1;
    mcol_redo.only_if = &status->colfail;
    MergePass mcol_seeded = mcol;   // after a seeded online column pass: out-of-range sums -> redo
    mcol_seeded.range_redo = 1;
    const bool colredo = sharded;   // unsharded: the scaled merge recomputes a failing column itself
    if (!colredo && fused) { mcol_scaled.Cst = C[0]; mcol_scaled.xw = X[0].pack; mcol_scaled.n_rows = slices[0].n; }
    auto exchange_and_merge_col = [&](const MergePass &mp0) -> sk_status {
        if (P.nccl && sharded) {   // this rank's pre-merged block partials
            const size_t cnt = (size_t)blk_per_rank * m * 2;
            const void *src = (const void *)(xchg + (long long)slices[0].rank * blk_per_rank * m);
            int r = g_nccl.allgather(src, (void *)xchg, cnt, kNcclFloat32, ctx->comm, st);
            if (r != 0) return fail(ctx, SK_ENCCL, "ncclAllGather failed: %s", g_nccl.errstr ? g_nccl.errstr(r) : "?");
        }
        MergePass mp = mp0;
        mp.tc_fold = tc && col_seed && sweep + 1 >= seed_from;   // the next column pass is seeded
        mp.tc_margin = tc_margin;
        CU(launch_merge(mp, st));
        return SK_OK;
    };

    CU(cudaEventRecord(ctx->ev0, st));
    int launched = 0, poll = 4;
    const int max_sweeps = P.max_iter + 1;  // + the column pass that measures err_L
    for (int it = 0; it < max_sweeps;) {
        const int chunk = std::min(poll, max_sweeps - it);
        for (int c = 0; c < chunk; ++c, ++it) {
            if (fused) {
                if (first) {  // g^1 from f^0 with a plain column pass
                    CK(col_stage(nullptr, false));
                    CK(exchange_and_merge_col(mcol));
                    launched += ns + 1;
                    first = false;
                }
                for (int i = 0; i < ns; ++i) {
                    FusedLaunch fl{C[i], slices[i].n, m, P.eps, Y.pack, X[i].c, {X[i].pot[0], X[i].pot[1]},
                                   X[i].pack, X[i].lse, col_part(i), bs_rows, sharded ? blk_per_rank : nblk_glob,
                                   split_q, status, sharded ? 1 : 0, i + 1 < ns ? 1 : 0};
                    const int t0 = tm.start();
                    CU(launch_stored_fused(fl, st));   // also advances the sweep counter (row bookkeeping)
                    tm.stop(t0, sweep, LaunchTimer::FUSED, 2.0 * slices[i].n * m, 4.0 * slices[i].n * m);
                    const long long xoff = sharded ? (long long)slices[i].rank * blk_per_rank * m : 0;
                    CU(launch_premerge(col_part(i), sharded ? blk_per_rank : nblk_glob, split_q, m, xchg + xoff,
                                       &status->stop, nullptr, st));
                    launched += 2;
                }
                CK(exchange_and_merge_col(mcol_scaled));
                launched += 1;
                if (colredo) {
                    CK(col_stage(&status->colfail, false));   // no-ops unless colfail
                    CK(exchange_and_merge_col(mcol_redo));
                    launched += 1 + 2 * ns;
                }
                ++sweep;
                continue;
            }
            const bool cseed = col_seed && sweep >= seed_from;
            CK(col_stage(nullptr, cseed));
            CK(exchange_and_merge_col(cseed ? mcol_seeded : mcol));
            launched += (tc || stored ? 2 : 1) * ns + 1;   // (+ the premerge on the tensor-core / stored paths)
            if (cseed) {   // the exact redo when a seeded column sum left the safe range (no-ops otherwise)
                CK(col_stage(&status->colfail, false));
                CK(exchange_and_merge_col(mcol_redo));
                launched += (tc || stored ? 2 : 1) * ns + 1;
            }
            for (int i = 0; i < ns; ++i) {
                const int t0 = tm.start();
                if (stored) {
                    StoredPass srow{C[i], slices[i].n, m, P.eps, Y.pack, part, 0, 1, 1, &status->stop};
                    CU(launch_stored_rows(srow, st));
                } else if (tc) {
                    TcPass rowp{ximg + offi[i], yimg, (int)slices[i].n, m, ksteps, 1, 0, split_row, part,
                                P.eps, &status->stop};
                    rowp.seeded = row_seed && sweep >= seed_from;
                    rowp.emu = T.tc_emu;
                    rowp.epi = T.tc_epi;
                    rowp.pipe = T.tc_pipe;
                    rowp.rb = tc_rb;
                    CU(launch_lse_tc(rowp, st));
                } else {
                    LsePass rowp{&X[i], &Y, 1, 0, split_row, part, P.eps, &status->stop};
                    rowp.seeded = row_seed && sweep >= seed_from;
                    rowp.emu8 = T.lse_emu8;
                    rowp.margin = T.lse_margin;
                    rowp.R = r1 ? 1 : 0;
                    rowp.xchg = xrow;
                    rowp.cnt = xcnt2;
                    CU(launch_lse(rowp, st));
                }
                tm.stop(t0, sweep, LaunchTimer::ROW, (double)slices[i].n * m, stored ? 4.0 * slices[i].n * m : 0.0);
                // only the last slice's merge advances the sweep counter
                MergePass mrow{MERGE_ROW, &X[i], xrow ? xrow : part, (stored || xrow) ? 1 : split_row, P.eps, nullptr,
                               status, blke, blkb, nullptr, 0.f, sharded ? 1 : 0, i + 1 < ns ? 1 : 0};
                if (row_seed) mrow.Q = &Y;
                mrow.omega = P.omega;
                mrow.adapt = adapt;
                mrow.accum = i > 0 ? 1 : 0;
                mrow.wts = slices[i].a;   // (the relaxed row error term weighs rows by a)
                mrow.n_uniform = n_glob;  //  uniform: 1 / n_total (a slice holds part of the rows)
                mrow.tc_fold = tc && row_seed && sweep + 1 >= seed_from;   // the next row pass is seeded
                mrow.tc_margin = tc_margin;
                mrow.anderson = amem ? 1 : 0;
                mrow.and_err = amem ? andvec + anderson_vec_doubles() * i + 8 : nullptr;
                CU(launch_merge(mrow, st));
                launched += 2;
                if (amem) {   // this slice's residual into the ring and its Gram dots
                    CU(launch_anderson_dots(X[i], status, andst, amem, andF(i), andR(i), andblk,
                                            andvec + anderson_vec_doubles() * i, st));
                    launched += 2;
                }
            }
            if (rterms && P.nccl && sharded) {   // relaxed: the row terms of err and E over the ranks
                int r = g_nccl.allreduce(&status->row_err, &status->row_err, 2, kNcclFloat64, kNcclSum, ctx->comm, st);
                if (r != 0) return fail(ctx, SK_ENCCL, "ncclAllReduce(row terms) failed");
            }
            if (amem) {   // the sums over the ranks, the decision, f^{l+1} = sum_u alpha_u T(f_u)
                if (P.nccl && sharded) {
                    int r = g_nccl.allreduce(andvec, andvec, 9, kNcclFloat64, kNcclSum, ctx->comm, st);
                    if (r != 0) return fail(ctx, SK_ENCCL, "ncclAllReduce(Anderson) failed");
                }
                CU(launch_anderson_decide(status, andst, amem, andvec, ns, st));
                for (int i = 0; i < ns; ++i) CU(launch_anderson_mix(X[i], status, andst, andF(i), P.eps, st));
                launched += 1 + ns;
            }
            ++sweep;
        }
        CU(cudaMemcpyAsync(ctx->h_status, status, sizeof(DevStatus), cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        if (ctx->h_status->stop) break;
        poll = std::min(poll * 2, 64);
    }
    CU(cudaEventRecord(ctx->ev1, st));
    // E = <f,a> - eps sum(a) summed per fixed row block (bit-identical for every partition of the
    // rows), plus <g,b> (replicated)
    ENSURE(fa, double, B_FA, SK_SHARD_BLOCKS + 1);
    CU(cudaMemsetAsync(fa, 0, sizeof(double) * (SK_SHARD_BLOCKS + 1), st));
    for (int i = 0; i < ns; ++i) {
        CU(launch_report_blocks(X[i], slices[i].a, P.eps, status, n_glob, slices[i].row0, bs_rows, fa, st));
        launched++;
    }
    CU(launch_report(X[0], Y, slices[0].a, P.b, P.eps, status, 1, n_glob, st));   // <g,b> into status->E
    launched++;
    if (P.nccl && sharded) {  // every rank's blocks: allgather its slots of the 8-block array
        int r = g_nccl.allgather(fa + (long long)slices[0].rank * blk_per_rank, fa, (size_t)blk_per_rank,
                                 kNcclFloat64, ctx->comm, st);
        if (r != 0) return fail(ctx, SK_ENCCL, "ncclAllGather(E) failed");
    }
    std::vector<double> fa_h(SK_SHARD_BLOCKS + 1, 0.0);
    CU(cudaMemcpyAsync(fa_h.data(), fa, sizeof(double) * (SK_SHARD_BLOCKS + 1), cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(ctx->h_status, status, sizeof(DevStatus), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    const double gb_part = ctx->h_status->E;
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    DevStatus hs = *ctx->h_status;
    if (!hs.stop) return fail(ctx, SK_ECUDA, "solver loop ended without a stop flag");
    const int L = hs.final_iter;
    tm.collect(hs.iter);
    double E = 0.0;
    for (int b = 0; b < SK_SHARD_BLOCKS; ++b) E += fa_h[b];
    E += gb_part;
    // relaxed: after the f-update sum_ij P_ij = sum(a) + mass_dev (kept by the last row merge)
    if (rterms) E -= (double)P.eps * hs.mass_dev;
    for (int i = 0; i < ns; ++i)
        CU(cudaMemcpyAsync(slices[i].f, X[i].pot[L & 1], sizeof(float) * slices[i].n, cudaMemcpyDeviceToDevice, st));
    // (Anderson: the pair is (f^L, g_sk(f^L)), g one buffer ahead; L + 1 sweeps were evaluated)
    CU(cudaMemcpyAsync(P.g, Y.pot[(L + hs.g_off) & 1], sizeof(float) * m, cudaMemcpyDeviceToDevice, st));
    ctx->cnt.kernel_launches += launched;
    ctx->cnt.lse_launches += (long long)(ns + 1) * (hs.iter + 1);
    if (ctx->timing) ctx->cnt.lse_ms += ms;
    const double entries = (double)n_sum * m * (amem ? 2.0 * (L + 1) : 2.0 * L + 1.0);
    ctx->cnt.lse_ex2 += entries;
    if (stored) ctx->cnt.lse_bytes += 4.0 * (double)n_sum * m * (fused ? (1.0 + hs.iter) : (2.0 * L + 1.0));
    rep->iterations = L + hs.g_off;   // (Anderson: the sweeps evaluated)
    rep->converged = hs.converged;
    rep->marginal_error = hs.err;
    rep->dual_objective = E;
    rep->build_ms = build_ms;
    rep->solve_ms = ms;
    if (hs.nonfinite) return fail(ctx, SK_ENONFINITE, "potentials became non-finite after sweep %d", L);
    return SK_OK;
}

// eps-decay (R-25) around solve_core for the sharded entries: with omega = 1 a sweep is a map
// f -> f, so the T decay sweeps are one-sweep solves at eps_l chained through each slice's f
// (as the unsharded multi-kernel path does in solve_impl), then the solve at the target eps.
sk_status solve_core_decay(sk_ctx *ctx, const Problem &P, std::vector<Slice> &slices, sk_report *rep) {
    if (ctx->decay_init <= 0.f) return solve_core(ctx, P, slices, rep);
    if (P.omega != 1.f) return fail(ctx, SK_EUNSUPPORTED, "eps-decay with omega != 1 runs on the on-chip solver only");
    if (ctx->anderson >= 2) return fail(ctx, SK_EUNSUPPORTED, "Anderson acceleration does not combine with eps-decay");
    if (ctx->adapt) return fail(ctx, SK_EUNSUPPORTED, "adaptive momentum does not combine with eps-decay");
    int T = 0;
    while (T < P.max_iter && (double)P.eps * ctx->decay_init * std::pow((double)ctx->decay_rate, T) > (double)P.eps) ++T;
    if (P.max_iter - T < 1) return fail(ctx, SK_EINVAL, "max_iter must exceed the %d eps-decay sweeps", T);
    double extra_ms = 0.0;
    for (int t = 0; t < T; ++t) {
        Problem Pt = P;
        Pt.eps = (float)((double)P.eps * ctx->decay_init * std::pow((double)ctx->decay_rate, t));
        Pt.max_iter = 1;
        sk_report r1{};
        CK(solve_core(ctx, Pt, slices, &r1));
        extra_ms += r1.solve_ms;
        for (auto &sl : slices) sl.f_init = sl.f;   // chained through f
    }
    Problem Pf = P;
    Pf.max_iter = P.max_iter - T;
    CK(solve_core(ctx, Pf, slices, rep));
    rep->iterations += T;
    rep->solve_ms += extra_ms;
    return SK_OK;
}

sk_status validate_common(sk_ctx *ctx, long long n, long long m, int d, float eps, float tol,
                          int max_iter, int check_every) {
    if (!ctx) return SK_EINVAL;
    if (n < 1 || m < 1) return fail(ctx, SK_EINVAL, "n and m must be >= 1 (n=%lld m=%lld)", n, m);
    if (n > (1LL << 31) - 1 || m > (1LL << 31) - 1) return fail(ctx, SK_EUNSUPPORTED, "n, m < 2^31");
    if (d < 1 || d > 256) return fail(ctx, SK_EINVAL, "d must be in [1, 256] (d=%d)", d);
    if (!(eps > 0.f) || bad_scalar(eps)) return fail(ctx, SK_EINVAL, "eps must be finite and > 0");
    if (!(tol > 0.f) || bad_scalar(tol)) return fail(ctx, SK_EINVAL, "tol must be finite and > 0");
    if (max_iter < 1) return fail(ctx, SK_EINVAL, "max_iter must be >= 1");
    if (check_every < 1) return fail(ctx, SK_EINVAL, "check_every must be >= 1");
    return SK_OK;
}
}  // namespace

// =============================================================== ABI entries
extern "C" {

int32_t sk_version(void) { return 1; }

const char *sk_status_string(int s) {
    switch (s) {
        case SK_OK: return "SK_OK";
        case SK_EINVAL: return "SK_EINVAL";
        case SK_ECUDA: return "SK_ECUDA";
        case SK_ENONFINITE: return "SK_ENONFINITE";
        case SK_ENCCL: return "SK_ENCCL";
        case SK_ENOMEM: return "SK_ENOMEM";
        case SK_EUNSUPPORTED: return "SK_EUNSUPPORTED";
        default: return "SK_UNKNOWN";
    }
}

sk_status sk_create(sk_ctx **out, int device, void *stream) {
    if (!out) return SK_EINVAL;
    *out = nullptr;
    sk_ctx *ctx = new sk_ctx();
    ctx->bufs.resize(B_NBUF);
    ctx->device = device;
    ctx->stream = (cudaStream_t)stream;
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaMallocHost(&ctx->h_flag, sizeof(int));
    if (e == cudaSuccess) e = cudaMallocHost(&ctx->h_status, sizeof(DevStatus));
    if (e == cudaSuccess) e = cudaEventCreate(&ctx->ev0);
    if (e == cudaSuccess) e = cudaEventCreate(&ctx->ev1);
    if (e != cudaSuccess) {
        cudaGetLastError();
        delete ctx;
        return SK_ECUDA;
    }
    *out = ctx;
    return SK_OK;
}

sk_status sk_set_stream(sk_ctx *ctx, void *stream) {
    if (!ctx) return SK_EINVAL;
    ctx->stream = (cudaStream_t)stream;
    return SK_OK;
}

sk_status sk_set_eps_decay(sk_ctx *ctx, float init, float rate) {
    if (!ctx) return SK_EINVAL;
    if (init <= 1.f) { ctx->decay_init = 0.f; ctx->decay_rate = 1.f; return SK_OK; }   // off
    if (!(rate > 0.f && rate < 1.f) || bad_scalar(init))
        return fail(ctx, SK_EINVAL, "eps-decay needs init > 1 (finite) and rate in (0, 1)");
    ctx->decay_init = init;
    ctx->decay_rate = rate;
    return SK_OK;
}

sk_status sk_set_anderson(sk_ctx *ctx, int32_t mem) {
    if (!ctx) return SK_EINVAL;
    if (mem < 0 || mem > 8) return fail(ctx, SK_EINVAL, "Anderson memory must lie in [0, 8], got %d", (int)mem);
    ctx->anderson = mem >= 2 ? mem : 0;
    return SK_OK;
}

sk_status sk_set_force_nccl(sk_ctx *ctx, int32_t enable) {
    if (!ctx) return SK_EINVAL;
    ctx->force_nccl = enable ? 1 : 0;
    return SK_OK;
}

sk_status sk_get_solver_options(const sk_ctx *ctx, float *omega, float *decay_init, float *decay_rate,
                                int32_t *anderson, int32_t *adapt_iters) {
    if (!ctx) return SK_EINVAL;
    if (omega) *omega = ctx->omega;
    if (decay_init) *decay_init = ctx->decay_init;
    if (decay_rate) *decay_rate = ctx->decay_rate;
    if (anderson) *anderson = ctx->anderson;
    if (adapt_iters) *adapt_iters = ctx->adapt;
    return SK_OK;
}

sk_status sk_set_adaptive_momentum(sk_ctx *ctx, int32_t adapt_iters) {
    if (!ctx) return SK_EINVAL;
    if (adapt_iters < 0 || adapt_iters > 100000)
        return fail(ctx, SK_EINVAL, "adapt_iters must lie in [0, 100000], got %d", (int)adapt_iters);
    ctx->adapt = adapt_iters;
    return SK_OK;
}

sk_status sk_set_tuning(sk_ctx *ctx, const char *key, double value) {
    if (!ctx) return SK_EINVAL;
    if (!key) return fail(ctx, SK_EINVAL, "key is NULL");
    auto &T = ctx->tune;
    const std::string k(key);
    const int iv = (int)value;
    auto need = [&](bool ok) -> sk_status {
        return ok ? SK_OK : fail(ctx, SK_EINVAL, "sk_set_tuning(%s, %g): value out of range", key, value);
    };
    if (k == "tc") { CK(need(iv == 0 || iv == 1)); T.tc = iv; }
    else if (k == "tc_min_d") { CK(need(iv >= 1 && iv <= 65)); T.tc_min_d = iv; }
    else if (k == "tc_small_d") { CK(need(iv == 0 || iv == 1)); T.tc_small_d = iv; }
    else if (k == "fused") { CK(need(iv == 0 || iv == 1)); T.fused = iv; }
    else if (k == "seeded") { CK(need(iv == 0 || iv == 1)); T.seeded = iv; }
    else if (k == "seed_from") { CK(need(iv >= 1 && iv <= 1000)); T.seed_from = iv; }
    else if (k == "tc_margin") { CK(need(value >= 0.0 && value <= 1000.0)); T.tc_margin = (float)value; }
    else if (k == "lse_margin") { CK(need(value >= 0.0 && value <= 1000.0)); T.lse_margin = (float)value; }
    else if (k == "lse_emu8") { CK(need(iv >= 0 && iv <= 2)); T.lse_emu8 = iv; }
    else if (k == "tc_emu") { CK(need(iv >= 0 && iv <= 6)); T.tc_emu = iv; }
    else if (k == "tc_epi") { CK(need(iv == 16 || iv == 162)); T.tc_epi = iv; }
    else if (k == "tc_pipe") { CK(need(iv == 0 || iv == 1)); T.tc_pipe = iv; }
    else if (k == "batched_shape") { CK(need(iv == 0 || iv == 1)); T.batched_shape = iv; }
    else if (k == "batched_cl") { CK(need(iv >= 0 && iv <= 2)); T.batched_cl = iv; }
    else if (k == "batched_park") { CK(need(iv >= 0 && iv <= 100000)); T.batched_park = iv; }
    else if (k == "grid_solver") { CK(need(iv == 0 || iv == 1)); T.grid_solver = iv; }
    else return fail(ctx, SK_EINVAL, "sk_set_tuning: unknown key '%s'", key);
    return SK_OK;
}

sk_status sk_set_relaxation(sk_ctx *ctx, float omega) {
    if (!ctx) return SK_EINVAL;
    if (!(omega > 0.f && omega < 2.f)) return fail(ctx, SK_EINVAL, "omega must lie in (0, 2), got %g", (double)omega);
    ctx->omega = omega;
    return SK_OK;
}

void sk_destroy(sk_ctx *ctx) {
    if (!ctx) return;
    cudaStreamSynchronize(ctx->stream);
    for (auto &b : ctx->bufs)
        if (b.p) cudaFree(b.p);
    if (ctx->comm && g_nccl.destroy) g_nccl.destroy(ctx->comm);
    if (ctx->h_flag) cudaFreeHost(ctx->h_flag);
    if (ctx->h_status) cudaFreeHost(ctx->h_status);
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    for (cudaEvent_t e : ctx->tev) cudaEventDestroy(e);
    delete ctx;
}

const char *sk_last_error(const sk_ctx *ctx) { return ctx ? ctx->err.c_str() : "null context"; }

sk_status sk_set_timing(sk_ctx *ctx, int32_t enable) {
    if (!ctx) return SK_EINVAL;
    ctx->timing = enable;
    return SK_OK;
}

sk_status sk_get_counters(const sk_ctx *ctx, sk_counters *out) {
    if (!ctx || !out) return SK_EINVAL;
    *out = ctx->cnt;
    return SK_OK;
}

sk_status sk_reset_counters(sk_ctx *ctx) {
    if (!ctx) return SK_EINVAL;
    ctx->cnt = sk_counters{};
    return SK_OK;
}

sk_status sk_shard_rows(int64_t n_total, int32_t rank, int32_t world, int64_t *row0, int64_t *n_local) {
    if (!row0 || !n_local || n_total < 1 || world < 1 || rank < 0 || rank >= world) return SK_EINVAL;
    if (SK_SHARD_BLOCKS % world) return SK_EUNSUPPORTED;  // world in {1, 2, 4, 8}
    const long long bs = shard_block_rows(n_total);
    const long long per = (long long)(SK_SHARD_BLOCKS / world) * bs;
    const long long r0 = std::min<long long>(n_total, rank * per);
    const long long r1 = std::min<long long>(n_total, (rank + 1) * per);
    *row0 = r0;
    *n_local = r1 - r0;
    return SK_OK;
}

sk_status sk_nccl_unique_id(sk_ctx *ctx, void *out) {
    if (!ctx || !out) return SK_EINVAL;
    if (!g_nccl.load()) return fail(ctx, SK_ENCCL, "libnccl.so.2 could not be loaded");
    nccl_id_t id;
    int r = g_nccl.get_id(&id);
    if (r != 0) return fail(ctx, SK_ENCCL, "ncclGetUniqueId failed (%d)", r);
    memcpy(out, &id, sizeof id);
    return SK_OK;
}

sk_status sk_comm_init(sk_ctx *ctx, const void *id, int32_t rank, int32_t world) {
    if (!ctx || !id || world < 1 || rank < 0 || rank >= world) return SK_EINVAL;
    if (SK_SHARD_BLOCKS % world) return fail(ctx, SK_EUNSUPPORTED, "world must divide %d", SK_SHARD_BLOCKS);
    if (!g_nccl.load()) return fail(ctx, SK_ENCCL, "libnccl.so.2 could not be loaded");
    cudaSetDevice(ctx->device);
    nccl_id_t nid;
    memcpy(&nid, id, sizeof nid);
    int r = g_nccl.init_rank(&ctx->comm, world, nid, rank);
    if (r != 0) return fail(ctx, SK_ENCCL, "ncclCommInitRank failed: %s", g_nccl.errstr ? g_nccl.errstr(r) : "?");
    ctx->rank = rank;
    ctx->world = world;
    return SK_OK;
}

sk_status sinkhorn_sort1d_batched(sk_ctx *ctx, int64_t B, int64_t n, const float *x, int32_t *perm,
                                  int32_t *rank) {
    if (!ctx) return SK_EINVAL;
    if (B < 1 || n < 1) return fail(ctx, SK_EINVAL, "B, n must be >= 1");
    if (n > (1LL << 24)) return fail(ctx, SK_EUNSUPPORTED, "sort rows of at most 2^24 keys");
    if (!x) return fail(ctx, SK_EINVAL, "x is NULL");
    Stager sg(ctx);
    const float *dx;
    int *dp, *dr;
    CK(sg.in_t(x, (size_t)B * n, &dx));
    CK(sg.out_t(perm, (size_t)B * n, &dp));
    CK(sg.out_t(rank, (size_t)B * n, &dr));
    ENSURE(flag, int, B_FLAG, 4);
    CU(cudaMemsetAsync(flag, 0, sizeof(int), ctx->stream));
    unsigned long long *gk = nullptr;
    if (sort_rows_scratch_keys((int)B, (int)n)) {
        ENSURE(kk, unsigned long long, B_SORTKEYS, sort_rows_scratch_keys((int)B, (int)n));
        gk = kk;
    }
    CU(launch_sort_rows(dx, (int)B, (int)n, n, dp, dr, nullptr, flag, ctx->stream, gk));
    ctx->cnt.kernel_launches++;
    CK(sg.flush());
    CU(cudaMemcpyAsync(ctx->h_flag, flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    if (*ctx->h_flag) return fail(ctx, SK_EINVAL, "NaN key");
    return SK_OK;
}

sk_status sinkhorn_fit_gmm(sk_ctx *ctx, int64_t n, int32_t d, const float *x, int32_t K, const int32_t *init_idx,
                           int32_t kmeans_iters, int32_t iters, float tol, float reg_covar, float *weights,
                           float *means, float *covs, double *loglik, int32_t *n_iter) {
    if (!ctx) return SK_EINVAL;
    if (n < 1 || K < 1 || K > n || !x || !init_idx || !weights || !means || !covs || iters < 0 || kmeans_iters < 0)
        return fail(ctx, SK_EINVAL, "bad arguments (need 1 <= K <= n, iters >= 0, kmeans_iters >= 0, non-NULL arrays)");
    if (d < 1 || d > 256) return fail(ctx, SK_EINVAL, "d must be in [1, 256]");
    if (K > 64) return fail(ctx, SK_EUNSUPPORTED, "GMM fitting supports K <= 64");
    if (!(reg_covar >= 0.f) || bad_scalar(reg_covar)) return fail(ctx, SK_EINVAL, "reg_covar must be >= 0");
    if (!(tol >= 0.f) || bad_scalar(tol)) return fail(ctx, SK_EINVAL, "tol must be finite and >= 0");
    // the start indices: in range and distinct (checked on the host: K values)
    std::vector<int32_t> hidx(K);
    if (is_device_ptr(init_idx)) CU(cudaMemcpy(hidx.data(), init_idx, sizeof(int32_t) * K, cudaMemcpyDeviceToHost));
    else memcpy(hidx.data(), init_idx, sizeof(int32_t) * K);
    {
        std::vector<int32_t> srt(hidx);
        std::sort(srt.begin(), srt.end());
        for (int k = 0; k < K; ++k)
            if (srt[k] < 0 || srt[k] >= n || (k && srt[k] == srt[k - 1]))
                return fail(ctx, SK_EINVAL, "init_idx must hold K distinct indices in [0, n)");
    }
    Stager sg(ctx);
    const float *dx;
    float *dw, *dm, *dc;
    CK(sg.in_t(x, (size_t)n * d, &dx));
    CK(sg.out_t(weights, (size_t)K, &dw));
    CK(sg.out_t(means, (size_t)K * d, &dm));
    CK(sg.out_t(covs, (size_t)K * d * d, &dc));
    CK(check_arrays(ctx, {{dx, n * d}}, {}, "GMM fit"));
    ENSURE(didx, int, B_EMIDX, K);
    CU(cudaMemcpyAsync(didx, hidx.data(), sizeof(int32_t) * K, cudaMemcpyHostToDevice, ctx->stream));
    ENSURE(st, double, B_EMST, 2 * em_state_doubles(K, d) + 2 * (size_t)d * d + d + 1);
    const size_t partn = std::max(em_work_doubles(K, d), (size_t)moments_blocks(d) * d * d);
    ENSURE(part, double, B_EMPART, partn);
    double *wide = nullptr;
    if (d > 32) {
        ENSURE(wd, double, B_EMWIDE, em_wide_doubles(n, K, d));
        wide = wd;
    }
    ENSURE(flag, int, B_FLAG, 4);
    double *mean0 = st + 2 * em_state_doubles(K, d), *cov0 = mean0 + d, *ll = cov0 + (size_t)d * d;
    CU(cudaMemsetAsync(flag, 0, 3 * sizeof(int), ctx->stream));
    CU(launch_moments(dx, nullptr, n, d, mean0, cov0, part, (long long)partn, ctx->stream));
    CU(launch_gmm_fit(dx, n, d, K, didx, cov0, kmeans_iters, iters, (double)tol, (double)reg_covar, st, part, flag, dw,
                      dm, dc, ll, ctx->h_flag, ctx->stream, wide));
    ctx->cnt.kernel_launches += 4 + 3 * (kmeans_iters > 0 ? kmeans_iters + 1 : 0) + 4 * (iters + 1) + 3;
    CK(sg.flush());
    double hll = 0.0;
    int hf[3] = {0, 0, 0};
    CU(cudaMemcpyAsync(hf, flag, sizeof hf, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaMemcpyAsync(&hll, ll, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    *ctx->h_flag = hf[0];
    if (loglik) *loglik = hll;
    if (n_iter) *n_iter = hf[2];
    if (*ctx->h_flag) return fail(ctx, SK_ENONFINITE, "a component covariance lost positive definiteness");
    return SK_OK;
}

sk_status sinkhorn_vjp(sk_ctx *ctx, int64_t n, int64_t m, int32_t d, const float *x, const float *y, float eps,
                       const float *f, const float *g, const float *zf, const float *zg, float cg_tol,
                       int32_t cg_max_iter, float *grad_x, float *grad_y, float *grad_a, float *grad_b,
                       int32_t *cg_iters, double *cg_relres) {
    if (!ctx) return SK_EINVAL;
    if (n < 1 || m < 1 || d < 1 || d > 256 || !x || !y || !f || !g || !zf || !zg || cg_max_iter < 1)
        return fail(ctx, SK_EINVAL, "bad arguments (d in [1, 256])");
    if (!(eps > 0.f) || bad_scalar(eps) || !(cg_tol > 0.f) || bad_scalar(cg_tol))
        return fail(ctx, SK_EINVAL, "eps and cg_tol must be > 0 and finite");
    Stager sg(ctx);
    const float *dx, *dy, *df, *dg, *dzf, *dzg;
    float *gx, *gy, *ga, *gb;
    CK(sg.in_t(x, (size_t)n * d, &dx));
    CK(sg.in_t(y, (size_t)m * d, &dy));
    CK(sg.in_t(f, (size_t)n, &df));
    CK(sg.in_t(g, (size_t)m, &dg));
    CK(sg.in_t(zf, (size_t)n, &dzf));
    CK(sg.in_t(zg, (size_t)m, &dzg));
    CK(sg.out_t(grad_x, grad_x ? (size_t)n * d : 0, &gx));
    CK(sg.out_t(grad_y, grad_y ? (size_t)m * d : 0, &gy));
    CK(sg.out_t(grad_a, grad_a ? (size_t)n : 0, &ga));
    CK(sg.out_t(grad_b, grad_b ? (size_t)m : 0, &gb));
    CK(check_arrays(ctx, {{dx, n * d}, {dy, m * d}, {df, n}, {dg, m}, {dzf, n}, {dzg, m}}, {}, "vjp"));
    ENSURE(work, double, B_VJP, vjp_work_doubles(n, m, d) + (size_t)std::max(n, m) * d);
    int it = 0;
    double rr = 0.0;
    CU(launch_vjp(n, m, d, dx, dy, eps, df, dg, dzf, dzg, (double)cg_tol, cg_max_iter, work, gx, gy, ga, gb, &it,
                  &rr, ctx->stream));
    ctx->cnt.kernel_launches += 3 + 3 * it + 1 + (gx ? 2 : 0) + (gy ? 2 : 0);
    CK(sg.flush());
    CU(cudaStreamSynchronize(ctx->stream));
    if (cg_iters) *cg_iters = it;
    if (cg_relres) *cg_relres = rr;
    return SK_OK;
}

sk_status sinkhorn_soft_rank_sort(sk_ctx *ctx, int64_t B, int64_t n, int64_t m, const float *x, const float *y,
                                  int32_t y_shared, float eps, const float *f, const float *g, const float *z,
                                  float *rank, float *sort) {
    if (!ctx) return SK_EINVAL;
    if (B < 1 || n < 1 || m < 1 || !x || !y || !f || !g) return fail(ctx, SK_EINVAL, "bad arguments");
    if (!(eps > 0.f) || bad_scalar(eps)) return fail(ctx, SK_EINVAL, "eps must be > 0 and finite");
    if (!rank && !sort) return SK_OK;
    if (n > (1 << 24) || m > (1 << 24) || B > 65535)
        return fail(ctx, SK_EUNSUPPORTED, "soft rank/sort: n, m <= 2^24, B <= 65535");
    Stager sg(ctx);
    const long long ycount = y_shared ? m : B * m;
    const float *dx, *dy, *df, *dg, *dz;
    float *dr, *ds;
    CK(sg.in_t(x, (size_t)B * n, &dx));
    CK(sg.in_t(y, (size_t)ycount, &dy));
    CK(sg.in_t(f, (size_t)B * n, &df));
    CK(sg.in_t(g, (size_t)B * m, &dg));
    CK(sg.in_t(z, z ? (size_t)m : 0, &dz));
    CK(sg.out_t(rank, rank ? (size_t)B * n : 0, &dr));
    CK(sg.out_t(sort, sort ? (size_t)B * m : 0, &ds));
    CK(check_arrays(ctx, {{dx, B * n}, {dy, ycount}, {df, B * n}, {dg, B * m}, {dz, dz ? m : 0}}, {},
                    "soft rank/sort"));
    CU(launch_soft_rank_sort(B, (int)n, (int)m, dx, dy, y_shared ? 0 : m, df, dg, dz, eps, dr, ds, ctx->stream));
    ctx->cnt.kernel_launches++;
    CK(sg.flush());
    return SK_OK;
}

sk_status sinkhorn_init_zero(sk_ctx *ctx, int64_t B, int64_t n, float *pot) {
    if (!ctx) return SK_EINVAL;
    if (B < 1 || n < 1 || !pot) return fail(ctx, SK_EINVAL, "B, n >= 1 and pot required");
    Stager sg(ctx);
    float *dp;
    CK(sg.out_t(pot, (size_t)B * n, &dp));
    CU(launch_fill(dp, B * n, 0.f, ctx->stream));
    ctx->cnt.kernel_launches++;
    CK(sg.flush());
    return SK_OK;
}

sk_status sinkhorn_init_sort1d(sk_ctx *ctx, int64_t B, int64_t n, int64_t m, const float *x,
                               const float *y, int32_t y_shared, int32_t dualsort_iters, float *pot,
                               int32_t *perm, int32_t *rank) {
    if (!ctx) return SK_EINVAL;
    if (B < 1 || n < 1 || m < 1 || !x || !y || !pot) return fail(ctx, SK_EINVAL, "bad arguments");
    if (n != m) return fail(ctx, SK_EUNSUPPORTED, "sort1d initializer needs n == m (sinkhorn_init_nw1d: any n, m)");
    if (n > (1LL << 24)) return fail(ctx, SK_EUNSUPPORTED, "sort1d initializer supports n <= 2^24");
    if (dualsort_iters > 0 && n > 4096)
        return fail(ctx, SK_EUNSUPPORTED, "paper-mode DualSort (L Jacobi sweeps, O(L n^2)) supports n <= 4096");
    if (dualsort_iters < 0) return fail(ctx, SK_EINVAL, "dualsort_iters >= 0");
    Stager sg(ctx);
    const float *dx, *dy;
    float *dpot;
    int *dperm_user, *drank;
    CK(sg.in_t(x, (size_t)B * n, &dx));
    CK(sg.in_t(y, (size_t)(y_shared ? 1 : B) * m, &dy));
    CK(sg.out_t(pot, (size_t)B * n, &dpot));
    CK(sg.out_t(perm, (size_t)B * n, &dperm_user));
    CK(sg.out_t(rank, (size_t)B * n, &drank));
    ENSURE(flag, int, B_FLAG, 4);
    ENSURE(xs, float, B_SORT, B * n);
    ENSURE(ys, float, B_YSORT, (y_shared ? 1 : B) * m);
    ENSURE(pscr, int, B_PERM, (y_shared ? 1 : B) * m + B * n);
    int *dperm = dperm_user ? dperm_user : pscr + (y_shared ? 1 : B) * m;
    CU(cudaMemsetAsync(flag, 0, sizeof(int), ctx->stream));
    unsigned long long *gk = nullptr;
    double *gd = nullptr;
    if (sort_rows_scratch_keys((int)B, (int)n)) {
        ENSURE(kk, unsigned long long, B_SORTKEYS, sort_rows_scratch_keys((int)B, (int)n));
        gk = kk;
    }
    if (n > 4096) {
        ENSURE(dd, double, B_DUALSCR, 4 * B * n);
        gd = dd;
    }
    CU(launch_sort_rows(dy, (int)(y_shared ? 1 : B), (int)m, m, pscr, nullptr, ys, flag, ctx->stream, gk));
    CU(launch_sort_rows(dx, (int)B, (int)n, n, dperm, drank, xs, flag, ctx->stream, gk));
    CU(launch_sort1d_dual(xs, dperm, ys, y_shared, (int)B, (int)n, dualsort_iters, dpot, ctx->stream, gd));
    ctx->cnt.kernel_launches += 3;
    CK(sg.flush());
    CU(cudaMemcpyAsync(ctx->h_flag, flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    if (*ctx->h_flag) return fail(ctx, SK_EINVAL, "NaN in x or y");
    return SK_OK;
}

sk_status sinkhorn_init_nw1d(sk_ctx *ctx, int64_t B, int64_t n, int64_t m, const float *x, const float *y,
                             int32_t y_shared, const float *a, const float *b, int32_t max_rounds, float *pot,
                             int32_t *rounds) {
    if (!ctx) return SK_EINVAL;
    if (B < 1 || n < 1 || m < 1 || !x || !y || !pot) return fail(ctx, SK_EINVAL, "bad arguments");
    if (max_rounds < 0) return fail(ctx, SK_EINVAL, "max_rounds >= 0 (0 = until converged)");
    if (n > (1 << 20) || m > (1 << 20))
        return fail(ctx, SK_EUNSUPPORTED, "general 1D initializer: n, m <= 2^20 (O(n m) per round on one CTA)");
    Stager sg(ctx);
    const long long ycount = (y_shared ? 1 : B) * m;
    const float *dx, *dy, *da, *db;
    float *dpot;
    int *drounds;
    CK(sg.in_t(x, (size_t)B * n, &dx));
    CK(sg.in_t(y, (size_t)ycount, &dy));
    CK(sg.in_t(a, a ? (size_t)B * n : 0, &da));
    CK(sg.in_t(b, b ? (size_t)ycount : 0, &db));
    CK(sg.out_t(pot, (size_t)B * n, &dpot));
    CK(sg.out_t(rounds, rounds ? (size_t)B : 0, &drounds));
    CK(check_arrays(ctx, {{dx, B * n}, {dy, ycount}}, {{da, da ? B * n : 0}, {db, db ? ycount : 0}}, "sinkhorn_init_nw1d"));
    ENSURE(flag, int, B_FLAG, 4);
    ENSURE(xs, float, B_SORT, B * n);
    ENSURE(ys, float, B_YSORT, ycount);
    ENSURE(pscr, int, B_PERM, ycount + B * n);
    CU(cudaMemsetAsync(flag, 0, sizeof(int), ctx->stream));
    unsigned long long *gk = nullptr;
    const size_t nk = std::max(sort_rows_scratch_keys((int)(y_shared ? 1 : B), (int)m), sort_rows_scratch_keys((int)B, (int)n));
    if (nk) {
        ENSURE(kk, unsigned long long, B_SORTKEYS, nk);
        gk = kk;
    }
    char *gslot = nullptr;
    if (nw1d_smem_bytes((int)n, (int)m) > 220 * 1024) {
        ENSURE(gs, char, B_DUALSCR, (size_t)B * nw1d_slot_bytes((int)n, (int)m));
        gslot = gs;
    }
    CU(launch_sort_rows(dy, (int)(y_shared ? 1 : B), (int)m, m, pscr, nullptr, ys, flag, ctx->stream, gk));
    CU(launch_sort_rows(dx, (int)B, (int)n, n, pscr + ycount, nullptr, xs, flag, ctx->stream, gk));
    CU(launch_nw1d(xs, pscr + ycount, ys, pscr, y_shared ? 1 : 0, da, db, (int)B, (int)n, (int)m,
                   max_rounds ? max_rounds : (int)(n + m + 2), dpot, drounds, ctx->stream, gslot));
    ctx->cnt.kernel_launches += 3;
    CK(sg.flush());
    CU(cudaMemcpyAsync(ctx->h_flag, flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    if (*ctx->h_flag) return fail(ctx, SK_EINVAL, "NaN in x or y");
    return SK_OK;
}

sk_status sinkhorn_init_gaussian(sk_ctx *ctx, int64_t n, int64_t m, int32_t d, const float *x,
                                 const float *a, const float *y, const float *b, float ridge_rel,
                                 float *pot, int32_t *side) {
    if (!ctx) return SK_EINVAL;
    if (n < 1 || m < 1 || d < 1 || d > 256 || !x || !y || !pot || !side)
        return fail(ctx, SK_EINVAL, "bad arguments (d in [1,256])");
    if (!(ridge_rel >= 0.f) || bad_scalar(ridge_rel)) return fail(ctx, SK_EINVAL, "ridge_rel >= 0");
    const bool swap = n > m;  // potential on the smaller side
    Stager sg(ctx);
    const float *dx, *dy, *da, *db;
    float *dpot;
    CK(sg.in_t(x, (size_t)n * d, &dx));
    CK(sg.in_t(y, (size_t)m * d, &dy));
    CK(sg.in_t(a, (size_t)n, &da));
    CK(sg.in_t(b, (size_t)m, &db));
    CK(sg.out_t(pot, (size_t)(swap ? m : n), &dpot));
    CK(check_arrays(ctx, {{dx, n * d}, {dy, m * d}}, {{da, n}, {db, m}}, "sinkhorn_init_gaussian"));
    if (swap) { std::swap(dx, dy); std::swap(da, db); std::swap(n, m); }
    const long long nbmax = moments_blocks(d);
    const long long D = std::max(d, 64), wide = d > 64 ? (long long)gauss_wide_work_doubles(d) : 0;
    ENSURE(gw, double, B_GAUSS, 2 * D + 3 * D * D + wide);
    ENSURE(scr, double, B_GAUSS2, nbmax * d * d + 64);
    double *mmu = gw, *mnu = gw + D, *Smu = gw + 2 * D, *Snu = Smu + D * D, *A = Snu + D * D;
    double *wk = d > 64 ? A + D * D : nullptr;
    ENSURE(flag, int, B_FLAG, 4);
    CU(cudaMemsetAsync(flag, 0, sizeof(int), ctx->stream));
    CU(launch_moments(dx, da, n, d, mmu, Smu, scr, nbmax * d * d, ctx->stream));
    CU(launch_moments(dy, db, m, d, mnu, Snu, scr, nbmax * d * d, ctx->stream));
    CU(launch_gauss_A(mmu, Smu, mnu, Snu, d, ridge_rel, A, flag, ctx->stream, wk));
    CU(launch_gauss_potential(dx, n, d, mmu, mnu, A, dpot, ctx->stream));
    ctx->cnt.kernel_launches += 10;
    CK(sg.flush());
    CU(cudaMemcpyAsync(ctx->h_flag, flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    if (*ctx->h_flag) return fail(ctx, SK_ENONFINITE, "Newton-Schulz did not converge (degenerate covariance)");
    *side = swap ? 1 : 0;
    return SK_OK;
}

sk_status sinkhorn_init_gmm(sk_ctx *ctx, int64_t n, int64_t m, int32_t d, const float *x, const float *y,
                            int32_t Kx, const float *wx, const float *mux, const float *covx, int32_t Ky,
                            const float *wy, const float *muy, const float *covy, float eps,
                            float inner_tol, int32_t inner_max_iter, float *pot, int32_t *side) {
    if (!ctx) return SK_EINVAL;
    if (n < 1 || m < 1 || d < 1 || d > 256 || !x || !y || !pot || !side)
        return fail(ctx, SK_EINVAL, "bad arguments (d in [1,256])");
    if (Kx < 1 || Ky < 1 || Kx > 64 || Ky > 64) return fail(ctx, SK_EINVAL, "1 <= K <= 64");
    if (!wx || !mux || !covx || !wy || !muy || !covy) return fail(ctx, SK_EINVAL, "mixture parameters required");
    if (!(eps > 0.f) || bad_scalar(eps) || !(inner_tol > 0.f) || inner_max_iter < 1)
        return fail(ctx, SK_EINVAL, "eps, inner_tol > 0, inner_max_iter >= 1");
    const bool swap = n > m;
    Stager sg(ctx);
    const float *dx, *dy, *dwx, *dmux, *dcovx, *dwy, *dmuy, *dcovy;
    float *dpot;
    CK(sg.in_t(x, (size_t)n * d, &dx));
    CK(sg.in_t(y, (size_t)m * d, &dy));
    CK(sg.in_t(wx, (size_t)Kx, &dwx));
    CK(sg.in_t(mux, (size_t)Kx * d, &dmux));
    CK(sg.in_t(covx, (size_t)Kx * d * d, &dcovx));
    CK(sg.in_t(wy, (size_t)Ky, &dwy));
    CK(sg.in_t(muy, (size_t)Ky * d, &dmuy));
    CK(sg.in_t(covy, (size_t)Ky * d * d, &dcovy));
    CK(sg.out_t(pot, (size_t)(swap ? m : n), &dpot));
    CK(check_arrays(ctx, {{dx, n * d}, {dy, m * d}, {dmux, (long long)Kx * d}, {dmuy, (long long)Ky * d},
                          {dcovx, (long long)Kx * d * d}, {dcovy, (long long)Ky * d * d}},
                    {{dwx, Kx}, {dwy, Ky}}, "sinkhorn_init_gmm"));
    if (swap) {
        std::swap(dx, dy); std::swap(n, m); std::swap(Kx, Ky);
        std::swap(dwx, dwy); std::swap(dmux, dmuy); std::swap(dcovx, dcovy);
    }
    ENSURE(work, double, B_GMM, gmm_work_doubles(d, Kx, Ky));
    ENSURE(flag, int, B_FLAG, 4);
    CU(cudaMemsetAsync(flag, 0, sizeof(int), ctx->stream));
    CU(launch_gmm_init(dx, n, d, Kx, dwx, dmux, dcovx, Ky, dwy, dmuy, dcovy, eps, inner_tol, inner_max_iter,
                       dpot, work, flag, ctx->stream));
    ctx->cnt.kernel_launches += 5;
    CK(sg.flush());
    CU(cudaMemcpyAsync(ctx->h_flag, flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    if (*ctx->h_flag & 4) return fail(ctx, SK_EINVAL, "a mixture covariance is not positive definite");
    if (*ctx->h_flag) return fail(ctx, SK_ENONFINITE, "GMM initializer failed (Newton-Schulz or K x K solve)");
    *side = swap ? 1 : 0;
    return SK_OK;
}

// forward
sk_status solve_impl(sk_ctx *ctx, int64_t B, int64_t n, int64_t m, int32_t d, const float *x, long long xs,
                     const float *y, long long ys, const float *a, long long as, const float *b, long long bs,
                     float eps, float tol, int32_t max_iter, int32_t check_every, sk_cost_mode mode,
                     const float *f_init, float *f, float *g, sk_report *rep);

sk_status sinkhorn_init_subsample(sk_ctx *ctx, int64_t n, int64_t m, int32_t d, const float *x, const float *y,
                                  int64_t ns, const int32_t *idx_x, int64_t ms, const int32_t *idx_y, float eps,
                                  float inner_tol, int32_t inner_max_iter, float *pot, int32_t *side,
                                  sk_report *inner) {
    if (!ctx) return SK_EINVAL;
    CK(validate_common(ctx, n, m, d, eps, inner_tol, inner_max_iter, 1));
    if (!x || !y || !pot || !side || !idx_x || !idx_y) return fail(ctx, SK_EINVAL, "NULL argument");
    if (ns < 1 || ms < 1 || ns > n || ms > m) return fail(ctx, SK_EINVAL, "1 <= ns <= n, 1 <= ms <= m");
    const bool swap = n > m;
    Stager sg(ctx);
    const float *dx, *dy;
    const int *dix, *diy;
    float *dpot;
    CK(sg.in_t(x, (size_t)n * d, &dx));
    CK(sg.in_t(y, (size_t)m * d, &dy));
    CK(sg.in_t(idx_x, (size_t)ns, &dix));
    CK(sg.in_t(idx_y, (size_t)ms, &diy));
    CK(sg.out_t(pot, (size_t)(swap ? m : n), &dpot));
    CK(check_arrays(ctx, {{dx, n * d}, {dy, m * d}}, {}, "sinkhorn_init_subsample"));
    {   // indices distinct and in range
        ENSURE(flag, int, B_FLAG, 4);
        ENSURE(mark, int, B_IDX, std::max(n, m));
        CU(cudaMemsetAsync(flag, 0, sizeof(int), ctx->stream));
        CU(launch_check_indices(dix, ns, n, flag, mark, ctx->stream));
        CU(launch_check_indices(diy, ms, m, flag, mark, ctx->stream));
        ctx->cnt.kernel_launches += 2;
        CU(cudaMemcpyAsync(ctx->h_flag, flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
        if (*ctx->h_flag) return fail(ctx, SK_EINVAL, "subsample indices out of range or repeated");
    }
    if (swap) { std::swap(dx, dy); std::swap(n, m); std::swap(dix, diy); std::swap(ns, ms); }
    ENSURE(w, float, B_SUBW, ns * d);
    ENSURE(z, float, B_SUBZ, ms * d);
    ENSURE(fb, float, B_SUBF, ns);
    ENSURE(gbv, float, B_SUBG, ms);
    CU(launch_gather_rows(dx, dix, ns, d, w, ctx->stream));
    CU(launch_gather_rows(dy, diy, ms, d, z, ctx->stream));
    ctx->cnt.kernel_launches += 2;
    // inner solve (uniform weights, same eps, inner_tol) -> g~ (Sec. 3.4)
    sk_report rin{};
    sk_status s;
    // plain Sinkhorn on a problem whose clouds fit every SM's shared memory: one grid-persistent
    // launch (K20) instead of the multi-kernel loop (C4's 4096^2 inner solve: 9.2 -> ~2 ms)
    const bool plain = ctx->anderson < 2 && ctx->omega == 1.f && ctx->decay_init <= 0.f && !ctx->adapt;
    if (plain && ctx->tune.grid_solver && grid_solver_supported(d, (int)ns, (int)ms) &&
        (double)ns * ms > (double)(1 << 18)) {
        int nsm = 148;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->device);
        ENSURE(gw, char, B_GRID, grid_solver_workspace_bytes((int)ns, (int)ms, nsm));
        GridLaunch GL{(int)ns, (int)ms, d, w, z, nullptr, nullptr, nullptr, eps, inner_tol, inner_max_iter, 1,
                      fb, gbv, gw, nullptr};
        GridResult hr{};
        GL.res_host = &hr;
        CU(cudaEventRecord(ctx->ev0, ctx->stream));
        const cudaError_t ge = launch_grid_solver(GL, ctx->stream);
        if (ge == cudaErrorCooperativeLaunchTooLarge || ge == cudaErrorInvalidConfiguration) {
            // (fewer SMs available than the grid needs co-resident: the general solver)
            cudaGetLastError();
            s = solve_impl(ctx, 1, ns, ms, d, w, 0, z, 0, nullptr, 0, nullptr, 0, eps, inner_tol,
                           inner_max_iter, 1, SK_COST_ONLINE, nullptr, fb, gbv, &rin);
            goto inner_done;
        }
        CU(ge);
        CU(cudaEventRecord(ctx->ev1, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
        float gms = 0.f;
        CU(cudaEventElapsedTime(&gms, ctx->ev0, ctx->ev1));
        ctx->cnt.kernel_launches += 1;
        ctx->cnt.lse_launches += 1;
        ctx->cnt.lse_ex2 += (double)ns * ms * (2.0 * hr.iterations + 1.0);
        rin.iterations = hr.iterations;
        rin.converged = hr.converged;
        rin.marginal_error = hr.err;
        rin.dual_objective = hr.E;
        rin.solve_ms = gms;
        s = hr.nonfinite ? SK_ENONFINITE : SK_OK;
    } else {
        s = solve_impl(ctx, 1, ns, ms, d, w, 0, z, 0, nullptr, 0, nullptr, 0, eps, inner_tol,
                       inner_max_iter, 1, SK_COST_ONLINE, nullptr, fb, gbv, &rin);
    }
inner_done:
    if (s != SK_OK && s != SK_ENONFINITE) return s;
    if (inner) *inner = rin;
    if (s == SK_ENONFINITE) return fail(ctx, SK_ENONFINITE, "inner subsample solve became non-finite");
    // Eq. (8): one online LSE pass of all x against (z, g~): f0_i = eps log ms + |x_i|^2 - eps ln2 LSE2
    const int D = lse_dpad(d);
    const int tq = lse_tq(D);
    const long long xt = lse_tiles(n, tq), zt = lse_tiles(ms, tq);
    ENSURE(xpack, float, B_XPACK, xt * (D + 1) * tq);
    ENSURE(xc, float, B_XC, n);
    ENSURE(xnk, float, B_XNK, n);
    ENSURE(xpot, float, B_XPOT, 2 * n);
    ENSURE(ypack, float, B_YPACK, zt * (D + 1) * tq);
    ENSURE(yc, float, B_YC, ms);
    ENSURE(ynk, float, B_YNK, ms);
    ENSURE(ypot, float, B_YPOT, 2 * ms);
    ENSURE(status, DevStatus, B_STATUS, 1);
    Side X{(int)n, d, D, tq, xpack, xc, xnk, {xpot, xpot + n}};
    Side Z{(int)ms, d, D, tq, ypack, yc, ynk, {ypot, ypot + ms}};
    CU(pack_side(X, dx, nullptr, 0.f, nullptr, eps, ctx->stream));   // c = |x|^2
    CU(pack_side(Z, z, nullptr, 0.f, gbv, eps, ctx->stream));       // w = (g~ - |z|^2) kappa
    const int occ = lse_occupancy_ctas(D);
    const int R = D <= 4 ? 4 : (D <= 16 ? 2 : 1);
    const int split = choose_split((n + 128LL * R - 1) / (128LL * R), zt, occ, 64);
    ENSURE(part, float2, B_PART, (long long)split * n);
    ENSURE(blke, double, B_BLKE, 2 * kMergeMaxBlocks);
    ENSURE(blkb, int, B_BLKB, 2048);
    CU(launch_status_init(status, 1, 1, 1.f, ctx->stream));
    LsePass lp{&X, &Z, 1, 0, split, part, eps, nullptr};
    CU(launch_lse(lp, ctx->stream));
    MergePass mp{MERGE_OUT, &X, part, split, eps, nullptr, status, blke, blkb, dpot,
                 (float)(eps * std::log((double)ms)), 0, 0};
    CU(launch_merge(mp, ctx->stream));
    ctx->cnt.kernel_launches += 5;
    CK(sg.flush());
    CU(cudaMemcpyAsync(ctx->h_status, status, sizeof(DevStatus), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    if (ctx->h_status->nonfinite) return fail(ctx, SK_ENONFINITE, "extrapolated potential non-finite");
    *side = swap ? 1 : 0;
    return SK_OK;
}

sk_status solve_impl(sk_ctx *ctx, int64_t B, int64_t n, int64_t m, int32_t d, const float *x, long long xs,
                     const float *y, long long ys, const float *a, long long as, const float *b, long long bs,
                     float eps, float tol, int32_t max_iter, int32_t check_every, sk_cost_mode mode,
                     const float *f_init, float *f, float *g, sk_report *rep) {
    cudaStream_t st = ctx->stream;
    const bool small = batched_supported(d, (int)n, (int)m, ctx->anderson) &&
                       (B > 1 || (double)n * m <= (double)(1 << 18));
    if (ctx->anderson >= 2 && (ctx->omega != 1.f || ctx->decay_init > 0.f))
        return fail(ctx, SK_EUNSUPPORTED, "Anderson acceleration combines with neither omega != 1 nor eps-decay");
    if (ctx->adapt && (ctx->anderson >= 2 || ctx->omega != 1.f || ctx->decay_init > 0.f))
        return fail(ctx, SK_EUNSUPPORTED, "adaptive momentum combines with neither Anderson, a fixed omega nor eps-decay");
    if (small && mode != SK_COST_STORED) {
        ENSURE(rp, char, B_REP, (size_t)B * (3 * sizeof(int) + sizeof(float) + sizeof(double)) + 64);
        ENSURE(queue, int, B_QUEUE, 4);
        double *E = (double *)rp;
        int *iters = (int *)(E + B), *conv = iters + B, *nonf = conv + B;
        float *err = (float *)(nonf + B);
        BatchLaunch L;
        L.B = (int)B; L.n = (int)n; L.m = (int)m; L.d = d; L.queue = queue;
        L.x = x; L.x_stride = xs; L.y = y; L.y_stride = ys;
        L.a = a; L.a_stride = as; L.b = b; L.b_stride = bs;
        L.finit = f_init; L.f = f; L.g = g; L.eps = eps; L.tol = tol;
        L.max_iter = max_iter; L.check_every = check_every;
        L.iters = iters; L.conv = conv; L.nonfinite = nonf; L.err = err; L.E = E;
        L.omega = ctx->omega;
        L.decay_init = ctx->decay_init; L.decay_rate = ctx->decay_rate;
        L.anderson = ctx->anderson;
        L.adapt = ctx->adapt;
        if (B > 1 && ctx->tune.batched_park > 0) {
            // park / resume workspace: state, keys, finished count, headers, LSE seeds
            const size_t bytes = (size_t)B * (8 * sizeof(double) + sizeof(float) * (n + m)) + 16 +
                                 sizeof(int) * park_queue_ints((int)B);
            ENSURE(pk, char, B_PARK, bytes);
            char *q = pk;
            L.phdr = (double *)q; q += (size_t)B * 8 * sizeof(double);
            L.done = (int *)q; q += 16;
            L.pq = (int *)q; q += sizeof(int) * park_queue_ints((int)B);
            L.pseed = (float *)q;
            L.park = ctx->tune.batched_park;
        }
        L.shape = ctx->tune.batched_shape;
        L.cl = ctx->tune.batched_cl;
        CU(cudaEventRecord(ctx->ev0, st));
        CU(launch_batched(L, st));
        CU(cudaEventRecord(ctx->ev1, st));
        ctx->cnt.kernel_launches++;
        ctx->cnt.lse_launches++;
        std::vector<char> h((size_t)B * (3 * sizeof(int) + sizeof(float) + sizeof(double)));
        CU(cudaMemcpyAsync(h.data(), rp, h.size(), cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        float ms = 0.f;
        CU(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
        if (ctx->timing) { ctx->cnt.lse_ms += ms; ctx->cnt.dom_ms += ms; ctx->cnt.dom_launches++; }
        const double *hE = (const double *)h.data();
        const int *hi = (const int *)(hE + B), *hc = hi + B, *hn = hc + B;
        const float *he = (const float *)(hn + B);
        int any_nf = 0;
        for (long long p = 0; p < B; ++p) {
            rep[p].iterations = hi[p];
            rep[p].converged = hc[p];
            rep[p].marginal_error = he[p];
            rep[p].dual_objective = hE[p];
            rep[p].build_ms = 0.0;
            rep[p].solve_ms = ms;
            any_nf |= hn[p];
            const double passes = 2.0 * hi[p] + (ctx->anderson >= 2 ? 0.0 : 1.0);   // (Anderson: 2 per sweep)
            ctx->cnt.lse_ex2 += (double)n * m * passes;
            if (ctx->timing) ctx->cnt.dom_entries += (double)n * m * passes;
        }
        if (any_nf) return fail(ctx, SK_ENONFINITE, "potentials became non-finite");
        return SK_OK;
    }
    // eps-decay (R-25) on the multi-kernel path: with omega = 1 a sweep is a map f -> f (its
    // g-update reads only f), so the T decay sweeps run as one-sweep solves at eps_l, each
    // starting from the previous f; the solve at the target eps then starts from f^T
    int T = 0;
    if (ctx->decay_init > 0.f) {
        if (ctx->omega != 1.f)
            return fail(ctx, SK_EUNSUPPORTED, "eps-decay with omega != 1 runs on the on-chip solver only");
        while (T < max_iter && (double)eps * ctx->decay_init * std::pow((double)ctx->decay_rate, T) > (double)eps) ++T;
    }
    for (long long p = 0; p < B; ++p) {
        Problem P;
        P.n_total = n; P.m = m; P.d = d;
        P.y = y + p * ys; P.b = b ? b + p * bs : nullptr;
        P.eps = eps; P.tol = tol; P.max_iter = max_iter; P.check_every = check_every; P.mode = mode;
        P.g = g + p * m;
        P.world = 1; P.nccl = false; P.omega = ctx->omega;
        const float *fi = f_init ? f_init + p * n : nullptr;
        double extra_ms = 0.0;
        for (int t = 0; t < T; ++t) {
            Problem Pt = P;
            Pt.eps = (float)((double)eps * ctx->decay_init * std::pow((double)ctx->decay_rate, t));
            Pt.max_iter = 1;   // (its stop check measures err_1 at eps_l: one column pass more)
            std::vector<Slice> st{Slice{0, n, x + p * xs, a ? a + p * as : nullptr, fi, f + p * n, 0}};
            sk_report r1{};
            CK(solve_core(ctx, Pt, st, &r1));
            extra_ms += r1.solve_ms;
            fi = f + p * n;
        }
        P.max_iter = max_iter - T;
        std::vector<Slice> sl{Slice{0, n, x + p * xs, a ? a + p * as : nullptr, fi, f + p * n, 0}};
        if (P.max_iter < 1) return fail(ctx, SK_EINVAL, "max_iter must exceed the %d eps-decay sweeps", T);
        CK(solve_core(ctx, P, sl, &rep[p]));
        rep[p].iterations += T;
        rep[p].solve_ms += extra_ms;
    }
    return SK_OK;
}

sk_status sinkhorn_solve(sk_ctx *ctx, int64_t B, int64_t n, int64_t m, int32_t d, const float *x,
                         const float *y, int32_t y_shared, const float *a, const float *b, float eps,
                         float tol, int32_t max_iter, int32_t check_every, sk_cost_mode mode,
                         const float *f_init, const float *g_init, float *f, float *g, sk_report *rep) {
    if (!ctx) return SK_EINVAL;
    CK(validate_common(ctx, n, m, d, eps, tol, max_iter, check_every));
    if (B < 1) return fail(ctx, SK_EINVAL, "B must be >= 1");
    if (!x || !y || !f || !g || !rep) return fail(ctx, SK_EINVAL, "NULL argument");
    if (f_init && g_init) return fail(ctx, SK_EINVAL, "at most one of f_init, g_init (P:84)");
    if (mode < SK_COST_AUTO || mode > SK_COST_STORED) return fail(ctx, SK_EINVAL, "bad cost mode");
    const long long ny = y_shared ? 1 : B;
    Stager sg(ctx);
    const float *dx, *dy, *da, *db, *dfi, *dgi;
    float *df, *dg;
    CK(sg.in_t(x, (size_t)B * n * d, &dx));
    CK(sg.in_t(y, (size_t)ny * m * d, &dy));
    CK(sg.in_t(a, (size_t)B * n, &da));
    CK(sg.in_t(b, (size_t)ny * m, &db));
    CK(sg.in_t(f_init, (size_t)B * n, &dfi));
    CK(sg.in_t(g_init, (size_t)B * m, &dgi));
    CK(sg.out_t(f, (size_t)B * n, &df));
    CK(sg.out_t(g, (size_t)B * m, &dg));
    CK(check_arrays(ctx, {{dx, B * n * d}, {dy, ny * m * d}, {dfi, B * n}, {dgi, B * m}},
                    {{da, B * n}, {db, ny * m}}, "sinkhorn_solve"));
    for (long long p = 0; p < B; ++p) rep[p] = sk_report{};
    sk_status s;
    if (dgi)  // transposed problem: x<->y, a<->b, f<->g
        s = solve_impl(ctx, B, m, n, d, dy, y_shared ? 0 : m * d, dx, n * d, db, y_shared ? 0 : m, da, n, eps,
                       tol, max_iter, check_every, mode, dgi, dg, df, rep);
    else
        s = solve_impl(ctx, B, n, m, d, dx, n * d, dy, y_shared ? 0 : m * d, da, n, db, y_shared ? 0 : m, eps,
                       tol, max_iter, check_every, mode, dfi, df, dg, rep);
    if (s != SK_OK && s != SK_ENONFINITE) return s;
    sk_status s2 = sg.flush();
    CU(cudaStreamSynchronize(ctx->stream));
    return s != SK_OK ? s : s2;
}

sk_status sinkhorn_solve_sharded(sk_ctx *ctx, int64_t n_total, int64_t row0, int64_t n_local, int64_t m,
                                 int32_t d, const float *x_local, const float *y, const float *a_local,
                                 const float *b, float eps, float tol, int32_t max_iter, int32_t check_every,
                                 sk_cost_mode mode, const float *f_init_local, float *f_local, float *g,
                                 sk_report *rep) {
    if (!ctx) return SK_EINVAL;
    CK(validate_common(ctx, n_local, m, d, eps, tol, max_iter, check_every));
    if (!x_local || !y || !f_local || !g || !rep) return fail(ctx, SK_EINVAL, "NULL argument");
    int64_t r0, nl;
    CK(sk_shard_rows(n_total, ctx->rank, ctx->world, &r0, &nl));
    if (r0 != row0 || nl != n_local)
        return fail(ctx, SK_EINVAL, "rank %d must own rows [%lld, %lld) (sk_shard_rows)", ctx->rank,
                    (long long)r0, (long long)(r0 + nl));
    if (ctx->world > 1 && !ctx->comm) return fail(ctx, SK_ENCCL, "sk_comm_init was not called");
    Stager sg(ctx);
    const float *dx, *dy, *da, *db, *dfi;
    float *df, *dg;
    CK(sg.in_t(x_local, (size_t)n_local * d, &dx));
    CK(sg.in_t(y, (size_t)m * d, &dy));
    CK(sg.in_t(a_local, (size_t)n_local, &da));
    CK(sg.in_t(b, (size_t)m, &db));
    CK(sg.in_t(f_init_local, (size_t)n_local, &dfi));
    CK(sg.out_t(f_local, (size_t)n_local, &df));
    CK(sg.out_t(g, (size_t)m, &dg));
    CK(check_arrays(ctx, {{dx, n_local * d}, {dy, m * d}, {dfi, n_local}}, {{da, n_local}, {db, m}},
                    "sinkhorn_solve_sharded"));
    *rep = sk_report{};
    Problem P;
    P.n_total = n_total; P.m = m; P.d = d;
    P.y = dy; P.b = db;
    P.eps = eps; P.tol = tol; P.max_iter = max_iter; P.check_every = check_every; P.mode = mode;
    P.g = dg;
    P.world = ctx->world; P.nccl = ctx->world > 1 || (ctx->force_nccl && ctx->comm); P.partitioned = true;
    P.omega = ctx->omega;
    std::vector<Slice> sl{Slice{row0, n_local, dx, da, dfi, df, ctx->rank}};
    sk_status s = solve_core_decay(ctx, P, sl, rep);
    if (s != SK_OK && s != SK_ENONFINITE) return s;
    sk_status s2 = sg.flush();
    CU(cudaStreamSynchronize(ctx->stream));
    return s != SK_OK ? s : s2;
}

sk_status sinkhorn_solve_sharded_emulated(sk_ctx *ctx, int32_t world, int64_t n, int64_t m, int32_t d,
                                          const float *x, const float *y, const float *a, const float *b,
                                          float eps, float tol, int32_t max_iter, int32_t check_every,
                                          sk_cost_mode mode, const float *f_init, float *f, float *g,
                                          sk_report *rep) {
    if (!ctx) return SK_EINVAL;
    CK(validate_common(ctx, n, m, d, eps, tol, max_iter, check_every));
    if (!x || !y || !f || !g || !rep) return fail(ctx, SK_EINVAL, "NULL argument");
    if (world < 1 || SK_SHARD_BLOCKS % world) return fail(ctx, SK_EINVAL, "world must divide %d", SK_SHARD_BLOCKS);
    Stager sg(ctx);
    const float *dx, *dy, *da, *db, *dfi;
    float *df, *dg;
    CK(sg.in_t(x, (size_t)n * d, &dx));
    CK(sg.in_t(y, (size_t)m * d, &dy));
    CK(sg.in_t(a, (size_t)n, &da));
    CK(sg.in_t(b, (size_t)m, &db));
    CK(sg.in_t(f_init, (size_t)n, &dfi));
    CK(sg.out_t(f, (size_t)n, &df));
    CK(sg.out_t(g, (size_t)m, &dg));
    CK(check_arrays(ctx, {{dx, n * d}, {dy, m * d}, {dfi, n}}, {{da, n}, {db, m}},
                    "sinkhorn_solve_sharded_emulated"));
    *rep = sk_report{};
    Problem P;
    P.n_total = n; P.m = m; P.d = d;
    P.y = dy; P.b = db;
    P.eps = eps; P.tol = tol; P.max_iter = max_iter; P.check_every = check_every; P.mode = mode;
    P.g = dg;
    P.world = world; P.nccl = false; P.partitioned = true; P.omega = ctx->omega;
    std::vector<Slice> sl;
    for (int r = 0; r < world; ++r) {
        int64_t r0, nl;
        CK(sk_shard_rows(n, r, world, &r0, &nl));
        if (nl < 1) return fail(ctx, SK_EUNSUPPORTED, "rank %d would own no rows (n too small for %d ranks)", r, world);
        sl.push_back(Slice{r0, nl, dx + r0 * d, da ? da + r0 : nullptr, dfi ? dfi + r0 : nullptr, df + r0, r});
    }
    sk_status s = solve_core_decay(ctx, P, sl, rep);
    if (s != SK_OK && s != SK_ENONFINITE) return s;
    sk_status s2 = sg.flush();
    CU(cudaStreamSynchronize(ctx->stream));
    return s != SK_OK ? s : s2;
}

sk_status sk_selftest_tc_dot(sk_ctx *ctx, int32_t d, const float *x, const float *y, float *out) {
    if (!ctx) return SK_EINVAL;
    if (d < 1 || d > 256 || !x || !y || !out) return fail(ctx, SK_EINVAL, "d in [1, 256], non-NULL arrays");
    const int ksteps = (d + 15) / 16;
    Stager sg(ctx);
    const float *dx, *dy;
    float *dout;
    CK(sg.in_t(x, (size_t)128 * d, &dx));
    CK(sg.in_t(y, (size_t)128 * d, &dy));
    CK(sg.out_t(out, (size_t)128 * 128, &dout));
    const int rb = tc_row_bytes(d);   // (the solver's layout for this d)
    ENSURE(ximg, char, B_XIMG, tc_image_bytes(128, rb));
    ENSURE(yimg, char, B_YIMG, tc_image_bytes(128, rb));
    ENSURE(amax, unsigned, B_TCMAX, 2);
    ENSURE(part, float2, B_PART, 128);
    CU(cudaMemsetAsync(amax, 0, 2 * sizeof(unsigned), ctx->stream));
    CU(launch_absmax(dx, 128LL * d, amax, ctx->stream));
    CU(launch_absmax(dy, 128LL * d, amax + 1, ctx->stream));
    unsigned h[2];
    CU(cudaMemcpyAsync(h, amax, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    float hx, hy;
    memcpy(&hx, &h[0], 4);
    memcpy(&hy, &h[1], 4);
    if (!tc_fold_ok(hx, hy, 1.f)) return fail(ctx, SK_EUNSUPPORTED, "scaled coordinates outside the fp16 range");
    // eps = 1: the accumulator is 2 log2(e) <x, y> (+ w - sh = 0); the kernel unscales it
    CU(launch_pack_tc(dx, 128, d, amax, 0, 1.f, ximg, ctx->stream, rb));
    CU(launch_pack_tc(dy, 128, d, amax, 1, 1.f, yimg, ctx->stream, rb));
    CU(launch_pack_tc_ext(128, nullptr, ximg, ctx->stream, rb));
    CU(launch_pack_tc_ext(128, nullptr, yimg, ctx->stream, rb));
    TcPass tp{ximg, yimg, 128, 128, ksteps, 1, 0, 1, part, 1.f, nullptr};
    tp.rb = rb;
    tp.debug_acc = dout;
    CU(launch_lse_tc(tp, ctx->stream));
    ctx->cnt.kernel_launches += 7;
    CK(sg.flush());
    CU(cudaStreamSynchronize(ctx->stream));
    return SK_OK;
}

static int nsm_probe(sk_ctx *ctx) {
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, ctx->device);
    return n;
}

sk_status sk_microbench(sk_ctx *ctx, int32_t kind, double *value) {
    if (!ctx || !value || kind < 0 || (kind > 14 && kind < 100) || kind > 163)
        return fail(ctx, SK_EINVAL, "kind in [0, 14] or [100, 163]");
    if ((kind >= 5 && kind <= 8) || kind >= 100) {   // raw MMA issue rate of one shape, flop per SM clock
        ENSURE(scr, long long, B_OUT, 16);
        CU(microbench_mma(kind >= 100 ? kind - 100 : kind - 5, scr, ctx->stream, value));
        ctx->cnt.kernel_launches += 2;
        return SK_OK;
    }
    cudaStream_t st = ctx->stream;
    ENSURE(sink, float, B_OUT, 1024);
    float ms = 0.f;
    if (kind <= 1) {
        double ops = 0.0;
        CU(microbench_alu(kind, st, ctx->ev0, ctx->ev1, sink, &ops));
        CU(cudaEventSynchronize(ctx->ev1));
        CU(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
        *value = ops / (ms * 1e-3);
    } else if (kind == 2) {
        const long long bytes = 4LL << 30;
        cudaError_t e;
        float *buf = (float *)ensure(ctx, B_COST, bytes, &e);
        if (!buf) return fail(ctx, SK_ENOMEM, "4 GiB probe buffer");
        CU(cudaMemsetAsync(buf, 0, bytes, st));
        CU(microbench_hbm(buf, bytes, st, ctx->ev0, ctx->ev1, sink));
        CU(cudaEventSynchronize(ctx->ev1));
        CU(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
        *value = (double)bytes / (ms * 1e-3);
    } else {
        const long long P = 32768, Q = 32768;   // 256 x 256 tiles of 128 x 128 x 64, 3 fp16 MMAs each
        cudaError_t e1;
        char *img = (char *)ensure(ctx, B_XIMG, tc_image_bytes(P), &e1);
        ENSURE(part, float2, B_PART, P * 37);
        if (!img) return fail(ctx, SK_ENOMEM, "tc probe images");
        CU(cudaMemsetAsync(img, 0, tc_image_bytes(P), st));
        CU(launch_pack_tc_ext(P, nullptr, img, st));   // w = 0, shifts 0
        TcPass tp{img, img, (int)P, Q, 4, 1, 0, 37, part, 1.f, nullptr};
        tp.mma_only = (kind == 4 || kind == 10) ? 2 : (kind == 11 ? 3 : (kind == 12 ? 4 : (kind == 13 ? 5 : (kind == 14 ? 0 : 1))));
        tp.emu = ctx->tune.tc_emu;
        tp.epi = ctx->tune.tc_epi;
        tp.pipe = ctx->tune.tc_pipe;
        ENSURE(cyc, long long, B_FA, 16);
        tp.cyc = cyc;
        tp.seeded = kind == 11 || kind == 13 || kind == 14;   // the seeded (max-free) epilogue, as the solver runs
        CU(launch_lse_tc(tp, st));  // warm-up
        CU(cudaEventRecord(ctx->ev0, st));
        CU(launch_lse_tc(tp, st));
        CU(cudaEventRecord(ctx->ev1, st));
        CU(cudaEventSynchronize(ctx->ev1));
        CU(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
        long long c = 0;
        CU(cudaMemcpy(&c, cyc, sizeof c, cudaMemcpyDeviceToHost));
        // kinds 3, 4: flop/s; kinds 9, 10 (same runs): flop per SM clock of CTA 0
        const double flops = 3.0 * 2.0 * 64.0 * (double)P * (double)Q;
        *value = kind >= 9 ? flops / nsm_probe(ctx) / (double)(c > 0 ? c : 1) : flops / (ms * 1e-3);
    }
    ctx->cnt.kernel_launches += 2;
    return SK_OK;
}

}  // extern "C"
