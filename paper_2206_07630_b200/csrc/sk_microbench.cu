// sk_microbench.cu — K14: roofline denominators measured on the device the solver runs on.
//   SK_MB_EX2   MUFU.EX2 throughput (ex2/s): 8 independent ex2 chains per thread
//   SK_MB_FFMA  FP32 FMA throughput (FMA/s): 8 independent FFMA2 chains per thread (16 lanes)
//   SK_MB_HBM   streaming read bandwidth (B/s): 128-bit non-allocating loads over 4 GiB
//   SK_MB_TC    tcgen05 kind::f16 MMA throughput (flop/s): the K3 kernel with the epilogue
//               skipped (measured in sk_tc.cu)
#include "sk_internal.h"
#include "sk_common.cuh"

namespace sk {

__global__ void __launch_bounds__(256) k_mb_ex2(int iters, float *sink) {
    float v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = -0.001f * (threadIdx.x + k);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = ex2(v[k]) - 1.0f;   // stays in (-1, 0]
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += v[k];
    if (s == 12345.f) sink[threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) k_mb_ffma(int iters, float *sink) {
    float2 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = make_float2(1e-3f * threadIdx.x, 1e-3f * k);
    const float2 a = make_float2(0.9999f, 0.9998f), b = make_float2(1e-4f, 2e-4f);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = fma2(v[k], a, b);
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += v[k].x + v[k].y;
    if (s == 12345.f) sink[threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) k_mb_hbm(const float4 *__restrict__ p, long long n4, float *sink) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    const long long stride = (long long)gridDim.x * blockDim.x;
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n4; i += 4 * stride) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
            asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
                         : "=f"(v[u].x), "=f"(v[u].y), "=f"(v[u].z), "=f"(v[u].w)
                         : "l"(p + i + u * stride));
#pragma unroll
        for (int u = 0; u < 4; ++u) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
    }
    for (; i < n4; i += stride) { const float4 v = p[i]; acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w; }
    if (acc.x + acc.y + acc.z + acc.w == 12345.f) sink[threadIdx.x] = acc.x;
}

cudaError_t microbench_alu(int kind, cudaStream_t st, cudaEvent_t e0, cudaEvent_t e1, float *sink,
                           double *ops) {
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int blocks = nsm * 8, iters = 4096;
    // warm-up
    if (kind == 0) k_mb_ex2<<<blocks, 256, 0, st>>>(64, sink);
    else k_mb_ffma<<<blocks, 256, 0, st>>>(64, sink);
    cudaEventRecord(e0, st);
    if (kind == 0) k_mb_ex2<<<blocks, 256, 0, st>>>(iters, sink);
    else k_mb_ffma<<<blocks, 256, 0, st>>>(iters, sink);
    cudaEventRecord(e1, st);
    *ops = (double)blocks * 256 * iters * (kind == 0 ? 8 : 16);
    return cudaGetLastError();
}

cudaError_t microbench_hbm(const float *buf, long long bytes, cudaStream_t st, cudaEvent_t e0, cudaEvent_t e1,
                           float *sink) {
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const long long n4 = bytes / 16;
    k_mb_hbm<<<nsm * 8, 256, 0, st>>>(reinterpret_cast<const float4 *>(buf), n4, sink);  // warm-up
    cudaEventRecord(e0, st);
    k_mb_hbm<<<nsm * 8, 256, 0, st>>>(reinterpret_cast<const float4 *>(buf), n4, sink);
    cudaEventRecord(e1, st);
    return cudaGetLastError();
}

}  // namespace sk
