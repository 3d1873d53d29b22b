// Throughput of MUFU.EX2 in f32 vs f16x2 (and the f16x2 -> f32 conversions) on one B200.
#include <cstdio>
#include <cuda_fp16.h>
__global__ void k_f32(float *out, int iters) {
    float a0 = threadIdx.x * 1e-3f, a1 = a0 + 0.1f, a2 = a0 + 0.2f, a3 = a0 + 0.3f;
    float s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    for (int i = 0; i < iters; ++i) {
        float r0, r1, r2, r3;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r0) : "f"(a0));
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r1) : "f"(a1));
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r2) : "f"(a2));
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r3) : "f"(a3));
        s0 += r0; s1 += r1; s2 += r2; s3 += r3;
        a0 -= 1e-6f; a1 -= 1e-6f; a2 -= 1e-6f; a3 -= 1e-6f;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3;
}
__global__ void k_f16x2(float *out, int iters) {
    __half2 a0 = __floats2half2_rn(threadIdx.x * 1e-3f, 0.05f), a1 = __floats2half2_rn(0.1f, 0.15f);
    __half2 a2 = __floats2half2_rn(0.2f, 0.25f), a3 = __floats2half2_rn(0.3f, 0.35f);
    __half2 d = __floats2half2_rn(-1e-3f, -1e-3f);
    __half2 s0 = __floats2half2_rn(0, 0), s1 = s0, s2 = s0, s3 = s0;
    for (int i = 0; i < iters; ++i) {
        unsigned r0, r1, r2, r3;
        asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(r0) : "r"(*(unsigned *)&a0));
        asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(r1) : "r"(*(unsigned *)&a1));
        asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(r2) : "r"(*(unsigned *)&a2));
        asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(r3) : "r"(*(unsigned *)&a3));
        s0 = __hadd2(s0, *(__half2 *)&r0); s1 = __hadd2(s1, *(__half2 *)&r1);
        s2 = __hadd2(s2, *(__half2 *)&r2); s3 = __hadd2(s3, *(__half2 *)&r3);
        a0 = __hadd2(a0, d); a1 = __hadd2(a1, d); a2 = __hadd2(a2, d); a3 = __hadd2(a3, d);
    }
    float2 f = __half22float2(__hadd2(__hadd2(s0, s1), __hadd2(s2, s3)));
    out[blockIdx.x * blockDim.x + threadIdx.x] = f.x + f.y;
}
int main() {
    float *o; cudaMalloc(&o, 148 * 8 * 1024 * 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 4096, blocks = 148 * 8, nt = 256;
    for (int rep = 0; rep < 2; ++rep) {
        float ms;
        cudaEventRecord(e0); k_f32<<<blocks, nt>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double n32 = 4.0 * iters * blocks * nt;
        printf("f32   ex2: %.3f ms  %.3e values/s  %.2f values/clk/SM @1965\n", ms, n32 / (ms * 1e-3), n32 / (ms * 1e-3) / 148 / 1.965e9);
        cudaEventRecord(e0); k_f16x2<<<blocks, nt>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double n16 = 8.0 * iters * blocks * nt;
        printf("f16x2 ex2: %.3f ms  %.3e values/s  %.2f values/clk/SM @1965\n", ms, n16 / (ms * 1e-3), n16 / (ms * 1e-3) / 148 / 1.965e9);
    }
    return 0;
}
