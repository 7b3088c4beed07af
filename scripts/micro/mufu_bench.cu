// Microbenchmark: MUFU.EX2 (fp32) and F2FP/FFMA throughput per SM on this GPU.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void ex2_kernel(float* out, int iters, float seed) {
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = seed * (threadIdx.x + i) * 1e-6f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            float y;
            asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[i]));
            x[i] = y * -0.5f;
        }
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.f) out[0] = s;
}

__global__ void ffma_kernel(float* out, int iters, float seed) {
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = seed * (threadIdx.x + i);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], 0.999f, 0.001f);
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.f) out[0] = s;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float* out;
    cudaMalloc(&out, 4);
    for (int threads : {128, 256, 512, 1024}) {
        const int iters = 4096;
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        ex2_kernel<<<sms * 2, threads>>>(out, 16, 1.f);
        cudaEventRecord(a);
        ex2_kernel<<<sms * 2, threads>>>(out, iters, 1.f);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        double ops = (double)sms * 2 * threads * iters * 8;
        double per_clk_sm = ops / (ms * 1e-3) / sms / (clk * 1e3);
        cudaEventRecord(a);
        ffma_kernel<<<sms * 2, threads>>>(out, iters, 1.f);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms2;
        cudaEventElapsedTime(&ms2, a, b);
        double per_clk_sm2 = ops / (ms2 * 1e-3) / sms / (clk * 1e3);
        printf("threads/CTA %4d (2 CTAs/SM): ex2 %.1f /clk/SM (at nominal %d MHz)   ffma %.1f /clk/SM\n", threads,
               per_clk_sm, clk / 1000, per_clk_sm2);
    }
    return 0;
}
