// Legacy warp-level MMA (mma.sync.m16n8k16 f16 -> f32, SASS HMMA) throughput on sm_100a:
// every warp issues N independent accumulator chains; reports HMMA per SM per cycle and
// dense TFLOP/s.  Informs whether a decode kernel with 1-4 useful rows per m16 tile can
// use it.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 hmma_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int CH>
__global__ void hmma_loop(float* out, int iters) {
    uint32_t a0 = threadIdx.x, a1 = a0 * 3u, a2 = a0 * 5u, a3 = a0 * 7u, b0 = a0 ^ 0x3c00u, b1 = a0 ^ 0x3800u;
    float d[CH][4];
#pragma unroll
    for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = d[c][2] = d[c][3] = 0.f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                         "{%0,%1,%2,%3};"
                         : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
    if (s == 12345.f) out[threadIdx.x] = s;
}

template <int CH>
void run(int warps_per_cta, int ctas_per_sm, int sms, int clk_khz) {
    float* out;
    cudaMalloc(&out, 4096);
    const int iters = 4096;
    dim3 grid(sms * ctas_per_sm), block(32 * warps_per_cta);
    hmma_loop<CH><<<grid, block>>>(out, 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    hmma_loop<CH><<<grid, block>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double n = (double)grid.x * warps_per_cta * iters * CH;  // HMMA instructions
    const double cyc = ms * 1e-3 * clk_khz * 1e3;
    printf("{\"chains\": %d, \"warps_per_sm\": %d, \"ms\": %.3f, \"hmma_per_sm_per_clk\": %.3f, \"tflops\": %.1f}\n", CH,
           warps_per_cta * ctas_per_sm, ms, n / sms / cyc, n * 4096.0 * 2 / (ms * 1e-3) / 1e12);
    cudaFree(out);
}

int main() {
    int sms, clk;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    run<1>(4, 1, sms, clk);
    run<4>(4, 1, sms, clk);
    run<8>(4, 1, sms, clk);
    run<4>(8, 2, sms, clk);
    run<8>(8, 2, sms, clk);
    run<8>(16, 2, sms, clk);
    return 0;
}
