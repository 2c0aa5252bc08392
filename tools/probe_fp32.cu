// probe_fp32.cu — measured FP32 FFMA peak of this GPU ("There is no FP32/TF32 peak;
// measure it"). Every thread runs 8 independent FMA chains of `iters` steps; all SMs, 4 resident
// 256-thread blocks per SM; CUDA-event timing, best of 5. Prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void ffma_kernel(float* out, int iters, float a, float b) {
    float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
            x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
        }
    }
    const float s = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
    if (s == 1.2345f) out[blockIdx.x] = s;  // keep the chains live
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    float* out;
    cudaMalloc(&out, 1 << 20);
    const int blocks = sms * 4, threads = 256, iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    ffma_kernel<<<blocks, threads>>>(out, 64, 0.999f, 0.001f);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        ffma_kernel<<<blocks, threads>>>(out, iters, 0.999f, 0.001f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double flops = 2.0 * blocks * threads * static_cast<double>(iters) * 16 * 8;
    printf("{\"ffma_fp32_tflops\": %.2f, \"sms\": %d, \"max_clock_mhz\": %.0f, \"nominal_tflops\": %.2f, \"ms\": %.3f}\n",
           flops / (best * 1e-3) / 1e12, sms, clk / 1e3, 2.0 * 128 * sms * (clk / 1e6) / 1e3, best);
    return 0;
}
