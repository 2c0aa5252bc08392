// probe_store.cu — per-SM global store throughput for the tc_conv epilogue pattern (dev tooling).
// Each CTA writes `tiles` tiles of 128 columns x 64 channel rows (fp32) into a [rows][W] tensor:
// 4 warps, warp w owns columns 32w..32w+31, one 128-B warp store per (channel row, tile).
// Variants: scalar 4-B stores (the current epilogue), 16-B vector stores after an in-register
// 4x4 transpose (each lane writes 4 columns of one row), and the store count alone.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                           \
    do {                                                                \
        cudaError_t e = (x);                                            \
        if (e != cudaSuccess) {                                         \
            printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); \
            exit(1);                                                    \
        }                                                               \
    } while (0)

constexpr int W = 60000, ROWS_PER_ITEM = 64, ITEMS = 32;

__global__ void __launch_bounds__(512) store_probe(float* out, int tiles, int mode, long long* cyc) {
    const int nw = blockDim.x / 32;  // warps split the 64 rows
    const int warp = (threadIdx.x / 32) % 4, lane = threadIdx.x % 32, rgrp = threadIdx.x / 128;
    const int item = blockIdx.x % ITEMS;
    const int tile0 = (blockIdx.x / ITEMS) * tiles;
    float* base = out + static_cast<size_t>(item) * ROWS_PER_ITEM * W;
    __syncthreads();
    const long long t0 = clock64();
    for (int t = 0; t < tiles; ++t) {
        const int q = (tile0 + t) * 128 + warp * 32 + lane;
        if (mode == 0) {
            for (int k = rgrp; k < ROWS_PER_ITEM; k += nw / 4) base[static_cast<size_t>(k) * W + q] = static_cast<float>(k + t);
        } else {
            // lane l writes row (k0 + l/8 ... ) : 8 lanes x 16 B = 128 B per row, 4 rows per store
            const int r = lane / 8, c4 = (lane % 8) * 4;
            const int qb = (tile0 + t) * 128 + warp * 32 + c4;
#pragma unroll 4
            for (int k = 0; k < ROWS_PER_ITEM; k += 4) {
                float4 v = make_float4(k, k + 1, k + 2, t);
                *reinterpret_cast<float4*>(base + static_cast<size_t>(k + r) * W + qb) = v;
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main() {
    float* out;
    CK(cudaMalloc(&out, sizeof(float) * static_cast<size_t>(ITEMS) * ROWS_PER_ITEM * W));
    long long* cyc;
    CK(cudaMalloc(&cyc, 148 * sizeof(long long)));
    for (int threads : {128})
    for (int mode = 0; mode < 1; ++mode)
        for (int grid : {8, 37, 74, 148}) {
            const int tiles = 5;
            for (int rep = 0; rep < 2; ++rep) {
                store_probe<<<grid, threads>>>(out, tiles, mode, cyc);
                CK(cudaDeviceSynchronize());
            }
            long long h[148];
            CK(cudaMemcpy(h, cyc, grid * sizeof(long long), cudaMemcpyDeviceToHost));
            long long mx = 0, sum = 0;
            for (int i = 0; i < grid; ++i) {
                mx = h[i] > mx ? h[i] : mx;
                sum += h[i];
            }
            const double bytes = 5.0 * 128 * 64 * 4;
            printf("threads %d ", threads);
            printf("%s grid %3d: avg %.0f cycles per 5 tiles (%.1f B/clk/SM), max %lld\n",
                   mode == 0 ? "scalar 4B stores  " : "vector 16B stores ", grid, static_cast<double>(sum) / grid,
                   bytes / (static_cast<double>(sum) / grid), mx);
        }
    return 0;
}
