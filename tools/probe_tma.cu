// probe_tma.cu — TMA load throughput vs box shape on all SMs (dev tooling, not product code).
//
// Every CTA streams its own slice of a [N][C][W] bf16 tensor (the conv operands' natural layout)
// through a 4-slot smem ring: one thread issues the loads of a "stage", one thread waits for the
// stage to land and frees the slot. No compute, so the time is the copy engine's.
//   mode 0: 4-D box (8 cols, 64 ch, 8 chunks) -> q-chunk-major image (inner extent 16 B)
//   mode 1: 3-D box (16 cols, 64 ch) SWIZZLE_32B  (inner 32 B)
//   mode 2: 3-D box (32 cols, 64 ch) SWIZZLE_64B  (inner 64 B)
//   mode 3: 3-D box (64 cols, 64 ch) SWIZZLE_128B (inner 128 B)
//   mode 4: cp.async.bulk of contiguous 8 KB pieces
// Each stage moves 16 KB.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>

#include "../paper_2104_08002_b200/csrc/sm100.cuh"

using namespace c1d::sm100;

#define CK(x)                                                                  \
    do {                                                                       \
        cudaError_t e = (x);                                                   \
        if (e != cudaSuccess) {                                                \
            printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__);        \
            exit(1);                                                           \
        }                                                                      \
    } while (0)

constexpr int N = 32, C = 64, W = 60400;
constexpr int kSlots = 4, kStageBytes = 16384;

__global__ void __launch_bounds__(64, 1) probe(const __grid_constant__ CUtensorMap map, const uint16_t* g, int mode,
                                               int stages, int band, long long* cyc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint64_t full[kSlots], empty[kSlots];
    uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    if (threadIdx.x == 0) {
        for (int i = 0; i < kSlots; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const int item = blockIdx.x % N;
    const int col0 = (blockIdx.x / N) * 8192;  // 5 column bands of 8192 per item
    const long long t0 = clock64();
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            const int slot = s % kSlots;
            mbar_wait(smem_u32(&empty[slot]), ((s / kSlots) & 1) ^ 1);
            const uint32_t fb = smem_u32(&full[slot]);
            mbar_arrive_expect_tx(fb, kStageBytes);
            uint8_t* dst = smem + slot * kStageBytes;
            const int col = col0 + (s * 128) % band;  // 128 columns x 64 ch x 2 B = 16 KB per stage
            if (mode == 0) {
                for (int b = 0; b < 2; ++b)
                    asm volatile(
                        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
                        "[%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst + b * 8192)),
                        "l"(&map), "r"(0), "r"(0), "r"(col / 8 + b * 8), "r"(item), "r"(fb)
                        : "memory");
            } else if (mode >= 1 && mode <= 3) {
                const int bq = 8 << mode;  // 16, 32, 64
                const int nb = 128 / bq;
                for (int b = 0; b < nb; ++b)
                    tma_load_3d(smem_u32(dst + b * (kStageBytes / nb)), &map, col + b * bq, 0, item, fb);
            } else {
                const uint16_t* src = g + (static_cast<size_t>(item) * C) * W + col;
                for (int b = 0; b < 2; ++b)
                    bulk_g2s(smem_u32(dst + b * 8192), src + static_cast<size_t>(b) * 32 * W, 8192, fb);
            }
        }
    } else if (threadIdx.x == 32) {
        for (int s = 0; s < stages; ++s) {
            const int slot = s % kSlots;
            mbar_wait(smem_u32(&full[slot]), (s / kSlots) & 1);
            mbar_arrive(smem_u32(&empty[slot]));
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main(int argc, char** argv) {
    const int stages = argc > 1 ? atoi(argv[1]) : 512;
    const int band = argc > 2 ? atoi(argv[2]) : 8192;  // columns each CTA cycles over (L2 residency)
    printf("stages %d band %d cols\n", stages, band);
    uint16_t* g;
    const size_t bytes = static_cast<size_t>(N) * C * W * 2;
    CK(cudaMalloc(&g, bytes));
    CK(cudaMemset(g, 0, bytes));
    long long* cyc;
    CK(cudaMalloc(&cyc, 148 * sizeof(long long)));
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
    auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
    CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, kSlots * kStageBytes + 1024));
    const char* names[] = {"4d 16B-inner (L image)", "3d SW32 (16 cols)", "3d SW64 (32 cols)", "3d SW128 (64 cols)",
                           "bulk 8KB contiguous"};
    for (int mode = 0; mode < 5; ++mode) {
        CUtensorMap map{};
        CUresult r = CUDA_SUCCESS;
        if (mode == 0) {
            const cuuint64_t dims[4] = {8, C, W / 8, N};
            const cuuint64_t str[3] = {W * 2ull, 16, static_cast<cuuint64_t>(C) * W * 2};
            const cuuint32_t box[4] = {8, C, 8, 1};
            const cuuint32_t es[4] = {1, 1, 1, 1};
            r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else if (mode <= 3) {
            const cuuint64_t dims[3] = {W, C, N};
            const cuuint64_t str[2] = {W * 2ull, static_cast<cuuint64_t>(C) * W * 2};
            const cuuint32_t box[3] = {static_cast<cuuint32_t>(8 << mode), C, 1};
            const cuuint32_t es[3] = {1, 1, 1};
            const CUtensorMapSwizzle sw[] = {CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
                                             CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_SWIZZLE_128B};
            r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       sw[mode], CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        if (r != CUDA_SUCCESS) {
            printf("encode failed mode %d (%d)\n", mode, static_cast<int>(r));
            continue;
        }
        for (int rep = 0; rep < 2; ++rep) {
            cudaEvent_t a, b;
            CK(cudaEventCreate(&a));
            CK(cudaEventCreate(&b));
            CK(cudaEventRecord(a));
            probe<<<148, 64, kSlots * kStageBytes + 1024>>>(map, g, mode, stages, band, cyc);
            CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b));
            CK(cudaGetLastError());
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, a, b));
            long long h[148];
            CK(cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost));
            long long mx = 0;
            for (long long v : h) mx = v > mx ? v : mx;
            const double tot = 148.0 * stages * kStageBytes;
            if (rep)
                printf("%-26s %8.1f us  %7.1f GB/s  %6.1f B/clk/SM (max cyc %lld)\n", names[mode], ms * 1e3,
                       tot / (ms * 1e-3) / 1e9, static_cast<double>(stages) * kStageBytes / mx, mx);
        }
    }
    return 0;
}
