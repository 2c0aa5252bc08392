// probe_mma_layouts.cu — tcgen05.mma (kind::f16, M=128, cta_group::1) issue throughput for the
// smem operand layouts the conv kernels use (dev tooling, not product code). Operand contents are
// zeros: only the cycles per MMA are measured, on all SMs at once (one CTA per SM).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../paper_2104_08002_b200/csrc/sm100.cuh"

using namespace c1d::sm100;

#define CK(x)                                                           \
    do {                                                                \
        cudaError_t e = (x);                                            \
        if (e != cudaSuccess) {                                         \
            printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); \
            exit(1);                                                    \
        }                                                               \
    } while (0)

struct Cfg {
    const char* name;
    uint32_t a_lbo, a_sbo, a_layout, a_mn;  // A descriptor
    uint32_t b_lbo, b_sbo, b_layout;        // B descriptor (K-major)
    uint32_t n;
    uint32_t a_step, b_step;  // start-address advance per K-step (bytes), wraps in a 64 KB window
    int nacc;                 // accumulators per K-step (different A start, same B)
    uint32_t g_step;          // A start offset between accumulators
    int unroll;               // issue 8 K-steps straight-line (no address wrap)
    int rnd;                  // random operands (else zeros)
    int d_step;               // TMEM column advance per K-step (unrolled mode), wraps at 512-N
    int g_dcol;               // TMEM column advance between accumulators (0: N, disjoint)
    int a_tmem;               // A operand from TMEM columns [384 + 8g, ...) instead of shared memory
};


__global__ void __launch_bounds__(128, 1) mma_probe(Cfg c, int ksteps, long long* cyc, int bg, const uint4* gsrc,
                                                    volatile int* stop) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_s;
    uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x) {
        uint32_t h = (i * 2654435761u) ^ (blockIdx.x * 40503u);
        uint32_t w[4];
        for (int j = 0; j < 4; ++j) {  // random bf16 pairs in [-2, 2) when c.rnd, else zeros
            h = h * 1664525u + 1013904223u;
            const uint32_t lo = 0x3f80u | ((h >> 9) & 0x7fu) | ((h >> 16) & 0x8000u);
            const uint32_t hi = 0x3f80u | ((h >> 2) & 0x7fu) | ((h << 4) & 0x8000u);
            w[j] = c.rnd ? (lo | (hi << 16)) : 0u;
        }
        reinterpret_cast<uint4*>(smem)[i] = make_uint4(w[0], w[1], w[2], w[3]);
    }
    if (threadIdx.x / 32 == 0) tmem_alloc<512>(&tmem_s);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    __shared__ int done_s;
    if (threadIdx.x == 0) done_s = 0;
    __syncthreads();
    if (threadIdx.x >= 32 && bg) {
        // background smem traffic into [144 KB, 160 KB) until the MMA thread finishes
        const uint32_t base = smem_u32(smem) + 144 * 1024;
        const int t = threadIdx.x - 32;
        uint32_t i = 0;
        while (!*reinterpret_cast<volatile int*>(&done_s)) {
            for (int r = 0; r < 16; ++r, ++i) {
                const uint32_t off = ((i * 96 + t) & 1023) * 16;
                if (bg == 1) {
                    asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(base + off), "r"(i) : "memory");
                } else {
                    cp_async16_zfill(base + off, gsrc + ((blockIdx.x * 4096 + i * 96 + t) & ((1 << 22) - 1)), true);
                }
            }
            if (bg == 2) {
                cp_async_commit();
                cp_async_wait_group<4>();
            }
            if (bg == 3) __nanosleep(200);
        }
        if (bg == 2) cp_async_wait_group<0>();
    }
    if (threadIdx.x / 32 == 0 && elect_one()) {
        const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 80 * 1024);
        const uint32_t idesc = make_idesc(128, c.n, kFmtBF16, c.a_mn, 0);
        const uint64_t a0 = make_smem_desc(sa, c.a_lbo, c.a_sbo, c.a_layout);
        const uint64_t b0 = make_smem_desc(sb, c.b_lbo, c.b_sbo, c.b_layout);
        const uint32_t tb = tmem_s;  // register copy: a shared load between MMAs waits for them
        const long long t0 = clock64();
        uint32_t ao = 0, bo = 0;
        if (c.unroll == 2) {
            // straight line: 8 MMAs per iteration, descriptors from running adds, D cycles over
            // 4 accumulators d_step apart
            for (int k = 0; k < ksteps; k += 8) {
                uint64_t a = a0, b = b0;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    mma_bf16_ss(tb + static_cast<uint32_t>((u & 3) * c.d_step), a, b, idesc, 1u);
                    a += static_cast<uint64_t>(c.a_step >> 4);
                    b += static_cast<uint64_t>(c.b_step >> 4);
                }
            }
        } else if (c.unroll) {
            const uint32_t dwrap = 512 - c.n;
            uint32_t dc = 0;
            for (int k = 0; k < ksteps; k += 8) {
#pragma unroll
                for (int u = 0; u < 8; ++u) {
#pragma unroll 1
                    for (int g = 0; g < c.nacc; ++g) {
                        if (c.a_tmem)
                            mma_bf16_ts(tb + dc + g * (c.g_dcol ? c.g_dcol : c.n), tb + 384 + 8 * (g & 7),
                                        desc_advance(b0, u * c.b_step), idesc, 1u);
                        else
                            mma_bf16_ss(tb + dc + g * (c.g_dcol ? c.g_dcol : c.n), desc_advance(a0, u * c.a_step + g * c.g_step),
                                        desc_advance(b0, u * c.b_step), idesc, 1u);
                    }
                    dc += c.d_step;
                    if (dc > dwrap) dc = 0;
                }
            }
        } else
        for (int k = 0; k < ksteps; ++k) {
#pragma unroll 1
            for (int g = 0; g < c.nacc; ++g)
                mma_bf16_ss(tb + g * c.n, desc_advance(a0, ao + g * c.g_step), desc_advance(b0, bo), idesc,
                            k > 0 ? 1u : 0u);
            ao += c.a_step;
            if (ao >= 32768) ao -= 32768;
            bo += c.b_step;
            if (bo >= 32768) bo -= 32768;
        }
        mma_commit(smem_u32(&bar));
        mbar_wait(smem_u32(&bar), 0);
        cyc[blockIdx.x] = clock64() - t0;
        *reinterpret_cast<volatile int*>(&done_s) = 1;
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x / 32 == 0) tmem_dealloc<512>(tmem_s);
}

int main() {
    const Cfg cfgs[] = {
        // wgrad v3, CP=64: A K-major none (core matrices: 8 channels x 16 B; K-chunks 1 KB apart)
        {"wgrad A Kmaj none LBO1024 SBO128 | B SW32 (N=256)", 1024, 128, kLayoutNone, 0, 16, 256, kLayoutSw32, 256,
         2048, 2048, 2, 8192},
        {"same, 1 acc", 1024, 128, kLayoutNone, 0, 16, 256, kLayoutSw32, 256, 2048, 2048, 1, 0},
        {"wgrad A | B SW128 (N=256)", 1024, 128, kLayoutNone, 0, 16, 1024, kLayoutSw128, 256, 2048, 32, 2, 8192},
        {"A Kmaj none LBO128 SBO256 | B SW32", 128, 256, kLayoutNone, 0, 16, 256, kLayoutSw32, 256, 2048, 2048, 2, 8192},
        {"A SW128 | B SW128 (GEMM)", 16, 1024, kLayoutSw128, 0, 16, 1024, kLayoutSw128, 256, 32, 32, 2, 16384},
        {"A SW32 | B SW32", 16, 256, kLayoutSw32, 0, 16, 256, kLayoutSw32, 256, 4096, 2048, 2, 8192},
        {"fwd row-tap A MN none LBO128 SBO16 | B Kmaj none", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 256, 512,
         8192, 1, 0},
        {"DSTEP N=192 same D", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 192, 512, 8192, 1, 0, 1, 1, 0},
        {"DSTEP N=192 D+64 (overlap)", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 192, 512, 8192, 1, 0, 1, 1, 64},
        {"DSTEP N=192 D+192 (disjoint)", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 192, 512, 8192, 1, 0, 1, 1, 160},
        {"DSTEP N=256 D+64 (overlap)", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 256, 512, 8192, 1, 0, 1, 1, 64},
        {"DSTEP N=64 D+64 (disjoint)", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 64, 512, 8192, 1, 0, 1, 1, 64},
        {"DSTEP N=128 D+128 (disjoint)", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 128, 512, 8192, 1, 0, 1, 1, 128},
        {"RANDOM UNROLLED wgrad 2 acc", 1024, 128, kLayoutNone, 0, 16, 256, kLayoutSw32, 256, 2048, 2048, 2, 8192, 1, 1},
        {"RANDOM GEMM SW128 2 acc", 16, 1024, kLayoutSw128, 0, 16, 1024, kLayoutSw128, 256, 32, 32, 2, 16384, 1, 1},
        {"RANDOM fwd row-tap 1 acc", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 256, 512, 8192, 1, 0, 1, 1},
        {"UNROLLED same, 1 acc", 1024, 128, kLayoutNone, 0, 16, 256, kLayoutSw32, 256, 2048, 2048, 1, 0, 1},
        {"UNROLLED wgrad 2 acc", 1024, 128, kLayoutNone, 0, 16, 256, kLayoutSw32, 256, 2048, 2048, 2, 8192, 1},
        {"UNROLLED N=112 1 acc", 256, 128, kLayoutNone, 0, 16, 1024, kLayoutSw128, 112, 512, 32, 1, 0, 1},
        {"UNROLLED N=128 1 acc", 1024, 128, kLayoutNone, 0, 16, 256, kLayoutSw32, 128, 2048, 2048, 1, 0, 1},
        {"UNROLLED N=64 1 acc", 1024, 128, kLayoutNone, 0, 16, 256, kLayoutSw32, 64, 2048, 2048, 1, 0, 1},
        // small-N forward row-tap MMAs (C = K = 15 shapes): does a disjoint accumulator per MMA beat the chain?
        {"SMALLN N=64 same D", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 64, 512, 8192, 1, 0, 1, 1, 0},
        {"SMALLN N=64 D+64", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 64, 512, 8192, 1, 0, 1, 1, 64},
        {"SMALLN N=64 D+16 (overlap)", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 64, 512, 8192, 1, 0, 1, 1, 16},
        {"SMALLN N=48 same D", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 48, 512, 8192, 1, 0, 1, 1, 0},
        {"SMALLN N=48 D+16 (overlap)", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 48, 512, 8192, 1, 0, 1, 1, 16},
        {"SMALLN N=48 D+48", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 48, 512, 8192, 1, 0, 1, 1, 48},
        {"SMALLN N=32 same D", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 32, 512, 8192, 1, 0, 1, 1, 0},
        {"SMALLN N=32 D+32", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 32, 512, 8192, 1, 0, 1, 1, 32},
        {"SMALLN N=16 same D", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 16, 512, 8192, 1, 0, 1, 1, 0},
        {"SMALLN N=16 D+16", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 16, 512, 8192, 1, 0, 1, 1, 16},
        {"SMALLN N=16 4acc D+64", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 16, 512, 8192, 4, 512, 1, 1, 64},
        {"SMALLN N=64 4acc D+256", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 64, 512, 8192, 4, 512, 1, 1, 256},
        {"SMALLN carry N=48 8acc A+256 D+16", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 48, 2048, 8192, 8, 256, 1, 1, 0, 16},
        {"SMALLN carry N=48 8acc A+256 D+48", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 48, 2048, 8192, 8, 256, 1, 1, 0, 48},
        {"SMALLN carry N=64 8acc A+256 D+16", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 64, 2048, 8192, 8, 256, 1, 1, 0, 16},
        {"SMALLN carry N=64 4acc A+256 D+64", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 64, 2048, 8192, 4, 256, 1, 1, 0, 64},
        {"SMALLN carry N=16 8acc A+256 D+16", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 16, 2048, 8192, 8, 256, 1, 1, 0, 16},
        {"SMALLN carry N=32 8acc A+256 D+32", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 32, 2048, 8192, 8, 256, 1, 1, 0, 32},
        {"SMALLN carry N=16 8acc A+256 sameD", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 16, 2048, 8192, 8, 256, 1, 1, 0, 0},
        {"SMALLN Bsame N=64 1acc A+256", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 64, 256, 0, 1, 0, 1, 1, 0},
        {"SMALLN Bsame N=16 1acc A+256", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 16, 256, 0, 1, 0, 1, 1, 0},
        {"SMALLN Bsame N=16 1acc D+16", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 16, 256, 0, 1, 0, 1, 1, 16},
        {"SMALLN TMEM-A N=16 8acc", 128, 16, kLayoutNone, 0, 128, 256, kLayoutNone, 16, 2048, 8192, 8, 256, 1, 1, 0, 16, 1},
        {"SMALLN TMEM-A N=48 8acc D+16", 128, 16, kLayoutNone, 0, 128, 256, kLayoutNone, 48, 2048, 8192, 8, 256, 1, 1, 0, 16, 1},
        {"SMALLN TMEM-A N=64 4acc", 128, 16, kLayoutNone, 0, 128, 256, kLayoutNone, 64, 2048, 8192, 4, 256, 1, 1, 0, 64, 1},
        {"SMALLN TMEM-A N=128 2acc", 128, 16, kLayoutNone, 0, 128, 256, kLayoutNone, 128, 2048, 8192, 2, 256, 1, 1, 0, 128, 1},
        {"SMALLN GEMM-A SW128 N=16 8acc", 16, 1024, kLayoutSw128, 0, 128, 256, kLayoutNone, 16, 32, 8192, 8, 16384, 1, 1, 0, 16},
        {"SMALLN GEMM-A SW128 N=48 8acc", 16, 1024, kLayoutSw128, 0, 128, 256, kLayoutNone, 48, 32, 8192, 8, 16384, 1, 1, 0, 16},
        {"SMALLN N=128 2acc D+128", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 128, 2048, 8192, 2, 256, 1, 1, 0, 128},
        {"SMALLN N=256 2acc", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 256, 2048, 8192, 2, 256, 1, 1, 0, 0},
        {"WG N=112 A CP16 | B SW128, 1acc", 256, 128, kLayoutNone, 0, 16, 1024, kLayoutSw128, 112, 512, 32, 1, 0, 1, 1, 0},
        {"WG N=112 A CP16 | B SW128, 4 copies", 256, 128, kLayoutNone, 0, 16, 1024, kLayoutSw128, 112, 512, 32, 1, 0, 1, 1, 112},
        {"WG N=112 A CP16 | B none, 4 copies", 256, 128, kLayoutNone, 0, 128, 256, kLayoutNone, 112, 512, 256, 1, 0, 1, 1, 112},
        {"WG N=64 A CP16 | B SW128, 4 copies", 256, 128, kLayoutNone, 0, 16, 1024, kLayoutSw128, 64, 512, 32, 1, 0, 1, 1, 64},
        {"WG N=128 A CP16 | B SW128, 3 copies", 256, 128, kLayoutNone, 0, 16, 1024, kLayoutSw128, 128, 512, 32, 1, 0, 1, 1, 128},
        {"WG N=224 A CP16 | B SW128, 2 copies", 256, 128, kLayoutNone, 0, 16, 1024, kLayoutSw128, 224, 512, 32, 1, 0, 1, 1, 224},
        {"WG N=112 2 groups (A+1024) 2 copies", 256, 128, kLayoutNone, 0, 16, 1024, kLayoutSw128, 112, 512, 32, 2, 1024, 1, 1, 224},
        {"SMALLN carry N=64 1acc unrolled D+16", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 64, 256, 0, 1, 0, 1, 1, 16},
        {"SMALLN carry N=64 1acc unrolled same D", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 64, 256, 0, 1, 0, 1, 1, 0},
        {"STRAIGHT N=64 4 acc, A+256 B same", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 64, 256, 0, 1, 0, 2, 1, 64},
        {"STRAIGHT N=64 4 acc, A+256 B+2048", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 64, 256, 2048, 1, 0, 2, 1, 64},
        {"STRAIGHT N=64 same D, A+256 B same", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 64, 256, 0, 1, 0, 2, 1, 0},
        {"STRAIGHT N=16 4 acc", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 16, 256, 0, 1, 0, 2, 1, 16},
        {"STRAIGHT N=128 4 acc", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 128, 256, 0, 1, 0, 2, 1, 128},
        {"STRAIGHT N=256 2 acc", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 256, 256, 0, 1, 0, 2, 1, 0},
        {"STRAIGHT WG N=112 4 copies", 256, 128, kLayoutNone, 0, 16, 1024, kLayoutSw128, 112, 512, 32, 1, 0, 2, 1, 112},
        {"STRAIGHT WG N=112 same D", 256, 128, kLayoutNone, 0, 16, 1024, kLayoutSw128, 112, 512, 32, 1, 0, 2, 1, 0},
        {"SMALLN N=128 same D", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 128, 512, 8192, 1, 0, 1, 1, 0},
        {"SMALLN N=128 D+128", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 128, 512, 8192, 1, 0, 1, 1, 128},
        {"SMALLN N=256 same D", 128, 16, kLayoutNone, 1, 128, 256, kLayoutNone, 256, 512, 8192, 1, 0, 1, 1, 0},
        {"wgrad A | B SW32, 4 acc N=128", 1024, 128, kLayoutNone, 0, 16, 256, kLayoutSw32, 128, 2048, 2048, 4, 8192},
        {"GEMM SW128, 1 acc N=256", 16, 1024, kLayoutSw128, 0, 16, 1024, kLayoutSw128, 256, 32, 32, 1, 0},
        {"wgrad A | B SW32 N=128", 1024, 128, kLayoutNone, 0, 16, 256, kLayoutSw32, 128, 2048, 2048, 2, 8192},
        {"wgrad A | B SW32 N=112", 1024, 128, kLayoutNone, 0, 16, 256, kLayoutSw32, 112, 2048, 2048, 1, 8192},
        {"A Kmaj none LBO256 SBO128 (CP=16) | B SW128 N=112", 256, 128, kLayoutNone, 0, 16, 1024, kLayoutSw128, 112,
         512, 32, 1, 8192},
    };
    long long* cyc;
    CK(cudaMalloc(&cyc, 148 * sizeof(long long)));
    CK(cudaFuncSetAttribute(mma_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 161 * 1024));
    const int ksteps = 4096;
    uint4* gsrc;
    CK(cudaMalloc(&gsrc, (size_t(1) << 22) * 16));
    CK(cudaMemset(gsrc, 0, (size_t(1) << 22) * 16));
    const char* bgname[] = {"", " +st.shared bg", " +cp.async bg"};
    const char* only = getenv("PROBE_ONLY");
    for (const Cfg& c : cfgs)
      for (int bg = 0; bg < 3; ++bg) {
        if (bg && !c.unroll) continue;
        if (only && !strstr(c.name, only)) continue;
        if (only && bg && !getenv("PROBE_BG")) continue;
        for (int grid : {148}) {
            mma_probe<<<grid, 128, 161 * 1024>>>(c, ksteps, cyc, bg, gsrc, nullptr);
            CK(cudaDeviceSynchronize());
            long long h[148];
            CK(cudaMemcpy(h, cyc, grid * sizeof(long long), cudaMemcpyDeviceToHost));
            long long mx = 0;
            for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
            const double per = static_cast<double>(mx) / (ksteps * c.nacc);
            printf("%-40s%-16s grid %3d: %6.1f cyc/MMA (ideal %5.1f)\n", c.name, bgname[bg], grid, per, 128.0 * c.n / 256.0);
        }
      }
    return 0;
}
