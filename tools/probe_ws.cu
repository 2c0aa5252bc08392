// probe_ws.cu — tcgen05.mma.ws (weight-stationary, collector buffers for B) on sm_100a (dev tooling,
// not product code). Part 1 checks on one CTA that the ws MMA computes the same D as the regular
// MMA and that ::use / ::lastuse take B from the collector (the B descriptor is ignored). Part 2
// measures cycles per MMA on all SMs for the forward row-tap operand layout (A MN-major overlapped
// windows, B K-major), with and without the B collector.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../paper_2104_08002_b200/csrc/sm100.cuh"

using namespace c1d::sm100;

#ifndef RND
#define RND 0
#endif
#ifndef D_OVERLAP
#define D_OVERLAP 0
#endif
#define CK(x)                                                           \
    do {                                                                \
        cudaError_t e = (x);                                            \
        if (e != cudaSuccess) {                                         \
            printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); \
            exit(1);                                                    \
        }                                                               \
    } while (0)

#define WS_ASM(COLL)                                                                                     \
    __device__ __forceinline__ void ws_##COLL(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) { \
        asm volatile(                                                                                    \
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"                                           \
            "tcgen05.mma.ws.cta_group::1.kind::f16.collector::b0::" #COLL " [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d), \
            "l"(a), "l"(b), "r"(idesc), "r"(acc));                                                       \
    }
WS_ASM(fill)
WS_ASM(use)
WS_ASM(lastuse)
WS_ASM(discard)

__device__ __forceinline__ void ws_plain(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.ws.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// K-major SWIZZLE_NONE core-matrix order: element (row, k) at (row/8)*256 + (k/8)*128 + (row%8)*16 + (k%8)*2 bytes
__host__ __device__ inline int kmaj_off(int row, int k) { return (row / 8) * 128 + (k / 8) * 64 + (row % 8) * 8 + (k % 8); }

__global__ void __launch_bounds__(128, 1) ws_check(const uint16_t* a, const uint16_t* b1, const uint16_t* b2, int n,
                                                   float* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_s;
    uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    uint16_t* sa = reinterpret_cast<uint16_t*>(smem);
    uint16_t* sb1 = reinterpret_cast<uint16_t*>(smem + 8192);
    uint16_t* sb2 = reinterpret_cast<uint16_t*>(smem + 8192 + 16384);
    for (int i = threadIdx.x; i < 128 * 16; i += 128) sa[i] = a[i];
    for (int i = threadIdx.x; i < n * 16; i += 128) {
        sb1[i] = b1[i];
        sb2[i] = b2[i];
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
    const uint32_t tm = tmem_s;
    if (threadIdx.x / 32 == 0 && elect_one()) {
        const uint32_t idesc = make_idesc(128, n, kFmtBF16, 0, 0);
        const uint64_t ad = make_smem_desc(smem_u32(sa), 128, 256, kLayoutNone);
        const uint64_t bd1 = make_smem_desc(smem_u32(sb1), 128, 256, kLayoutNone);
        const uint64_t bd2 = make_smem_desc(smem_u32(sb2), 128, 256, kLayoutNone);
        mma_bf16_ss(tm + 0 * n, ad, bd1, idesc, 0);  // reference: A * B1
        ws_fill(tm + 1 * n, ad, bd1, idesc, 0);     // ws, fill collector with B1
        ws_use(tm + 2 * n, ad, bd2, idesc, 0);      // B from collector (B1) if the descriptor is ignored
        ws_lastuse(tm + 3 * n, ad, bd2, idesc, 0);  // same, then release
        ws_plain(tm + 4 * n, ad, bd2, idesc, 0);    // ws without collector: A * B2
        mma_commit(smem_u32(&bar));
    }
    __syncwarp();
    mbar_wait(smem_u32(&bar), 0);
    tc_fence_after();
    const int w = threadIdx.x / 32, l = threadIdx.x % 32;
    for (int c = 0; c < 5 * n; c += 16) {
        uint32_t r[16];
        tmem_ld16(tm + (static_cast<uint32_t>(w * 32) << 16) + c, r);
        tmem_ld_wait();
        for (int j = 0; j < 16; ++j) out[(w * 32 + l) * (5 * n) + c + j] = __uint_as_float(r[j]);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x / 32 == 0) tmem_dealloc<512>(tm);
}

// MODE: 0 regular ss; 1 ws discard each; 2 ws fill, use x(GRP-2), lastuse; 3 ws plain.
// Straight-line issue: 8 MMAs per iteration with compile-time descriptor / TMEM offsets.
template <int MODE, int N, int GRP>
__global__ void __launch_bounds__(256, 1) ws_rate(int ksteps, long long* cyc, int bg) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_s;
    uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) {
        uint32_t h = (i * 2654435761u) ^ (blockIdx.x * 40503u);
        uint32_t w[4];
        for (int j = 0; j < 4; ++j) {  // random bf16 pairs in (-2, 2) when RND, else zeros
            h = h * 1664525u + 1013904223u;
            const uint32_t lo = 0x3f80u | ((h >> 9) & 0x7fu) | ((h >> 16) & 0x8000u);
            const uint32_t hi = 0x3f80u | ((h >> 2) & 0x7fu) | ((h << 4) & 0x8000u);
            w[j] = RND ? (lo | (hi << 16)) : 0u;
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
    if (threadIdx.x >= 128 && bg) {
        // background TMEM traffic on columns [256, 512) (the MMAs use [0, 256)) until the MMAs finish
        const int w = (threadIdx.x / 32) & 3;
        const uint32_t ta = tmem_s + (static_cast<uint32_t>(w * 32) << 16) + 256;
        uint32_t r[16] = {};
        int it = 0;
        while (!*reinterpret_cast<volatile int*>(&done_s)) {
            for (int j = 0; j < 16; ++j) {
                if (bg == 1) {
                    tmem_ld16(ta + ((it * 16) & 255), r);
                    tmem_ld_wait();
                } else if (bg == 2) {
                    tmem_st16(ta + ((it * 16) & 255), r);
                    tmem_st_wait();
                } else {
                    __nanosleep(100);
                }
                ++it;
            }
            if (bg == 1 && r[3] == 12345u) done_s = 2;
        }
    }
    if (threadIdx.x / 32 == 0 && elect_one()) {
        const uint32_t tb = tmem_s;
        // forward row-tap A: MN-major none, LBO 128 (K groups), SBO 16 (M groups), overlapped rows
        const uint64_t a0 = make_smem_desc(smem_u32(smem), 128, 16, kLayoutNone);
        const uint64_t b0 = make_smem_desc(smem_u32(smem + 64 * 1024), 128, 256, kLayoutNone);
        const uint32_t idesc = make_idesc(128, N, kFmtBF16, 1, 0);
        constexpr int kSlots = 512 / N;
        const long long t0 = clock64();
        for (int k = 0; k < ksteps; k += GRP) {
#pragma unroll
            for (int u = 0; u < GRP; ++u) {
                const uint64_t a = a0 + static_cast<uint64_t>((u & 15) * 16);  // +256 B per MMA
                const uint32_t d = tb + static_cast<uint32_t>((u % kSlots) * (D_OVERLAP ? 16 : N)) % 256;
                if (MODE == 0) {
                    mma_bf16_ss(d, a, b0, idesc, 1);
                } else if (MODE == 1) {
                    ws_discard(d, a, b0, idesc, 1);
                } else if (MODE == 3) {
                    ws_plain(d, a, b0, idesc, 1);
                } else {
                    if (u == 0) ws_fill(d, a, b0, idesc, 1);
                    else if (u == GRP - 1) ws_lastuse(d, a, b0, idesc, 1);
                    else ws_use(d, a, b0, idesc, 1);
                }
            }
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

// The forward kernel's narrow-layer MMA pattern (config 2): per super-tile, for each of 15
// channels a run over tiles 3..7, then for each channel a run over tiles 0..2; A of (channel c,
// tile t) at c*2560 + t*256 B, B of channel c at 64 KB + c*2048 B, D at region + 16*t (N = 64),
// region alternating 0 / 256. WS: 1 = ws fill/use/lastuse runs, 0 = regular MMAs.
template <int WS>
__global__ void __launch_bounds__(256, 1) kpattern(int supers, long long* cyc, const uint8_t* gsrc, int bg_bytes) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_s;
    uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x / 32 == 0) tmem_alloc<512>(&tmem_s);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    __shared__ int done_k;
    __shared__ uint64_t bgbar;
    if (threadIdx.x == 0) {
        done_k = 0;
        mbar_init(&bgbar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 32 && bg_bytes > 0) {
        // background bulk copies (like the producer's TMA loads): bg_bytes per ~1000 cycles into
        // [120 KB, 150 KB)
        uint32_t ph = 0;
        long long t_next = clock64();
        int i = 0;
        while (!*reinterpret_cast<volatile int*>(&done_k)) {
            while (clock64() < t_next) {}
            t_next += 1000;
            mbar_arrive_expect_tx(smem_u32(&bgbar), static_cast<uint32_t>(bg_bytes));
            bulk_g2s(smem_u32(smem + 120 * 1024), gsrc + (static_cast<size_t>(blockIdx.x * 64 + (i++ & 63)) << 15),
                     static_cast<uint32_t>(bg_bytes), smem_u32(&bgbar));
            mbar_wait(smem_u32(&bgbar), ph);
            ph ^= 1;
        }
    }
    if (threadIdx.x / 32 == 0 && elect_one()) {
        const uint32_t tb = tmem_s;
        const uint64_t a0 = make_smem_desc(smem_u32(smem), 128, 16, kLayoutNone);
        const uint64_t b0 = make_smem_desc(smem_u32(smem + 64 * 1024), 128, 256, kLayoutNone);
        const uint32_t idesc = make_idesc(128, 64, kFmtBF16, 1, 0);
        const long long t0 = clock64();
        for (int sidx = 0; sidx < supers; ++sidx) {
            const uint32_t region = (sidx & 1) ? 256u : 0u;
            for (int part = 0; part < 2; ++part) {
                const int t0r = part == 0 ? 3 : 0;
                for (int c = 0; c < 15; ++c) {
                    const uint64_t ac = a0 + static_cast<uint64_t>((c * 2560 + t0r * 256) >> 4);
                    const uint64_t bc = b0 + static_cast<uint64_t>((c * 2048) >> 4);
                    const uint32_t dc = tb + region + 16u * t0r;
                    if (part == 0) {
#pragma unroll
                        for (int t = 0; t < 5; ++t) {
                            const uint64_t a = ac + static_cast<uint64_t>(t * 16);
                            const uint32_t d = dc + 16u * t;
                            if (!WS) mma_bf16_ss(d, a, bc, idesc, 1);
                            else if (t == 0) ws_fill(d, a, bc, idesc, 1);
                            else if (t == 4) ws_lastuse(d, a, bc, idesc, 1);
                            else ws_use(d, a, bc, idesc, 1);
                        }
                    } else {
#pragma unroll
                        for (int t = 0; t < 3; ++t) {
                            const uint64_t a = ac + static_cast<uint64_t>(t * 16);
                            const uint32_t d = dc + 16u * t;
                            if (!WS) mma_bf16_ss(d, a, bc, idesc, 1);
                            else if (t == 0) ws_fill(d, a, bc, idesc, 1);
                            else if (t == 2) ws_lastuse(d, a, bc, idesc, 1);
                            else ws_use(d, a, bc, idesc, 1);
                        }
                    }
                }
            }
        }
        mma_commit(smem_u32(&bar));
        mbar_wait(smem_u32(&bar), 0);
        cyc[blockIdx.x] = clock64() - t0;
        *reinterpret_cast<volatile int*>(&done_k) = 1;
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x / 32 == 0) tmem_dealloc<512>(tmem_s);
}

template <int WS>
void run_kpattern(const char* name, long long* cyc, int bg_bytes = 0) {
    static uint8_t* gsrc = nullptr;
    if (!gsrc) {
        CK(cudaMalloc(&gsrc, size_t(148) * 64 * 32768 + 65536));
        CK(cudaMemset(gsrc, 0, size_t(148) * 64 * 32768 + 65536));
    }
    const int supers = 64;
    CK(cudaFuncSetAttribute(kpattern<WS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    for (int rep = 0; rep < 2; ++rep) {
        kpattern<WS><<<148, 256, 160 * 1024>>>(supers, cyc, gsrc, bg_bytes);
        CK(cudaDeviceSynchronize());
    }
    long long h[148];
    CK(cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost));
    long long mx = 0;
    for (long long v : h) mx = v > mx ? v : mx;
    printf("%-26s bg %5d B/kcyc: %6.1f cyc/MMA\n", name, bg_bytes, static_cast<double>(mx) / (supers * 120));
}

template <int MODE, int N, int GRP>
void run_rate(const char* name, long long* cyc, int bg = 0) {
    const int ksteps = 8192;
    CK(cudaFuncSetAttribute(ws_rate<MODE, N, GRP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 97 * 1024));
    for (int rep = 0; rep < 2; ++rep) {
        ws_rate<MODE, N, GRP><<<148, 256, 97 * 1024>>>(ksteps, cyc, bg);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("%-24s: %s\n", name, cudaGetErrorString(e));
            exit(1);
        }
    }
    long long h[148];
    CK(cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost));
    long long mx = 0;
    for (long long v : h) mx = v > mx ? v : mx;
    printf("%-26s bg%d: %6.1f cyc/MMA (math floor %5.1f)\n", name, bg, static_cast<double>(mx) / ksteps, 128.0 * N / 256.0);
}

static uint16_t f2bf(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    return static_cast<uint16_t>(u >> 16);
}

int main() {
    // ---- part 1: correctness
    for (int n : {64, 128, 256}) {
        uint16_t ha[128 * 16], hb1[256 * 16], hb2[256 * 16];
        float A[128][16], B1[256][16], B2[256][16];
        srand(1234 + n);
        for (int m = 0; m < 128; ++m)
            for (int k = 0; k < 16; ++k) {
                A[m][k] = static_cast<float>(rand() % 7 - 3);
                ha[kmaj_off(m, k)] = f2bf(A[m][k]);
            }
        for (int r = 0; r < n; ++r)
            for (int k = 0; k < 16; ++k) {
                B1[r][k] = static_cast<float>(rand() % 7 - 3);
                B2[r][k] = static_cast<float>(rand() % 5 - 2);
                hb1[kmaj_off(r, k)] = f2bf(B1[r][k]);
                hb2[kmaj_off(r, k)] = f2bf(B2[r][k]);
            }
        uint16_t *da, *db1, *db2;
        float* dout;
        const int ncol = 5 * n;
        if (ncol > 512) {
            printf("N=%d: skipped (needs %d columns)\n", n, ncol);
            continue;
        }
        CK(cudaMalloc(&da, sizeof(ha)));
        CK(cudaMalloc(&db1, sizeof(hb1)));
        CK(cudaMalloc(&db2, sizeof(hb2)));
        CK(cudaMalloc(&dout, 128 * ncol * 4));
        CK(cudaMemcpy(da, ha, sizeof(ha), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(db1, hb1, sizeof(hb1), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(db2, hb2, sizeof(hb2), cudaMemcpyHostToDevice));
        CK(cudaFuncSetAttribute(ws_check, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
        ws_check<<<1, 128, 64 * 1024>>>(da, db1, db2, n, dout);
        CK(cudaDeviceSynchronize());
        static float out[128 * 1280];
        CK(cudaMemcpy(out, dout, 128 * ncol * 4, cudaMemcpyDeviceToHost));
        const char* names[5] = {"ss A*B1", "ws fill(B1)", "ws use(desc B2)", "ws lastuse(desc B2)", "ws plain(B2)"};
        for (int t = 0; t < 5; ++t) {
            int ok1 = 0, ok2 = 0, tot = 0;
            for (int m = 0; m < 128; ++m)
                for (int j = 0; j < n; ++j) {
                    float r1 = 0, r2 = 0;
                    for (int k = 0; k < 16; ++k) {
                        r1 += A[m][k] * B1[j][k];
                        r2 += A[m][k] * B2[j][k];
                    }
                    const float v = out[m * ncol + t * n + j];
                    ok1 += v == r1;
                    ok2 += v == r2;
                    ++tot;
                }
            printf("N=%3d %-22s matches A*B1 %5d/%d  A*B2 %5d/%d\n", n, names[t], ok1, tot, ok2, tot);
        }
        cudaFree(da);
        cudaFree(db1);
        cudaFree(db2);
        cudaFree(dout);
    }
    // ---- part 2: rates
    long long* cyc;
    CK(cudaMalloc(&cyc, 148 * sizeof(long long)));
    run_kpattern<0>("kernel pattern ss", cyc);
    run_kpattern<1>("kernel pattern ws", cyc);
    for (int bgb : {2048, 4096, 8192, 16384}) run_kpattern<1>("kernel pattern ws", cyc, bgb);
    run_rate<0, 64, 8>("ss N=64", cyc);
    run_rate<3, 64, 8>("ws plain N=64", cyc);
    run_rate<1, 64, 8>("ws discard N=64", cyc);
    run_rate<2, 64, 8>("ws fill/use x8 N=64", cyc);
    run_rate<2, 64, 16>("ws fill/use x16 N=64", cyc);
    run_rate<0, 128, 8>("ss N=128", cyc);
    run_rate<3, 128, 8>("ws plain N=128", cyc);
    run_rate<2, 128, 8>("ws fill/use x8 N=128", cyc);
    for (int bg = 1; bg <= 3; ++bg) {
        run_rate<0, 64, 8>("ss N=64", cyc, bg);
        run_rate<2, 64, 8>("ws fill/use x8 N=64", cyc, bg);
        run_rate<0, 256, 8>("ss N=256", cyc, bg);
    }
    run_rate<0, 256, 8>("ss N=256", cyc);
    run_rate<3, 256, 8>("ws plain N=256", cyc);
    run_rate<2, 256, 8>("ws fill/use x8 N=256", cyc);
    return 0;
}
