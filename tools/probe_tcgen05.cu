// probe_tcgen05.cu — hardware probe for the UMMA operand layouts the conv1d kernels rely on.
//
// Dev tooling, not product code. It checks on a real B200:
//   1. SS MMA with an MN-major SWIZZLE_NONE "row = tap" A operand read straight out of a natural
//      (contiguous) bf16 row: element (m, r) at byte 2*m + 16*r, i.e. M-group stride 16 B and
//      K-group stride 128 B (core matrices overlap in memory). Both LBO/SBO assignments are run.
//   2. TS MMA (A from TMEM) and the bf16 packing order of an A row in TMEM columns.
//   3. SS MMA with a K-major SWIZZLE_128B B operand (the TMA 128B-swizzle image), K advanced
//      inside the 128 B row by moving the start address.
//   4. Issue-to-completion throughput (cycles per MMA) of the shapes the kernels use.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2104_08002_b200/csrc/sm100.cuh"

using namespace c1d::sm100;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

static uint16_t f2bf(float f) { uint32_t u; memcpy(&u, &f, 4); u += 0x7fffu + ((u >> 16) & 1u); return (uint16_t)(u >> 16); }
static float bf2f(uint16_t b) { uint32_t u = (uint32_t)b << 16; float f; memcpy(&f, &u, 4); return f; }

// mode: 0 = SS row-tap A (MN-major none) x B K-major none, N=n
//       1 = TS A (tmem) x B K-major none
//       2 = SS A K-major none (K=64, 4 steps) x B K-major SW128
struct Params {
    int mode, n, a_swap, b_swap, reps, ts_pack_hi_first, nacc, vary, dcol, split;
};

__global__ void __launch_bounds__(128, 1) probe_kernel(Params p, const uint16_t* gx, const uint16_t* gw,
                                                       const uint16_t* ga, float* gd, long long* cycles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base_s;
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    uint8_t* base = smem + ((1024 - (smem_u32(smem) & 1023)) & 1023);
    uint8_t* sx = base;              // row for A (mode 0) or K-major A (mode 2: 128x64 bf16=16KB)
    uint8_t* sb = base + 32768;      // B operand
    if (warp == 0) tmem_alloc<512>(&tmem_base_s);
    if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    // ---- fill smem
    if (p.mode == 0) {
        for (int i = tid; i < 1024; i += 128) reinterpret_cast<uint16_t*>(sx)[i] = gx[i & 511];
    } else if (p.mode == 2) {
        // A K-major interleave: 128 rows x 64 k; addr = (m/8)*1024 + (k/8)*128 + (m%8)*16 + (k%8)*2
        for (int i = tid; i < 128 * 64; i += 128) {
            int m = i / 64, k = i % 64;
            int off = (m / 8) * 1024 + (k / 8) * 128 + (m % 8) * 16 + (k % 8) * 2;
            *reinterpret_cast<uint16_t*>(sx + off) = ga[i];
        }
    }
    if (p.mode == 3) {
        // A K-major SW64: 128 rows x 32 k, row = 64 B, 8-row atoms of 512 B, 16B chunk XOR (row%8)>>1... write generic pattern
        for (int i = tid; i < 128 * 32; i += 128) {
            int m = i / 32, k = i % 32;
            int chunk = (k / 8) ^ ((m % 8) >> 1);  // SW64: XOR 16B-chunk index (2 bits) with row bits
            int off = (m / 8) * 512 + (m % 8) * 64 + chunk * 16 + (k % 8) * 2;
            *reinterpret_cast<uint16_t*>(sx + off) = ga[(m * 32 + k) % (128 * 64)];
        }
        // B: 256 rows, K = 16; interleave; fill a 16 KB region with a pattern (timing only)
        for (int i = tid; i < 8192; i += 128) reinterpret_cast<uint16_t*>(sb)[i] = gw[i % (256 * 64)];
    }
    if (p.mode == 0 || p.mode == 1) {
        // B K-major interleave: n rows x 16 k; addr = (n/8)*256 + (k/8)*128 + (n%8)*16 + (k%8)*2
        for (int i = tid; i < p.n * 16; i += 128) {
            int n = i / 16, k = i % 16;
            int off = (n / 8) * 256 + (k / 8) * 128 + (n % 8) * 16 + (k % 8) * 2;
            *reinterpret_cast<uint16_t*>(sb + off) = gw[i];
        }
    } else {
        // B K-major SW128: n rows x 64 k, row = 128 B, 8-row atoms of 1024 B, 16B chunk XOR row%8
        for (int i = tid; i < p.n * 64; i += 128) {
            int n = i / 64, k = i % 64;
            int chunk = (k / 8) ^ (n % 8);
            int off = (n / 8) * 1024 + (n % 8) * 128 + chunk * 16 + (k % 8) * 2;
            *reinterpret_cast<uint16_t*>(sb + off) = gw[i];
        }
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = tmem_base_s;
    const uint32_t tA = tbase + 496;  // A operand columns for TS (cols 496..503)
    if (p.mode == 1) {
        // each thread = lane row m = tid; A[m][k] for k=0..15 -> 8 cols
        uint32_t r[8];
        for (int j = 0; j < 8; ++j) {
            uint16_t e0 = ga[tid * 16 + 2 * j], e1 = ga[tid * 16 + 2 * j + 1];
            r[j] = p.ts_pack_hi_first ? pack_bf16x2(e1, e0) : pack_bf16x2(e0, e1);
        }
        tmem_st8(tA + ((uint32_t)(warp * 32) << 16), r);
        tmem_st_wait();
        tc_fence_before();
    }
    __syncthreads();
    long long t0 = 0, t1 = 0;
    if (tid == 0) {
        tc_fence_after();
        const uint32_t sxa = smem_u32(sx), sba = smem_u32(sb);
        uint32_t idesc;
        uint64_t adesc = 0, bdesc;
        if (p.mode == 0) {
            idesc = make_idesc(128, p.n, kFmtBF16, /*a MN*/ 1, /*b K*/ 0);
            adesc = p.a_swap ? make_smem_desc(sxa + 2 * 8, 16, 128, kLayoutNone)
                             : make_smem_desc(sxa + 2 * 8, 128, 16, kLayoutNone);  // start at q0 = 8
            bdesc = p.b_swap ? make_smem_desc(sba, 256, 128, kLayoutNone) : make_smem_desc(sba, 128, 256, kLayoutNone);
        } else if (p.mode == 1) {
            idesc = make_idesc(128, p.n, kFmtBF16, 0, 0);
            bdesc = p.b_swap ? make_smem_desc(sba, 256, 128, kLayoutNone) : make_smem_desc(sba, 128, 256, kLayoutNone);
        } else if (p.mode == 2) {
            idesc = make_idesc(128, p.n, kFmtBF16, 0, 0);
            adesc = p.a_swap ? make_smem_desc(sxa, 1024, 128, kLayoutNone) : make_smem_desc(sxa, 128, 1024, kLayoutNone);
            bdesc = make_smem_desc(sba, 16, 1024, kLayoutSw128);
        } else {
            idesc = make_idesc(128, p.n, kFmtBF16, 0, 0);
            adesc = make_smem_desc(sxa, 16, 512, kLayoutSw64);
            bdesc = p.a_swap ? make_smem_desc(sba, 1024, 128, kLayoutNone) : make_smem_desc(sba, 128, 256, kLayoutNone);
        }
        t0 = clock64();
        const uint32_t nstep = (uint32_t)p.n;
        uint32_t vi = 0;
        auto issue = [&](uint32_t dcol, uint32_t accf) {
            if (p.mode == 3) {
                vi = (vi + 1) & 3;
                mma_bf16_ss(dcol, desc_advance(adesc, (vi & 1) * 32), desc_advance(bdesc, p.vary ? vi * 2048 : 0), idesc, accf);
            } else if (p.mode == 0) {
                if (p.split) {
                    vi = (vi + 1) & 3;
                    const uint64_t ad = desc_advance(adesc, vi * 256);
                    const uint32_t n1 = (uint32_t)p.split, n2 = 256 - n1;
                    if (p.split > 0 && p.vary == 2) {
                        mma_bf16_ss_afill(tbase + p.dcol, ad, bdesc, make_idesc(128, n1, kFmtBF16, 1, 0), accf);
                        mma_bf16_ss_alastuse(tbase + p.dcol + n1, ad, desc_advance(bdesc, n1 * 32), make_idesc(128, n2, kFmtBF16, 1, 0), accf);
                    } else {
                        mma_bf16_ss(tbase + p.dcol, ad, bdesc, make_idesc(128, n1, kFmtBF16, 1, 0), accf);
                        mma_bf16_ss(tbase + p.dcol + n1, ad, desc_advance(bdesc, n1 * 32), make_idesc(128, n2, kFmtBF16, 1, 0), accf);
                    }
                } else if (p.vary) {
                    vi = (vi + 1) & 3;
                    mma_bf16_ss(dcol + p.dcol, desc_advance(adesc, vi * 256), desc_advance(bdesc, (vi & 1) * 8192), idesc, accf);
                } else {
                    mma_bf16_ss(dcol + p.dcol, adesc, bdesc, idesc, accf);
                }
            }
            else if (p.mode == 1) mma_bf16_ts(dcol, tA, bdesc, idesc, accf);
            else {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                    mma_bf16_ss(dcol, desc_advance(adesc, kk * 256), desc_advance(bdesc, kk * 32), idesc, (accf || kk > 0));
            }
        };
        switch (p.nacc) {
#define ROUND(NA) case NA: { \
            _Pragma("unroll") for (int a = 0; a < NA; ++a) issue(tbase + a * nstep, 0); \
            for (int it = NA; it < p.reps; it += NA) { _Pragma("unroll") for (int a = 0; a < NA; ++a) issue(tbase + a * nstep, 1); } \
            break; }
            ROUND(1) ROUND(2) ROUND(4) ROUND(7)
#undef ROUND
        }
        mma_commit(smem_u32(&bar));
        mbar_wait(smem_u32(&bar), 0);
        t1 = clock64();
        cycles[0] = t1 - t0;
    }
    __syncthreads();
    tc_fence_after();
    // read D: 128 lanes x n cols
    for (int c0 = 0; c0 < p.n; c0 += 16) {
        uint32_t r[16];
        tmem_ld16(tbase + ((uint32_t)(warp * 32) << 16) + ((c0 + (uint32_t)p.dcol) & 511), r);
        tmem_ld_wait();
        for (int j = 0; j < 16; ++j) gd[tid * 256 + c0 + j] = __uint_as_float(r[j]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tbase);
}

int main() {
    int dev = 0;
    CK(cudaSetDevice(dev));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, dev));
    printf("device %s sm_%d%d SMs=%d clock=%d kHz\n", prop.name, prop.major, prop.minor, prop.multiProcessorCount, prop.clockRate);
    srand(1234);
    std::vector<uint16_t> hx(512), hw(256 * 64), ha(128 * 64);
    for (auto& v : hx) v = f2bf((rand() % 17 - 8) / 8.0f);
    for (auto& v : hw) v = f2bf((rand() % 17 - 8) / 8.0f);
    for (auto& v : ha) v = f2bf((rand() % 17 - 8) / 8.0f);
    uint16_t *dx, *dw, *da; float* dd; long long* dc;
    CK(cudaMalloc(&dx, 512 * 2)); CK(cudaMalloc(&dw, hw.size() * 2)); CK(cudaMalloc(&da, ha.size() * 2));
    CK(cudaMalloc(&dd, 128 * 256 * 4)); CK(cudaMalloc(&dc, 8));
    CK(cudaMemcpy(dx, hx.data(), 512 * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dw, hw.data(), hw.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(da, ha.data(), ha.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
    std::vector<float> hd(128 * 256);
    auto run = [&](Params p, const char* name) {
        CK(cudaMemset(dd, 0, 128 * 256 * 4));
        probe_kernel<<<1, 128, 96 * 1024>>>(p, dx, dw, da, dd, dc);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("%s: CUDA error %s\n", name, cudaGetErrorString(e)); exit(2); }
        long long cyc; CK(cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(hd.data(), dd, hd.size() * 4, cudaMemcpyDeviceToHost));
        double maxerr = 0, maxref = 0;
        for (int m = 0; m < 128; ++m)
            for (int n = 0; n < p.n; ++n) {
                double ref = 0;
                if (p.mode == 0) for (int r = 0; r < 16; ++r) ref += (double)bf2f(hx[8 + m + 8 * r]) * bf2f(hw[n * 16 + r]);
                else if (p.mode == 1) for (int k = 0; k < 16; ++k) ref += (double)bf2f(ha[m * 16 + k]) * bf2f(hw[n * 16 + k]);
                else for (int k = 0; k < 64; ++k) ref += (double)bf2f(ha[m * 64 + k]) * bf2f(hw[n * 64 + k]);
                ref *= p.reps / p.nacc;
                maxerr = fmax(maxerr, fabs(ref - hd[m * 256 + n]));
                maxref = fmax(maxref, fabs(ref));
            }
        int nmma = p.mode == 2 ? 4 * p.reps : p.reps;
        printf("%-44s N=%3d reps=%5d maxerr=%.3g (maxref %.3g) %s  cycles/mma=%.1f\n", name, p.n, p.reps, maxerr, maxref,
               maxerr <= 1e-3 * fmax(1.0, maxref) ? "OK" : "MISMATCH", (double)cyc / nmma);
    };
    // correctness (reps = 1)
    run({0, 64, 0, 0, 1, 0, 1, 0, 0, 0}, "SS rowtap A(LBO=128,SBO=16) B(LBO=128,SBO=256)");
    run({0, 64, 1, 0, 1, 0, 1, 0, 0, 0}, "SS rowtap A(LBO=16,SBO=128) B(LBO=128,SBO=256)");
    run({0, 64, 0, 1, 1, 0, 1, 0, 0, 0}, "SS rowtap A(LBO=128,SBO=16) B(LBO=256,SBO=128)");
    run({0, 64, 1, 1, 1, 0, 1, 0, 0, 0}, "SS rowtap A(LBO=16,SBO=128) B(LBO=256,SBO=128)");
    run({1, 64, 0, 0, 1, 0, 1, 0, 0, 0}, "TS A(lo=even) B(LBO=128,SBO=256)");
    run({1, 64, 0, 0, 1, 1, 1, 0, 0, 0}, "TS A(lo=odd)  B(LBO=128,SBO=256)");
    run({1, 64, 0, 1, 1, 0, 1, 0, 0, 0}, "TS A(lo=even) B(LBO=256,SBO=128)");
    run({2, 64, 0, 0, 1, 0, 1, 0, 0, 0}, "SS Kmaj A(LBO=128,SBO=1024) B SW128");
    run({2, 64, 1, 0, 1, 0, 1, 0, 0, 0}, "SS Kmaj A(LBO=1024,SBO=128) B SW128");
    run({2, 256, 0, 0, 1, 0, 1, 0, 0, 0}, "SS Kmaj A(LBO=128,SBO=1024) B SW128");
    // throughput (values are garbage-scaled by reps but we only time)
    char nm[128];
    run({3, 256, 0, 0, 2048, 0, 1, 0, 0, 0}, "TPUT3 A SW64, B interleave std, fixed");
    run({3, 256, 0, 0, 2048, 0, 1, 1, 0, 0}, "TPUT3 A SW64, B interleave std, vary");
    run({3, 256, 1, 0, 2048, 0, 1, 0, 0, 0}, "TPUT3 A SW64, B interleave overlap, fixed");
    run({3, 256, 1, 0, 2048, 0, 1, 1, 0, 0}, "TPUT3 A SW64, B interleave overlap, vary");
    run({3, 256, 1, 0, 2048, 0, 2, 1, 0, 0}, "TPUT3 A SW64, B overlap, vary, nacc2");
    for (int dc : {0, 64, 128, 192, 256}) { snprintf(nm, 128, "TPUT SS rowtap VARY N=256 dcol=%d", dc); run({0, 256, 0, 0, 2048, 0, 1, 1, dc, 0}, nm); }
    for (int sp : {64, 128, 192}) { snprintf(nm, 128, "TPUT split %d+%d plain", sp, 256 - sp); run({0, 256, 0, 0, 2048, 0, 1, 1, 0, sp}, nm); }
    for (int sp : {64, 128, 192}) { snprintf(nm, 128, "TPUT split %d+%d collector", sp, 256 - sp); run({0, 256, 0, 0, 2048, 0, 1, 2, 0, sp}, nm); }
    for (int sp : {64, 128, 192}) { snprintf(nm, 128, "TPUT split %d+%d plain dcol64", sp, 256 - sp); run({0, 256, 0, 0, 2048, 0, 1, 1, 64, sp}, nm); }
    for (int na : {1, 2, 4})
        for (int n : {64, 128, 192, 256}) if (n * na <= 512) { snprintf(nm, 128, "TPUT SS rowtap nacc=%d", na); run({0, n, 0, 0, 2048, 0, na, 0, 0, 0}, nm); }
    for (int na : {1, 2, 4, 7})
        for (int n : {64, 128, 256}) if (n * na <= 480) { snprintf(nm, 128, "TPUT TS nacc=%d", na); run({1, n, 0, 0, 2048, 0, na, 0, 0, 0}, nm); }
    for (int na : {1, 2, 4})
        for (int n : {64, 128, 256}) if (n * na <= 512) { snprintf(nm, 128, "TPUT SS Kmaj/SW128 nacc=%d", na); run({2, n, 0, 0, 512, 0, na, 0, 0, 0}, nm); }
    printf("done\n");
    return 0;
}
