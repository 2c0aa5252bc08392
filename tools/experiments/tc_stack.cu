// tc_stack.cu — tap-stacked tcgen05 convolution for narrow layers (dilation 8, <= 16 output
// channels, <= 32 input channels): the forward and backward-data passes of BASELINE config 2 and
// of the config-5 body layers.
//
//   out[k][q] = sum_s sum_c W[k][c][s] in[c][q + 8s + off]
//
// The row-tap kernel (tc_conv.cu) puts 128 output columns on M and (tap block, filter) on N; with
// 15 filters its MMAs are 128x64x16 and each one re-reads a 4 KB A tile from shared memory, so
// shared-memory bandwidth holds it at ~48-65 cycles per MMA. Here the weights are the A operand
// and the output columns are N:
//   M = 128 = 16 output channels x 8 taps (row m = 8k + t), N = 256 columns, K = 16 input channels;
//   tap group g (taps 8g .. 8g+7) reads the input window 64g columns further on, so all groups
//   accumulate into one TMEM tile:   D[(k,t)][q] = sum_g sum_c W[k][c][8g+t] in[c][q + 64g + off]
// and out[k][q] = sum_t D[(k,t)][q + 8t]. One 256-column tile is G = ceil(S/8) MMAs of
// 128x256x16 (config 2: 7 x 128 cycles) reading 8 KB of B each (64 B/clk of shared memory).
//
// The shifted row sum runs in the epilogue. The 8 tap rows of an output channel are 8 consecutive
// TMEM lanes of one warp, so it is a rolling shuffle over 8-column chunks: at chunk a, lane t adds
// its chunk a to the partial sum of output chunk a - t that lane t-1 held one chunk earlier
// (shfl.up), and lane 7 then holds the finished chunk a - 7. The sum order per output is fixed
// (tap row 0 first), and each accumulation chain in TMEM is G * C_in products long.
//
// The input arrives as the q-chunk-major image the B operand reads (TMA 4-D boxes of 8 columns x
// CP channels x 32 chunks, OOB zero fill = the backward-data padding) into a ring of 32-chunk
// stages; a D tile reads 32 + 8(G-1) chunks, i.e. its own stage and `reach` more, and the first
// `reach` ring slots are mirrored past the end so no MMA operand wraps.
//
// Work: output tiles (item, 256 columns) split contiguously over persistent CTAs; a run of tiles
// inside one item computes one extra D tile for the last tiles' 56-column reach.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "sm100.cuh"

namespace c1d {
namespace {

using namespace sm100;

__host__ __device__ inline int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

constexpr int kStackThreads = 256;  // warp 0 TMA, 1 MMA, 2 TMEM alloc, 4-7 epilogue
constexpr int kTileCols = 256;
constexpr int kChunksPerTile = kTileCols / 8;
constexpr uint32_t kStackTmemCols = 512;  // two 256-column D tiles
constexpr int kMaxRing = 8;

struct StackPlan {
    int cp, nks, groups, reach, ring;
    uint32_t chunk_bytes, stage_bytes, a_bytes;
    size_t smem_bytes;
};

bool make_stack_plan(const ConvGeom& g, StackPlan* out) {
    if (g.dil != 8 || g.xr_rows || g.xr_inline) return false;
    if (g.in_off % 8 != 0 || g.out_w % 8 != 0 || g.out_w < 8) return false;
    const int64_t pitch = g.in_stride ? g.in_stride : g.in_w;
    if (pitch % 8 != 0 || pitch < g.in_w) return false;
    if (g.out_ch > 16 || g.in_ch > 32 || g.taps < 1) return false;
    if (g.n * g.in_ch >= (int64_t{1} << 31)) return false;
    StackPlan p{};
    p.cp = g.in_ch <= 16 ? 16 : 32;
    p.nks = p.cp / 16;
    p.groups = static_cast<int>(ceil_div(g.taps, 8));
    p.reach = static_cast<int>(ceil_div(8 * (p.groups - 1), kChunksPerTile));
    p.chunk_bytes = static_cast<uint32_t>(p.cp * 16);
    p.stage_bytes = kChunksPerTile * p.chunk_bytes;
    p.a_bytes = static_cast<uint32_t>(p.groups * p.nks) * 4096u;
    const uint32_t budget = 200 * 1024;
    if (p.a_bytes > 96 * 1024) return false;
    p.ring = 0;
    for (int r = kMaxRing; r >= p.reach + 2; --r)
        if (p.a_bytes + static_cast<uint32_t>(r + p.reach) * p.stage_bytes <= budget) {
            p.ring = r;
            break;
        }
    if (p.ring == 0) return false;
    p.smem_bytes = p.a_bytes + static_cast<size_t>(p.ring + p.reach) * p.stage_bytes + 1024;
    *out = p;
    return true;
}

struct StackParams {
    int64_t n, in_ch, out_ch, out_w;
    int64_t off8;             // input column offset in chunks (in_off / 8)
    int64_t tiles_per_item;   // ceil(out_w / 256)
    int64_t units;            // n * tiles_per_item
    StackPlan pl;
    const uint16_t* aimg;     // packed weights [g][ks][4 KB]
    float* out;               // [n][out_ch][out_w]
    unsigned long long* prof;
    int dbg;  // dev timing switch (C1D_STACK_DBG): 1 = TMEM loads only, 2 = no TMEM loads (wrong results)
};

// Packed A image of tap group g, K-step ks: rows m = 8o + t (output channel o, tap s = 8g + t),
// K = 16 input channels i = 16ks + c, bf16 RNE, in the K-major no-swizzle core-matrix order
// (8 rows x 16 B per core matrix; K-core stride 128 B, M-core stride 256 B). mode 1 (backward-data)
// takes the caller's KCS weights of the original conv transposed, taps reversed
// (pack_weights_backward, tensor.cpp:23-41).
__global__ void pack_stack_kernel(const float* __restrict__ w, uint16_t* __restrict__ img, int64_t O, int64_t I,
                                  int64_t S, int groups, int nks, int mode) {
    const int64_t total = static_cast<int64_t>(groups) * nks * 2048;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t blk = e / 2048;
        const int g = static_cast<int>(blk / nks), ks = static_cast<int>(blk % nks);
        const int r = static_cast<int>(e % 2048);
        const int core = r / 64, within = r % 64;
        const int m = (core / 2) * 8 + within / 8;
        const int c16 = (core % 2) * 8 + within % 8;
        const int64_t o = m / 8, t = m % 8, s = 8 * g + t, i = 16 * ks + c16;
        float v = 0.0f;
        if (o < O && i < I && s < S) v = mode == 0 ? w[(o * I + i) * S + s] : w[(i * O + o) * S + (S - 1 - s)];
        img[e] = fp32_to_bf16_bits(v);
    }
}

__device__ __forceinline__ void st_global_v4(float* p, float a, float b, float c, float d) {
    asm volatile("st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

__global__ void __launch_bounds__(kStackThreads, 1)
    tc_stack_kernel(const __grid_constant__ CUtensorMap xmap, const StackParams p) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint64_t full[kMaxRing], empty[kMaxRing];
    __shared__ uint64_t tmem_full[2], tmem_empty[2], a_full;
    __shared__ uint32_t tmem_base_s;

    const StackPlan& pl = p.pl;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    const uint32_t a_s = smem_u32(smem);
    const uint32_t ring_s = a_s + pl.a_bytes;
    // this CTA's output tiles
    const int64_t u0 = p.units * blockIdx.x / gridDim.x, u1 = p.units * (blockIdx.x + 1) / gridDim.x;

    if (threadIdx.x == 0) {
        for (int s = 0; s < pl.ring; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tmem_full[b], 1);
            mbar_init(&tmem_empty[b], 4);
        }
        mbar_init(&a_full, 1);
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc<kStackTmemCols>(&tmem_base_s);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_s;
    pdl_wait();

    if (warp == 0) {
        if (lane == 0) {
            prefetch_tmap(&xmap);
            mbar_arrive_expect_tx(smem_u32(&a_full), pl.a_bytes);
            bulk_g2s(a_s, p.aimg, pl.a_bytes, smem_u32(&a_full));
            int64_t st = 0;  // stages issued (all runs)
            long long tw = 0;
            const long long tb = clock64();
            for (int64_t u = u0; u < u1;) {
                const int64_t n = u / p.tiles_per_item, i0 = u % p.tiles_per_item;
                const int64_t i1 = imin64(p.tiles_per_item, i0 + (u1 - u));
                const int64_t stages = (i1 - i0 + 1) + pl.reach;
                for (int64_t j = 0; j < stages; ++j, ++st) {
                    const int slot = static_cast<int>(st % pl.ring);
                    const long long t0 = clock64();
                    mbar_wait(smem_u32(&empty[slot]), static_cast<uint32_t>(((st / pl.ring) & 1) ^ 1));
                    tw += clock64() - t0;
                    const uint32_t fb = smem_u32(&full[slot]);
                    mbar_arrive_expect_tx(fb, pl.stage_bytes * (slot < pl.reach ? 2u : 1u));
                    const int32_t chunk0 = static_cast<int32_t>(kChunksPerTile * (i0 + j) + p.off8);
                    tma_load_4d(ring_s + static_cast<uint32_t>(slot) * pl.stage_bytes, &xmap, 0, 0, chunk0,
                                static_cast<int32_t>(n), fb);
                    if (slot < pl.reach)  // mirror past the ring end
                        tma_load_4d(ring_s + static_cast<uint32_t>(pl.ring + slot) * pl.stage_bytes, &xmap, 0, 0, chunk0,
                                    static_cast<int32_t>(n), fb);
                }
                u = i1 + n * p.tiles_per_item;
            }
            if (p.prof) {
                p.prof[blockIdx.x * 8 + 0] = tw;
                p.prof[blockIdx.x * 8 + 1] = clock64() - tb;
            }
        }
    } else if (warp == 1) {
        // A (weights): K-major, K-core stride 128 B, M-core stride 256 B; B (input): MN-major
        // q-chunk-major rows, K-core (8 channels) stride 128 B, MN-core (8 columns) stride CP*16 B
        const uint32_t idesc = make_idesc(128, kTileCols, kFmtBF16, 0, 1);
        mbar_wait(smem_u32(&a_full), 0);
        tc_fence_after();
        int64_t st_base = 0, waited = 0, dcount = 0;
        long long tf = 0, tt = 0;
        const long long tb = clock64();
        for (int64_t u = u0; u < u1;) {
            const int64_t n = u / p.tiles_per_item, i0 = u % p.tiles_per_item;
            const int64_t i1 = imin64(p.tiles_per_item, i0 + (u1 - u));
            const int64_t nd = i1 - i0 + 1;
            for (int64_t j = 0; j < nd; ++j, ++dcount) {
                const long long t0 = clock64();
                while (waited <= st_base + j + pl.reach) {
                    mbar_wait(smem_u32(&full[waited % pl.ring]), static_cast<uint32_t>((waited / pl.ring) & 1));
                    ++waited;
                }
                const long long t1 = clock64();
                const int buf = static_cast<int>(dcount & 1);
                mbar_wait(smem_u32(&tmem_empty[buf]), static_cast<uint32_t>(((dcount >> 1) & 1) ^ 1));
                tf += t1 - t0;
                tt += clock64() - t1;
                tc_fence_after();
                const int slot = static_cast<int>((st_base + j) % pl.ring);
                if (elect_one()) {
                    const uint32_t d = tmem + static_cast<uint32_t>(buf * kTileCols);
                    const uint32_t b_slot = ring_s + static_cast<uint32_t>(slot) * pl.stage_bytes;
                    for (int g = 0; g < pl.groups; ++g) {
#pragma unroll 2
                        for (int ks = 0; ks < pl.nks; ++ks) {
                            const uint64_t ad = make_smem_desc(a_s + static_cast<uint32_t>(g * pl.nks + ks) * 4096u, 128, 256,
                                                               kLayoutNone);
                            const uint64_t bd = make_smem_desc(
                                b_slot + static_cast<uint32_t>(8 * g) * pl.chunk_bytes + static_cast<uint32_t>(ks) * 256u, 128,
                                pl.chunk_bytes, kLayoutNone);
                            mma_bf16_ss(d, ad, bd, idesc, (g | ks) != 0 ? 1u : 0u);
                        }
                    }
                    mma_commit(smem_u32(&tmem_full[buf]));
                    mma_commit(smem_u32(&empty[slot]));
                }
                __syncwarp();
            }
            // the run's reach stages: read by its last tiles, released now
            if (elect_one())
                for (int r = 0; r < pl.reach; ++r) mma_commit(smem_u32(&empty[(st_base + nd + r) % pl.ring]));
            __syncwarp();
            st_base += nd + pl.reach;
            u = i1 + n * p.tiles_per_item;
        }
        if (p.prof && lane == 0) {
            p.prof[blockIdx.x * 8 + 2] = tf;
            p.prof[blockIdx.x * 8 + 3] = tt;
            p.prof[blockIdx.x * 8 + 4] = clock64() - tb;
        }
    } else if (warp >= 4) {
        // ---- epilogue: rolling shifted row sum (see the file comment)
        const int quarter = warp - 4;
        const int m = quarter * 32 + lane;
        const int k = m >> 3, t = m & 7;
        const uint32_t lane_base = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
        const int64_t qc = p.out_w / 8;  // output chunks per item
        int64_t dcount = 0;
        long long tw = 0;
        const long long tb = clock64();
        for (int64_t u = u0; u < u1;) {
            const int64_t n = u / p.tiles_per_item, i0 = u % p.tiles_per_item;
            const int64_t i1 = imin64(p.tiles_per_item, i0 + (u1 - u));
            const int64_t nd = i1 - i0 + 1;
            const int64_t oc_end = imin64(kChunksPerTile * i1, qc);
            float* orow = p.out + (n * p.out_ch + k) * p.out_w;
            const bool emitter = t == 7 && k < p.out_ch;
            float s_acc[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) s_acc[e] = 0.0f;
            for (int64_t j = 0; j < nd; ++j, ++dcount) {
                const int buf = static_cast<int>(dcount & 1);
                const long long t0 = clock64();
                mbar_wait_sleep(smem_u32(&tmem_full[buf]), static_cast<uint32_t>((dcount >> 1) & 1), 64);
                tw += clock64() - t0;
                tc_fence_after();
                // quads of 4 chunks (32 columns): the next quad's TMEM load is in flight while this
                // quad is summed; emission predicates and the store base are per quad
                const uint32_t tcol = lane_base + static_cast<uint32_t>(buf * kTileCols);
                const int a_tile = kChunksPerTile * static_cast<int>(j);  // run-relative D chunk of the tile
                uint32_t v[32], vn[32];
                if (p.dbg != 2) {
                    tmem_ld32(tcol, v);
                    tmem_ld_wait();
                } else {
#pragma unroll
                    for (int e = 0; e < 32; ++e) v[e] = static_cast<uint32_t>(e + lane);
                }
#pragma unroll 1
                for (int q4 = 0; q4 < kChunksPerTile / 4; ++q4) {
                    const bool more = q4 + 1 < kChunksPerTile / 4;
                    if (more && p.dbg != 2) tmem_ld32(tcol + static_cast<uint32_t>(32 * (q4 + 1)), vn);
                    if (p.dbg == 1) {  // loads only
                        if (more) {
                            tmem_ld_wait();
#pragma unroll
                            for (int e = 0; e < 32; ++e) v[e] += vn[e];
                        }
                        continue;
                    }
                    const int a0 = a_tile + 4 * q4;                     // D chunk of step 0
                    const int oc0 = static_cast<int>(kChunksPerTile * i0) + a0 - 7;  // its output chunk
                    unsigned emit = 0;
#pragma unroll
                    for (int cc = 0; cc < 4; ++cc)
                        emit |= (emitter && a0 + cc >= 7 && oc0 + cc < oc_end) ? (1u << cc) : 0u;
                    float* ob = orow + 8 * static_cast<int64_t>(oc0);
#pragma unroll
                    for (int cc = 0; cc < 4; ++cc) {
                        float r[8];
#pragma unroll
                        for (int e = 0; e < 8; ++e) r[e] = __shfl_up_sync(0xffffffffu, s_acc[e], 1, 8);
#pragma unroll
                        for (int e = 0; e < 8; ++e) s_acc[e] = (t == 0 ? 0.0f : r[e]) + __uint_as_float(v[8 * cc + e]);
                        if (emit & (1u << cc)) {
                            st_global_v4(ob + 8 * cc, s_acc[0], s_acc[1], s_acc[2], s_acc[3]);
                            st_global_v4(ob + 8 * cc + 4, s_acc[4], s_acc[5], s_acc[6], s_acc[7]);
                        }
                    }
                    if (more) {
                        if (p.dbg != 2) tmem_ld_wait();
#pragma unroll
                        for (int e = 0; e < 32; ++e) v[e] = p.dbg != 2 ? vn[e] : v[e] + 1u;
                    }
                }
                if (p.dbg == 1 && emitter) orow[0] = __uint_as_float(v[0]);  // keep the loads live
                tc_fence_before();  // every column of the tile has been read
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&tmem_empty[buf]));
            }
            u = i1 + n * p.tiles_per_item;
        }
        if (p.prof && warp == 4 && lane == 0) {
            p.prof[blockIdx.x * 8 + 5] = tw;
            p.prof[blockIdx.x * 8 + 6] = clock64() - tb;
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 2) tmem_dealloc<kStackTmemCols>(tmem);
}

PFN_cuTensorMapEncodeTiled_v12000 stack_encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }();
    return fn;
}

}  // namespace

bool tc_stack_supported(const ConvGeom& g) {
    StackPlan p;
    return make_stack_plan(g, &p);
}

size_t tc_stack_workspace_bytes(const ConvGeom& g) {
    StackPlan p;
    return make_stack_plan(g, &p) ? p.a_bytes : 0;
}

cudaError_t launch_tc_stack(const uint16_t* in_bf16, const float* w_kcs, float* out, const ConvGeom& g,
                            void* workspace, cudaStream_t stream, bool w_bwd_raw) {
    StackPlan pl;
    if (!make_stack_plan(g, &pl)) return cudaErrorNotSupported;
    auto encode = stack_encode_fn();
    if (!encode) return cudaErrorNotSupported;
    if (reinterpret_cast<uintptr_t>(in_bf16) & 15u) return cudaErrorInvalidValue;
    uint16_t* aimg = static_cast<uint16_t*>(workspace);
    {
        const int64_t total = static_cast<int64_t>(pl.groups) * pl.nks * 2048;
        const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(total, 256), 4 * num_sms()));
        pack_stack_kernel<<<blocks, 256, 0, stream>>>(w_kcs, aimg, g.out_ch, g.in_ch, g.taps, pl.groups, pl.nks,
                                                      w_bwd_raw ? 1 : 0);
        note_launch();
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    const int64_t pitch = g.in_stride ? g.in_stride : g.in_w;
    CUtensorMap xmap;
    {
        // x as (8 elements, channel, 8-column chunk, item): element (e, c, ch, n) at
        // n*C*pitch + c*pitch + 8*ch + e; the box (8, CP, 32, 1) lands q-chunk-major
        const cuuint64_t dims[4] = {8, static_cast<cuuint64_t>(g.in_ch), static_cast<cuuint64_t>(pitch / 8),
                                    static_cast<cuuint64_t>(g.n)};
        const cuuint64_t strides[3] = {static_cast<cuuint64_t>(pitch) * 2, 16,
                                       static_cast<cuuint64_t>(g.in_ch * pitch) * 2};
        const cuuint32_t box[4] = {8, static_cast<cuuint32_t>(pl.cp), static_cast<cuuint32_t>(kChunksPerTile), 1};
        const cuuint32_t estr[4] = {1, 1, 1, 1};
        if (encode(&xmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<uint16_t*>(in_bf16), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    StackParams sp{};
    sp.n = g.n;
    sp.in_ch = g.in_ch;
    sp.out_ch = g.out_ch;
    sp.out_w = g.out_w;
    sp.off8 = g.in_off / 8;
    sp.tiles_per_item = ceil_div(g.out_w, kTileCols);
    sp.units = g.n * sp.tiles_per_item;
    sp.pl = pl;
    sp.aimg = aimg;
    sp.out = out;
    sp.prof = nullptr;
    static const int dbg = getenv("C1D_STACK_DBG") ? atoi(getenv("C1D_STACK_DBG")) : 0;
    sp.dbg = dbg;
    if (sp.units == 0) return cudaSuccess;
    static const bool profile = getenv("C1D_PROFILE") != nullptr;
    const int grid = static_cast<int>(std::min<int64_t>(num_sms(), sp.units));
    cudaError_t e = cudaFuncSetAttribute(tc_stack_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(pl.smem_bytes));
    if (e != cudaSuccess) return e;
    if (profile) {
        cudaMalloc(&sp.prof, sizeof(unsigned long long) * 8 * grid);
        cudaMemset(sp.prof, 0, sizeof(unsigned long long) * 8 * grid);
    }
    e = launch_pdl(tc_stack_kernel, dim3(grid), dim3(kStackThreads), pl.smem_bytes, stream, xmap, sp);
    note_launch();
    if (profile && e == cudaSuccess) {
        std::vector<unsigned long long> h(8 * grid);
        cudaMemcpy(h.data(), sp.prof, h.size() * 8, cudaMemcpyDeviceToHost);
        double a[8] = {0};
        for (int b = 0; b < grid; ++b)
            for (int i = 0; i < 8; ++i) a[i] += static_cast<double>(h[b * 8 + i]) / grid;
        fprintf(stderr, "[tc_stack prof] G=%d reach=%d ring=%d | producer wait_empty %.0f / total %.0f | mma wait_full %.0f "
                "wait_tmem %.0f total %.0f | epilogue wait %.0f total %.0f (cycles, CTA avg)\n",
                pl.groups, pl.reach, pl.ring, a[0], a[1], a[2], a[3], a[4], a[5], a[6]);
        cudaFree(sp.prof);
    }
    return e;
}

}  // namespace c1d
