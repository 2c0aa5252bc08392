// tc_conv.cu — tcgen05 (sm_100a) BF16 tensor-core convolution for dilation 8: forward and
// backward-data (the same contraction with flipped, transposed filters).
//
// Contraction (forward-shaped):  out[n][o][q] = sum_i sum_s W[o][i][s] * in[n][i][q + 8s + off]
//
// Mapping ("row-tap" implicit GEMM, one MMA per (128-column tile, input channel)):
//   M = 128 consecutive output columns q (TMEM lanes)
//   K = 16 consecutive taps r of ONE input channel
//   N = G blocks x KP filters, block g holding taps 16g..16g+15
//   A[m][r] = in[i][q0 + m + 8r]   read straight out of a natural bf16 row in shared memory:
//            an MN-major SWIZZLE_NONE operand with M-group stride 16 B and K-group stride 128 B
//            (rows of 8 elements = 16 B = one dilation step; core matrices overlap in memory)
//   B[(g,o)][r] = W[o][i][16g + r]  (K-major SWIZZLE_NONE image prepared once per call)
// Tap 16g + r of input tile p lands on output tile p - g (16 taps x 8 = 128 = one tile), in the
// same TMEM lane. TMEM therefore holds a ring of R = 512/KP per-output-tile accumulators laid out
// in descending order, so one MMA's N columns cover output tiles p, p-1, .., p-G+1; no
// cross-lane reduction ever happens and the epilogue is a plain TMEM -> global store.
//
// Pipeline per CTA (persistent, one CTA per SM, 256 threads):
//   warp 0   TMA producer: per stage, CC channel windows (2-D TMA boxes of 256 columns, OOB
//            zero fill implements the backward-data zero padding) + the CC channels' B image
//            (one cp.async.bulk)
//   warp 1   MMA issuer (one elected thread): tcgen05.mma kind::f16, commits to stage_empty and,
//            when an output tile has seen all its taps, to slot_full
//   warp 2   TMEM allocator
//   warps 4-7 epilogue: tcgen05.ld 32 lanes x KP columns -> coalesced fp32 stores, then zero the
//            slot with tcgen05.st and hand it back (slot_empty)
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>

#include "common.cuh"
#include "kernels.h"
#include "sm100.cuh"

namespace c1d {
namespace {

using namespace sm100;

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

constexpr int kTileQ = 128;      // output columns per tile (MMA M)
constexpr int kSegQ = 256;       // TMA box width in elements
constexpr int kTapsPerBlock = 16;
constexpr int kMaxStages = 6;
constexpr int kMaxSlots = 32;
constexpr int kThreads = 256;
constexpr uint32_t kTmemCols = 512;

struct Plan {
    int kp;          // padded filters per block (16, 32, 64)
    int g;           // tap blocks
    int r;           // ring slots = 512 / kp
    int t;           // input tiles per super-tile
    int cc;          // channels per stage
    int stages;
    int n_seg;       // TMA segments per channel window
    int xw;          // window elements per channel (n_seg * 256)
    int ntot;        // g * kp (B rows)
    uint32_t b_chan_bytes;
    uint32_t x_stage_bytes;
    uint32_t w_stage_bytes;
    size_t smem_bytes;
    int kgroups;     // filter groups of kp
};

struct KParams {
    int64_t n_items, in_ch, in_w, out_ch, out_w, in_off;
    int64_t tiles_per_item, total_tiles;
    int taps, k_begin;
    Plan pl;
    const uint16_t* bimg;  // this filter group's B image: [in_ch][ntot*16] bf16
    float* out;
};

bool make_plan(const ConvGeom& g, Plan* pl) {
    if (g.dil != 8) return false;
    if (g.in_w % 8 != 0 || g.in_w < 8) return false;  // TMA global stride must be a multiple of 16 B
    if (g.n * g.in_ch >= (int64_t{1} << 31) || g.in_w >= (int64_t{1} << 31)) return false;
    Plan p{};
    p.kp = g.out_ch <= 16 ? 16 : (g.out_ch <= 32 ? 32 : 64);
    p.kgroups = static_cast<int>(ceil_div(g.out_ch, p.kp));
    p.g = static_cast<int>(ceil_div(g.taps, kTapsPerBlock));
    p.r = static_cast<int>(kTmemCols) / p.kp;
    p.ntot = p.g * p.kp;
    if (p.ntot > static_cast<int>(kTmemCols) / 2 && p.kp == 64) {
        if (p.g > 4) return false;
    }
    if (p.g + 1 > p.r) return false;
    p.t = std::min(4, p.r - p.g);
    if (p.t < 1) return false;
    p.n_seg = static_cast<int>(ceil_div(p.t * kTileQ + 8 * (kTapsPerBlock - 1), kSegQ));
    p.xw = p.n_seg * kSegQ;
    p.b_chan_bytes = static_cast<uint32_t>(p.ntot * kTapsPerBlock * 2);
    const uint32_t per_chan = static_cast<uint32_t>(p.xw * 2) + p.b_chan_bytes;
    p.cc = static_cast<int>(std::max<uint32_t>(1, std::min<uint32_t>(48 * 1024 / per_chan, 16)));
    p.cc = static_cast<int>(std::min<int64_t>(p.cc, g.in_ch));
    {
        const int64_t nch = ceil_div(g.in_ch, p.cc);  // balance the chunks
        p.cc = static_cast<int>(ceil_div(g.in_ch, nch));
    }
    p.x_stage_bytes = static_cast<uint32_t>(p.cc * p.xw * 2);
    p.w_stage_bytes = static_cast<uint32_t>(p.cc) * p.b_chan_bytes;
    const uint32_t stage = p.x_stage_bytes + p.w_stage_bytes;
    p.stages = static_cast<int>(std::min<uint32_t>(kMaxStages, (200 * 1024) / stage));
    if (p.stages < 2) return false;
    p.smem_bytes = static_cast<size_t>(p.stages) * stage + 1024;
    *pl = p;
    return true;
}

// ---------------------------------------------------------------------------- B image packing
// img[kg][c][row][r] in the K-major SWIZZLE_NONE core-matrix order:
//   element (row, r) at (row/8)*128 + (r/8)*64 + (row%8)*8 + (r%8)   (SBO 256 B, LBO 128 B)
__global__ void pack_bimg_kernel(const float* __restrict__ wg, uint16_t* __restrict__ img, int64_t out_ch,
                                 int64_t in_ch, int64_t taps, int kp, int g, int kgroups) {
    const int64_t ntot = static_cast<int64_t>(g) * kp;
    const int64_t per_chan = ntot * kTapsPerBlock;
    const int64_t total = static_cast<int64_t>(kgroups) * in_ch * per_chan;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e % kTapsPerBlock;
        const int64_t row = (e / kTapsPerBlock) % ntot;
        const int64_t c = (e / per_chan) % in_ch;
        const int64_t kg = e / (per_chan * in_ch);
        const int64_t blk = row / kp, o = kg * kp + row % kp, s = blk * kTapsPerBlock + r;
        float v = 0.0f;
        if (o < out_ch && s < taps) v = wg[(o * in_ch + c) * taps + s];
        const int64_t off = (row / 8) * 128 + (r / 8) * 64 + (row % 8) * 8 + (r % 8);
        img[(kg * in_ch + c) * per_chan + off] = fp32_to_bf16_bits(v);
    }
}

// ---------------------------------------------------------------------------- schedule
// Each CTA owns output tiles [b, e) of the flattened (item, tile) list. For each item segment
// (n, j0..j1) it processes input tiles j0 .. j1+G-1 in super-tiles of up to T tiles. Positions
// are consecutive across segments and start at G-1 (positions 0..G-2 are warm-up phantoms).
struct Cursor {
    int64_t cur, end;         // flattened output-tile cursor
    int64_t n, j0, j1;        // current segment
    int64_t i;                // next input tile in the segment
    bool valid;
};

__device__ __forceinline__ bool next_segment(Cursor& c, int64_t J) {
    if (c.cur >= c.end) return false;
    c.n = c.cur / J;
    c.j0 = c.cur % J;
    const int64_t last = imin64(c.end, (c.n + 1) * J) - 1;
    c.j1 = last % J;
    c.cur = last + 1;
    c.i = c.j0;
    return true;
}

// Returns the number of input tiles in the next super-tile (0 = done) and its first tile index.
__device__ __forceinline__ int next_super(Cursor& c, int64_t J, int G, int T, int64_t* n_out, int64_t* i_out,
                                          int64_t* j1_out) {
    if (!c.valid) return 0;
    if (c.i > c.j1 + G - 1) {
        if (!next_segment(c, J)) {
            c.valid = false;
            return 0;
        }
    }
    const int64_t remain = c.j1 + G - 1 - c.i + 1;
    const int tcur = static_cast<int>(imin64(T, remain));
    *n_out = c.n;
    *i_out = c.i;
    *j1_out = c.j1;
    c.i += tcur;
    return tcur;
}

__device__ __forceinline__ Cursor make_cursor(const KParams& p) {
    Cursor c{};
    const int64_t b = p.total_tiles * blockIdx.x / gridDim.x;
    const int64_t e = p.total_tiles * (blockIdx.x + 1) / gridDim.x;
    c.cur = b;
    c.end = e;
    c.valid = next_segment(c, p.tiles_per_item);
    return c;
}

__device__ __forceinline__ uint32_t slot_col(int64_t x, int R, int KP) {
    int64_t m = (-x) % R;
    if (m < 0) m += R;
    return static_cast<uint32_t>(m * KP);
}

__global__ void __launch_bounds__(kThreads, 1)
    tc_conv_kernel(const __grid_constant__ CUtensorMap tmap, const KParams p) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint64_t stage_full[kMaxStages], stage_empty[kMaxStages];
    __shared__ uint64_t slot_full[kMaxSlots], slot_empty[kMaxSlots];
    __shared__ uint32_t tmem_base_s;

    const Plan& pl = p.pl;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t* xs_base = smem;
    uint8_t* ws_base = smem + static_cast<size_t>(pl.stages) * pl.x_stage_bytes;
    const int G = pl.g, T = pl.t, R = pl.r, KP = pl.kp;
    const int64_t J = p.tiles_per_item;
    const int n_chunks = static_cast<int>(ceil_div(p.in_ch, pl.cc));

    if (threadIdx.x == 0) {
        for (int s = 0; s < pl.stages; ++s) {
            mbar_init(&stage_full[s], 1);
            mbar_init(&stage_empty[s], 1);
        }
        for (int s = 0; s < R; ++s) {
            mbar_init(&slot_full[s], 1);
            mbar_init(&slot_empty[s], 4);  // one arrival per epilogue warp
        }
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc<kTmemCols>(&tmem_base_s);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_s;

    if (warp == 0) {
        // ------------------------------------------------------------------ TMA producer
        if (lane == 0) {
            prefetch_tmap(&tmap);
            Cursor cur = make_cursor(p);
            int stage = 0;
            uint32_t phase = 0;
            int64_t n, i0, j1;
            int tcur;
            while ((tcur = next_super(cur, J, G, T, &n, &i0, &j1)) > 0) {
                const int32_t x_start = static_cast<int32_t>(i0 * kTileQ + p.in_off);
                for (int ch = 0; ch < n_chunks; ++ch) {
                    const int c0 = ch * pl.cc;
                    const int ccn = static_cast<int>(imin64(pl.cc, p.in_ch - c0));
                    mbar_wait(smem_u32(&stage_empty[stage]), phase ^ 1);
                    const uint32_t full = smem_u32(&stage_full[stage]);
                    const uint32_t bytes = static_cast<uint32_t>(ccn) * (pl.n_seg * kSegQ * 2 + pl.b_chan_bytes);
                    mbar_arrive_expect_tx(full, bytes);
                    const uint32_t xs = smem_u32(xs_base + static_cast<size_t>(stage) * pl.x_stage_bytes);
                    for (int c = 0; c < ccn; ++c) {
                        const int32_t row = static_cast<int32_t>(n * p.in_ch + c0 + c);
                        for (int sg = 0; sg < pl.n_seg; ++sg)
                            tma_load_2d(xs + static_cast<uint32_t>((c * pl.xw + sg * kSegQ) * 2), &tmap,
                                        x_start + sg * kSegQ, row, full);
                    }
                    const uint32_t wsm = smem_u32(ws_base + static_cast<size_t>(stage) * pl.w_stage_bytes);
                    bulk_g2s(wsm, p.bimg + static_cast<size_t>(c0) * (pl.b_chan_bytes / 2),
                             static_cast<uint32_t>(ccn) * pl.b_chan_bytes, full);
                    if (++stage == pl.stages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            Cursor cur = make_cursor(p);
            int stage = 0;
            uint32_t phase = 0;
            int64_t pos = G - 1;         // position of the next input tile
            int64_t completed = -1;      // highest committed output position
            int64_t n, i0, j1;
            int tcur;
            // warm-up phantom positions 0..G-2 are touched first by input tile G-1
            for (int64_t x = 0; x < G - 1; ++x) mbar_wait(smem_u32(&slot_empty[x % R]), 0);
            while ((tcur = next_super(cur, J, G, T, &n, &i0, &j1)) > 0) {
                for (int t = 0; t < tcur; ++t) {
                    const int64_t x = pos + t;
                    mbar_wait(smem_u32(&slot_empty[x % R]), static_cast<uint32_t>((x / R) & 1));
                }
                tc_fence_after();
                // MMA runs of this super-tile (identical for every channel): contiguous TMEM
                // column ranges of output blocks, split where the slot ring wraps.
                uint32_t rcol[4][2], rboff[4][2], ridesc[4][2];
                int nr[4];
                for (int t = 0; t < tcur; ++t) {
                    const int64_t x = pos + t;
                    int gblk = 0, k = 0;
                    while (gblk < G) {
                        const uint32_t col = slot_col(x - gblk, R, KP);
                        int run = 1;
                        while (gblk + run < G && slot_col(x - gblk - run, R, KP) == col + run * KP &&
                               (run + 1) * KP <= 256)
                            ++run;
                        rcol[t][k] = col;
                        rboff[t][k] = static_cast<uint32_t>((gblk * KP / 8) * 256);
                        ridesc[t][k] = make_idesc(128, static_cast<uint32_t>(run * KP), kFmtBF16, 1, 0);
                        ++k;
                        gblk += run;
                    }
                    nr[t] = k;
                }
                for (int ch = 0; ch < n_chunks; ++ch) {
                    const int c0 = ch * pl.cc;
                    const int ccn = static_cast<int>(imin64(pl.cc, p.in_ch - c0));
                    mbar_wait(smem_u32(&stage_full[stage]), phase);
                    tc_fence_after();
                    const uint32_t xs = smem_u32(xs_base + static_cast<size_t>(stage) * pl.x_stage_bytes);
                    const uint32_t wsm = smem_u32(ws_base + static_cast<size_t>(stage) * pl.w_stage_bytes);
                    const uint64_t a0 = make_smem_desc(xs, 128, 16, kLayoutNone);
                    const uint64_t b0 = make_smem_desc(wsm, 128, 256, kLayoutNone);
                    for (int c = 0; c < ccn; ++c) {
                        const uint32_t bchan = static_cast<uint32_t>(c) * pl.b_chan_bytes;
                        const uint32_t achan = static_cast<uint32_t>(c * pl.xw * 2);
                        for (int t = 0; t < tcur; ++t) {
                            const uint64_t adesc = desc_advance(a0, achan + static_cast<uint32_t>(t * kTileQ * 2));
                            for (int k = 0; k < nr[t]; ++k)
                                mma_bf16_ss(tmem + rcol[t][k], adesc, desc_advance(b0, bchan + rboff[t][k]),
                                            ridesc[t][k], 1);
                        }
                    }
                    mma_commit(smem_u32(&stage_empty[stage]));
                    if (++stage == pl.stages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                pos += tcur;
                const int64_t done_upto = pos - 1 - (G - 1);
                for (int64_t x = completed + 1; x <= done_upto; ++x) mma_commit(smem_u32(&slot_full[x % R]));
                completed = (completed > done_upto ? completed : done_upto);
            }
        }
    } else if (warp >= 4) {
        // ------------------------------------------------------------------ epilogue
        const int quarter = warp - 4;  // TMEM lanes 32*quarter .. +31
        const uint32_t lane_base = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
        // zero every slot once, then hand them out
        {
            uint32_t z[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) z[j] = 0;
            for (uint32_t col = 0; col < kTmemCols; col += 16) tmem_st16(lane_base + col, z);
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0)
                for (int s = 0; s < R; ++s) mbar_arrive(smem_u32(&slot_empty[s]));
        }
        Cursor cur = make_cursor(p);
        // ring of what sits at recent positions: real output? (n, tile)
        int64_t ring_n[kMaxSlots];
        int64_t ring_j[kMaxSlots];
        bool ring_real[kMaxSlots];
        (void)ring_n;
        int64_t pos = G - 1;
        for (int x = 0; x < G - 1; ++x) ring_real[x % kMaxSlots] = false;
        int64_t n, i0, j1;
        int tcur;
        int64_t drained = 0;
        while ((tcur = next_super(cur, J, G, T, &n, &i0, &j1)) > 0) {
            for (int t = 0; t < tcur; ++t) {
                const int64_t x = pos + t;
                ring_n[x % kMaxSlots] = n;
                ring_j[x % kMaxSlots] = i0 + t;
                ring_real[x % kMaxSlots] = (i0 + t) <= j1;
            }
            pos += tcur;
            const int64_t done_upto = pos - 1 - (G - 1);
            for (; drained <= done_upto; ++drained) {
                const int64_t x = drained;
                mbar_wait(smem_u32(&slot_full[x % R]), static_cast<uint32_t>((x / R) & 1));
                tc_fence_after();
                const uint32_t col = slot_col(x, R, KP);
                const int sl = static_cast<int>(x % kMaxSlots);
                if (ring_real[sl]) {
                    const int64_t nn = ring_n[sl];
                    const int64_t q = ring_j[sl] * kTileQ + quarter * 32 + lane;
                    for (int kb = 0; kb < KP; kb += 16) {
                        uint32_t v[16];
                        tmem_ld16(lane_base + col + kb, v);
                        tmem_ld_wait();
                        if (q < p.out_w) {
#pragma unroll
                            for (int j = 0; j < 16; ++j) {
                                const int64_t o = p.k_begin + kb + j;
                                if (o < p.out_ch) p.out[(nn * p.out_ch + o) * p.out_w + q] = __uint_as_float(v[j]);
                            }
                        }
                    }
                }
                uint32_t z[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) z[j] = 0;
                for (int kb = 0; kb < KP; kb += 16) tmem_st16(lane_base + col + kb, z);
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&slot_empty[x % R]));
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 2) tmem_dealloc<kTmemCols>(tmem);
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
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

bool tc_conv_supported(const ConvGeom& g) {
    Plan pl;
    return make_plan(g, &pl);
}

size_t tc_conv_workspace_bytes(const ConvGeom& g) {
    Plan pl;
    if (!make_plan(g, &pl)) return 0;
    return static_cast<size_t>(pl.kgroups) * static_cast<size_t>(g.in_ch) * pl.b_chan_bytes;
}

cudaError_t launch_tc_conv(const uint16_t* in_bf16, const float* wg, float* out, const ConvGeom& g, void* workspace,
                           cudaStream_t stream) {
    Plan pl;
    if (!make_plan(g, &pl)) return cudaErrorNotSupported;
    auto encode = get_encode_fn();
    if (!encode) return cudaErrorNotSupported;
    uint16_t* img = static_cast<uint16_t*>(workspace);
    {
        const int64_t total = static_cast<int64_t>(pl.kgroups) * g.in_ch * pl.ntot * kTapsPerBlock;
        const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(total, 256), 4096));
        pack_bimg_kernel<<<blocks, 256, 0, stream>>>(wg, img, g.out_ch, g.in_ch, g.taps, pl.kp, pl.g, pl.kgroups);
        note_launch();
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    CUtensorMap tmap;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(g.in_w), static_cast<cuuint64_t>(g.n * g.in_ch)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(g.in_w) * 2};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(kSegQ), 1};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<uint16_t*>(in_bf16), dims, strides,
                        box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(tc_conv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(pl.smem_bytes));
    if (e != cudaSuccess) return e;
    KParams kp{};
    kp.n_items = g.n;
    kp.in_ch = g.in_ch;
    kp.in_w = g.in_w;
    kp.out_ch = g.out_ch;
    kp.out_w = g.out_w;
    kp.in_off = g.in_off;
    kp.tiles_per_item = ceil_div(g.out_w, kTileQ);
    kp.total_tiles = g.n * kp.tiles_per_item;
    kp.taps = static_cast<int>(g.taps);
    kp.pl = pl;
    kp.out = out;
    const int grid = static_cast<int>(std::min<int64_t>(num_sms(), kp.total_tiles));
    for (int kg = 0; kg < pl.kgroups; ++kg) {
        kp.k_begin = kg * pl.kp;
        kp.bimg = img + static_cast<size_t>(kg) * g.in_ch * (pl.b_chan_bytes / 2);
        tc_conv_kernel<<<grid, kThreads, pl.smem_bytes, stream>>>(tmap, kp);
        note_launch();
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace c1d
