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
#include <cstdlib>
#include <vector>

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
    uint32_t acc2;   // TMEM column offset of the second accumulator region (0 = none)
    // Tail taps (the last, partly filled tap block): instead of a 16-tap block per channel that
    // is mostly zero, one MMA per (tile, stage) contracts tail x cc (tap, channel) pairs (K <= 16)
    // from a q-chunk-major copy of the stage's channels (4-D TMA box), into the same slot.
    int tail;              // taps in the last block (0 = off: the last block is a regular block)
    int tail_chunks;       // q-chunks (8 columns x cc channels) of the tail box
    uint32_t tx_stage_bytes, tw_stage_bytes;  // tail X box / tail weight image per stage
    // Double-buffered TMEM (narrow filter blocks): super-tiles alternate between two 256-column
    // regions, so the epilogue's output stores overlap the next super-tile's MMAs; the MMA only
    // waits for the carry of the G-1 partial slots into the other region.
    int dbuf;
};

struct KParams {
    int64_t n_items, in_ch, in_w, out_ch, out_w, in_off;
    const uint16_t* bimg_tail;  // this filter group's tail image: [chunk][KP rows][16] bf16
    int64_t tiles_per_item, total_tiles;
    int taps, k_begin;
    Plan pl;
    const uint16_t* bimg;  // this filter group's B image: [in_ch][ntot*16] bf16
    int64_t main_ch;       // channels < main_ch -> region 0, others -> region acc2 (split FP32)
    float* out;
    unsigned long long* prof;  // optional per-CTA cycle counters (C1D_PROFILE=1), else nullptr
};

bool make_plan(const ConvGeom& g, Plan* pl, int64_t main_ch = 0) {
    const bool two_regions = main_ch > 0;
    if (g.dil != 8) return false;
    const int64_t pitch = g.in_stride ? g.in_stride : g.in_w;
    if (pitch % 8 != 0 || pitch < g.in_w || g.in_w < 8) return false;  // TMA global stride: multiple of 16 B
    if (g.n * g.in_ch >= (int64_t{1} << 31) || g.in_w >= (int64_t{1} << 31)) return false;
    Plan p{};
    p.kp = g.out_ch <= 16 ? 16 : (g.out_ch <= 32 ? 32 : 64);
    p.kgroups = static_cast<int>(ceil_div(g.out_ch, p.kp));
    p.g = static_cast<int>(ceil_div(g.taps, kTapsPerBlock));
    p.r = static_cast<int>(kTmemCols) / p.kp;
    p.ntot = p.g * p.kp;
    if (p.ntot > 256) return false;  // one MMA covers all tap blocks of a tile
    p.t = std::min(8, p.r - (p.g - 1));  // linear TMEM: T + G - 1 slots
    p.acc2 = 0;
    p.dbuf = 0;
    if (two_regions) {  // two accumulator regions of 256 columns each
        p.t = std::min(p.t, 256 / p.kp - (p.g - 1));
        p.acc2 = 256;
    } else if (std::min(8, 256 / p.kp - (p.g - 1)) >= 4 && getenv("C1D_NO_DBUF") == nullptr) {
        p.t = std::min(8, 256 / p.kp - (p.g - 1));
        p.dbuf = 1;
    }
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
    // tail path: wide filter blocks only (the N = (G-1)*KP main MMA stays >= 128) and the stage's
    // (tap, channel) pairs must fit one K = 16 MMA; in split mode stages may not straddle main_ch
    p.tail = 0;
    {
        const int tail = static_cast<int>(g.taps - static_cast<int64_t>(kTapsPerBlock) * (p.g - 1));
        if (p.g >= 2 && p.kp == 64 && (p.g - 1) * p.kp >= 128 && tail * p.cc <= kTapsPerBlock &&
            (!two_regions || main_ch % p.cc == 0) && getenv("C1D_NO_TAIL") == nullptr) {
            p.tail = tail;
            p.tail_chunks = 16 * p.t + static_cast<int>(ceil_div(kTapsPerBlock, p.cc));
        }
    }
    p.x_stage_bytes = static_cast<uint32_t>(p.cc * p.xw * 2);
    p.w_stage_bytes = static_cast<uint32_t>(p.cc) * p.b_chan_bytes;
    p.tx_stage_bytes = p.tail ? ((static_cast<uint32_t>(p.tail_chunks * p.cc * 16) + 1023) & ~1023u) : 0;
    p.tw_stage_bytes = p.tail ? static_cast<uint32_t>(p.kp * kTapsPerBlock * 2) : 0;
    const uint32_t stage = p.x_stage_bytes + p.w_stage_bytes + p.tx_stage_bytes + p.tw_stage_bytes;
    p.stages = static_cast<int>(std::min<uint32_t>(kMaxStages, (200 * 1024) / stage));
    if (p.stages < 2) return false;
    p.smem_bytes = static_cast<size_t>(p.stages) * stage + 1024;
    *pl = p;
    return true;
}

// ---------------------------------------------------------------------------- B image packing
// Weight value (o, i, s) of the forward-shaped problem: from prepped (o, i, s) weights, or straight
// from the caller's KCS weights for backward-data (o = c, i = k, taps reversed; tensor.cpp:23-41)
// so the separate prep launch disappears. BF16 RNE happens in the packing (bf16.hpp:29-40).
__device__ __forceinline__ float wval(const float* __restrict__ w, int bwd_raw, int64_t O, int64_t I, int64_t S,
                                      int64_t o, int64_t i, int64_t s) {
    return bwd_raw ? w[(i * O + o) * S + (S - 1 - s)] : w[(o * I + i) * S + s];
}

// One launch packs both images, in the K-major SWIZZLE_NONE core-matrix order
//   element (row, r) at (row/8)*128 + (r/8)*64 + (row%8)*8 + (r%8)   (SBO 256 B, LBO 128 B):
//  main: img[kg][c][row][r], row = b*KP + o, block b holds tap block G-1-b: input tile i0+t then
//        writes output slot t+b (column (t+b)*KP), because tap block g of tile p lands on tile p-g.
//  tail: timg[kg][chunk h][row o][k], k = r*cc + c: tap 16(G-1) + r of channel h*cc + c, zero for
//        k >= tail*cc or past C / K (the tail-tap MMAs, see Plan::tail).
__global__ void pack_images_kernel(const float* __restrict__ w, int bwd_raw, uint16_t* __restrict__ img,
                                   uint16_t* __restrict__ timg, int64_t out_ch, int64_t in_ch, int64_t taps, int kp,
                                   int g, int kgroups, int cc, int tail, int64_t chunks) {
    const int64_t ntot = static_cast<int64_t>(g) * kp;
    const int64_t per_chan = ntot * kTapsPerBlock;
    const int64_t main_total = static_cast<int64_t>(kgroups) * in_ch * per_chan;
    const int64_t per_tail = static_cast<int64_t>(kp) * kTapsPerBlock;
    const int64_t total = main_total + (tail ? static_cast<int64_t>(kgroups) * chunks * per_tail : 0);
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        if (e < main_total) {
            const int64_t r = e % kTapsPerBlock;
            const int64_t row = (e / kTapsPerBlock) % ntot;
            const int64_t c = (e / per_chan) % in_ch;
            const int64_t kg = e / (per_chan * in_ch);
            const int64_t blk = row / kp, o = kg * kp + row % kp, s = (g - 1 - blk) * kTapsPerBlock + r;
            float v = 0.0f;
            if (o < out_ch && s < taps) v = wval(w, bwd_raw, out_ch, in_ch, taps, o, c, s);
            const int64_t off = (row / 8) * 128 + (r / 8) * 64 + (row % 8) * 8 + (r % 8);
            img[(kg * in_ch + c) * per_chan + off] = fp32_to_bf16_bits(v);
        } else {
            const int64_t f = e - main_total;
            const int64_t k = f % kTapsPerBlock;
            const int64_t row = (f / kTapsPerBlock) % kp;
            const int64_t h = (f / per_tail) % chunks;
            const int64_t kg = f / (per_tail * chunks);
            const int64_t rr = k / cc, c = h * cc + k % cc, o = kg * kp + row;
            const int64_t s = static_cast<int64_t>(g - 1) * kTapsPerBlock + rr;
            float v = 0.0f;
            if (rr < tail && c < in_ch && o < out_ch && s < taps) v = wval(w, bwd_raw, out_ch, in_ch, taps, o, c, s);
            const int64_t off = (row / 8) * 128 + (k / 8) * 64 + (row % 8) * 8 + (k % 8);
            timg[(kg * chunks + h) * per_tail + off] = fp32_to_bf16_bits(v);
        }
    }
}

// ---------------------------------------------------------------------------- schedule
// Each CTA owns output tiles [b, e) of the flattened (item, tile) list. For each item segment
// (n, j0..j1) it walks input tiles j0 .. j1+G-1 in super-tiles of up to T tiles. Input tile
// i0+t of a super-tile writes output tiles i0+t-G+1 .. i0+t, which live at TMEM slots t..t+G-1
// (slot j <-> output i0-(G-1)+j, KP columns per slot): every MMA is one contiguous N = G*KP run.
struct Cursor {
    int64_t cur, end;         // flattened output-tile cursor
    int64_t n, j0, j1;        // current segment
    int64_t i;                // next input tile in the segment
    bool valid;
};

struct Super {
    int64_t n, i0, j0, j1;
    int tcur;
    bool last_in_segment;
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

__device__ __forceinline__ bool next_super(Cursor& c, int64_t J, int G, int T, Super* s) {
    if (!c.valid) return false;
    if (c.i > c.j1 + G - 1) {
        if (!next_segment(c, J)) {
            c.valid = false;
            return false;
        }
    }
    const int64_t remain = c.j1 + G - 1 - c.i + 1;
    s->tcur = static_cast<int>(imin64(T, remain));
    s->n = c.n;
    s->i0 = c.i;
    s->j0 = c.j0;
    s->j1 = c.j1;
    c.i += s->tcur;
    s->last_in_segment = c.i > c.j1 + G - 1;
    return true;
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

__global__ void __launch_bounds__(kThreads, 1)
    tc_conv_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap tmap_tail,
                   const KParams p) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint64_t stage_full[kMaxStages], stage_empty[kMaxStages];
    __shared__ uint64_t tmem_full, tmem_empty;
    __shared__ uint32_t tmem_base_s;

    const Plan& pl = p.pl;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t* xs_base = smem;
    uint8_t* ws_base = smem + static_cast<size_t>(pl.stages) * pl.x_stage_bytes;
    uint8_t* tx_base = ws_base + static_cast<size_t>(pl.stages) * pl.w_stage_bytes;
    uint8_t* tw_base = tx_base + static_cast<size_t>(pl.stages) * pl.tx_stage_bytes;
    const int G = pl.g, T = pl.t, KP = pl.kp;
    const int64_t J = p.tiles_per_item;
    const int n_chunks = static_cast<int>(ceil_div(p.in_ch, pl.cc));

    if (threadIdx.x == 0) {
        for (int s = 0; s < pl.stages; ++s) {
            mbar_init(&stage_full[s], 1);
            mbar_init(&stage_empty[s], 1);
        }
        mbar_init(&tmem_full, 1);
        mbar_init(&tmem_empty, 4);  // one arrival per epilogue warp
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
            if (pl.tail) prefetch_tmap(&tmap_tail);
            long long t_wait = 0;
            const long long t_begin = clock64();
            Cursor cur = make_cursor(p);
            int stage = 0;
            uint32_t phase = 0;
            Super su;
            while (next_super(cur, J, G, T, &su)) {
                const int32_t x_start = static_cast<int32_t>(su.i0 * kTileQ + p.in_off);
                const int nseg = static_cast<int>(ceil_div(su.tcur * kTileQ + 8 * (kTapsPerBlock - 1), kSegQ));
                for (int ch = 0; ch < n_chunks; ++ch) {
                    const int c0 = ch * pl.cc;
                    const int ccn = static_cast<int>(imin64(pl.cc, p.in_ch - c0));
                    const long long tw0 = clock64();
                    mbar_wait(smem_u32(&stage_empty[stage]), phase ^ 1);
                    t_wait += clock64() - tw0;
                    const uint32_t full = smem_u32(&stage_full[stage]);
                    const uint32_t bytes = static_cast<uint32_t>(ccn) * (nseg * kSegQ * 2 + pl.b_chan_bytes) +
                                           (pl.tail ? pl.tail_chunks * pl.cc * 16u + pl.tw_stage_bytes : 0u);
                    mbar_arrive_expect_tx(full, bytes);
                    const uint32_t xs = smem_u32(xs_base + static_cast<size_t>(stage) * pl.x_stage_bytes);
                    for (int c = 0; c < ccn; ++c) {
                        const int32_t row = static_cast<int32_t>(su.n * p.in_ch + c0 + c);
                        for (int sg = 0; sg < nseg; ++sg)
                            tma_load_2d(xs + static_cast<uint32_t>((c * pl.xw + sg * kSegQ) * 2), &tmap,
                                        x_start + sg * kSegQ, row, full);
                    }
                    const uint32_t wsm = smem_u32(ws_base + static_cast<size_t>(stage) * pl.w_stage_bytes);
                    bulk_g2s(wsm, p.bimg + static_cast<size_t>(c0) * (pl.b_chan_bytes / 2),
                             static_cast<uint32_t>(ccn) * pl.b_chan_bytes, full);
                    if (pl.tail) {
                        // q-chunk-major box of the stage's cc channels over the same input tiles
                        // (tap block G-1 of input tile p lands on output slot t, like block 0 of B)
                        const uint32_t tx = smem_u32(tx_base + static_cast<size_t>(stage) * pl.tx_stage_bytes);
                        const int32_t chunk0 = x_start / 8;  // in_off is a multiple of 8
                        asm volatile(
                            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
                            "[%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(tx),
                            "l"(&tmap_tail), "r"(0), "r"(c0), "r"(chunk0), "r"(static_cast<int32_t>(su.n)), "r"(full)
                            : "memory");
                        const uint32_t tw = smem_u32(tw_base + static_cast<size_t>(stage) * pl.tw_stage_bytes);
                        bulk_g2s(tw, p.bimg_tail + static_cast<size_t>(ch) * (pl.tw_stage_bytes / 2), pl.tw_stage_bytes,
                                 full);
                    }
                    if (++stage == pl.stages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
            if (p.prof) {
                p.prof[blockIdx.x * 8 + 0] = t_wait;
                p.prof[blockIdx.x * 8 + 1] = clock64() - t_begin;
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------------ MMA issuer
        // The whole warp walks the schedule (warp-uniform control flow keeps descriptors in
        // uniform registers); one elected lane issues each tcgen05 instruction.
        long long t_full = 0, t_tmem = 0;
        const long long t_begin = clock64();
        Cursor cur = make_cursor(p);
        int stage = 0;
        uint32_t phase = 0, tphase = 0;
        // tail mode: the main MMA covers blocks 1..G-1 (slots t+1..t+G-1), the tail MMA slot t
        const int gm = pl.tail ? G - 1 : G;
        const uint32_t idesc = make_idesc(128, static_cast<uint32_t>(gm * KP), kFmtBF16, 1, 0);
        const uint32_t idesc_tail = make_idesc(128, static_cast<uint32_t>(KP), kFmtBF16, 1, 0);
        const uint32_t main_slot = pl.tail ? static_cast<uint32_t>(KP) : 0u;       // D column offset
        const uint32_t main_brow = pl.tail ? static_cast<uint32_t>(KP) * 32u : 0u;  // skip block 0 of B
        uint32_t region = 0;  // TMEM region of the current super-tile (double buffering)
        Super su;
        while (next_super(cur, J, G, T, &su)) {
            const long long ts0 = clock64();
            mbar_wait(smem_u32(&tmem_empty), tphase);
            tphase ^= 1;
            t_tmem += clock64() - ts0;
            tc_fence_after();
            const uint32_t rtmem = tmem + region;
            for (int ch = 0; ch < n_chunks; ++ch) {
                const int c0 = ch * pl.cc;
                const int ccn = static_cast<int>(imin64(pl.cc, p.in_ch - c0));
                const long long tf0 = clock64();
                mbar_wait(smem_u32(&stage_full[stage]), phase);
                t_full += clock64() - tf0;
                tc_fence_after();
                const uint32_t xs = smem_u32(xs_base + static_cast<size_t>(stage) * pl.x_stage_bytes);
                const uint32_t wsm = smem_u32(ws_base + static_cast<size_t>(stage) * pl.w_stage_bytes);
                const uint64_t a0 = make_smem_desc(xs, 128, 16, kLayoutNone);
                const uint64_t b0 = make_smem_desc(wsm + main_brow, 128, 256, kLayoutNone);
                if (elect_one()) {
                    uint64_t bdesc = b0;
                    uint64_t achan = a0;
                    for (int c = 0; c < ccn; ++c) {
                        uint64_t adesc = achan;
                        uint32_t dcol = rtmem + ((c0 + c >= p.main_ch) ? pl.acc2 : 0u) + main_slot;
                        for (int t = 0; t < su.tcur; ++t) {
                            mma_bf16_ss(dcol, adesc, bdesc, idesc, 1);
                            adesc = desc_advance(adesc, static_cast<uint32_t>(kTileQ * 2));
                            dcol += static_cast<uint32_t>(KP);
                        }
                        bdesc = desc_advance(bdesc, pl.b_chan_bytes);
                        achan = desc_advance(achan, static_cast<uint32_t>(pl.xw * 2));
                    }
                    if (pl.tail) {
                        // A[m][k = r*cc + c] = x[c][q0 + m + 8r] (tap 16(G-1) + r): MN-major, K rows
                        // 16 B apart (contiguous), M groups of 8 columns one q-chunk (cc*16 B) apart
                        const uint32_t tx = smem_u32(tx_base + static_cast<size_t>(stage) * pl.tx_stage_bytes);
                        const uint32_t tw = smem_u32(tw_base + static_cast<size_t>(stage) * pl.tw_stage_bytes);
                        uint64_t adesc = make_smem_desc(tx, 128, static_cast<uint32_t>(pl.cc * 16), kLayoutNone);
                        const uint64_t bt = make_smem_desc(tw, 128, 256, kLayoutNone);
                        uint32_t dcol = rtmem + ((c0 >= p.main_ch) ? pl.acc2 : 0u);
                        for (int t = 0; t < su.tcur; ++t) {
                            mma_bf16_ss(dcol, adesc, bt, idesc_tail, 1);
                            adesc = desc_advance(adesc, static_cast<uint32_t>(16 * pl.cc * 16));
                            dcol += static_cast<uint32_t>(KP);
                        }
                    }
                }
                __syncwarp();
                if (elect_one()) mma_commit(smem_u32(&stage_empty[stage]));
                __syncwarp();
                if (++stage == pl.stages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if (elect_one()) mma_commit(smem_u32(&tmem_full));
            __syncwarp();
            if (pl.dbuf) region ^= 256u;
        }
        if (p.prof && lane == 0) {
            p.prof[blockIdx.x * 8 + 2] = t_full;
            p.prof[blockIdx.x * 8 + 3] = t_tmem;
            p.prof[blockIdx.x * 8 + 4] = clock64() - t_begin;
        }
    } else if (warp >= 4) {
        // ------------------------------------------------------------------ epilogue
        const int quarter = warp - 4;  // TMEM lanes 32*quarter .. +31
        const uint32_t lane_base = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
        uint32_t z[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) z[j] = 0;
        for (uint32_t col = 0; col < kTmemCols; col += 16) tmem_st16(lane_base + col, z);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&tmem_empty));
        Cursor cur = make_cursor(p);
        uint32_t tphase = 0;
        Super su;
        long long e_store = 0, e_carry = 0, e_zero = 0;  // C1D_PROFILE counters
        uint32_t region = 0;  // mirrors the MMA warp's double-buffer region
        const uint32_t used_cols = static_cast<uint32_t>((T + G - 1) * KP);
        // carry the G-1 partial slots (tcur..tcur+G-2) of `src` into slots 0..G-2 of `dst` (or zero
        // them at a segment end) and zero dst's remaining used slots: dst is then ready
        auto prepare = [&](uint32_t src, uint32_t dst, const Super& s2) {
            for (uint32_t reg = 0; reg <= pl.acc2; reg += (pl.acc2 ? pl.acc2 : 1u)) {
                for (int j = 0; j < G - 1; ++j) {
                    for (int kb = 0; kb < KP; kb += 16) {
                        uint32_t v[16];
                        if (!s2.last_in_segment) {
                            tmem_ld16(lane_base + src + reg + static_cast<uint32_t>((s2.tcur + j) * KP + kb), v);
                            tmem_ld_wait();
                            tmem_st16(lane_base + dst + reg + static_cast<uint32_t>(j * KP + kb), v);
                        } else if (dst != src) {
                            tmem_st16(lane_base + dst + reg + static_cast<uint32_t>(j * KP + kb), z);
                        }
                    }
                }
                for (uint32_t col = static_cast<uint32_t>((G - 1) * KP); col < used_cols; col += 16)
                    tmem_st16(lane_base + dst + reg + col, z);
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&tmem_empty));
        };
        while (next_super(cur, J, G, T, &su)) {
            mbar_wait_sleep(smem_u32(&tmem_full), tphase, 256);
            tphase ^= 1;
            tc_fence_after();
            const long long e0 = clock64();
            if (pl.dbuf) prepare(region, region ^ 256u, su);  // next super-tile may start now
            const long long e1 = clock64();
            // store the completed outputs (slots 0..tcur-1)
            const int64_t out_w = p.out_w;
            float* const out_item = p.out + su.n * p.out_ch * out_w;
            for (int j = 0; j < su.tcur; ++j) {
                const int64_t o = su.i0 - (G - 1) + j;
                if (o < su.j0 || o > su.j1) continue;  // phantom (warm-up / beyond the segment)
                const int64_t q = o * kTileQ + quarter * 32 + lane;
                for (int kb = 0; kb < KP; kb += 16) {
                    uint32_t v[16];
                    tmem_ld16(lane_base + region + static_cast<uint32_t>(j * KP + kb), v);
                    tmem_ld_wait();
                    if (pl.acc2) {  // main term + the correction terms' separate accumulator
                        uint32_t v2[16];
                        tmem_ld16(lane_base + pl.acc2 + static_cast<uint32_t>(j * KP + kb), v2);
                        tmem_ld_wait();
#pragma unroll
                        for (int jj = 0; jj < 16; ++jj) v[jj] = __float_as_uint(__uint_as_float(v[jj]) + __uint_as_float(v2[jj]));
                    }
                    if (q < p.out_w) {
                        // running pointer: one add + one store per channel row (the stores, not the
                        // address math, should limit this loop: it shares sub-partitions with the
                        // TMA and MMA warps)
                        float* dst = out_item + (p.k_begin + kb) * out_w + q;
                        const int kvalid = static_cast<int>(imin64(16, p.out_ch - p.k_begin - kb));
#pragma unroll
                        for (int jj = 0; jj < 16; ++jj) {
                            if (jj < kvalid) *dst = __uint_as_float(v[jj]);
                            dst += out_w;
                        }
                    }
                }
            }
            const long long e2 = clock64();
            e_store += e2 - e1;
            if (!pl.dbuf) {
                prepare(0, 0, su);  // in place: carry down, zero the rest, release
                e_carry += clock64() - e2;
            } else {
                e_carry += e1 - e0;
                region ^= 256u;
            }
        }
        if (p.prof && threadIdx.x == 128) {
            p.prof[blockIdx.x * 8 + 5] = e_store;
            p.prof[blockIdx.x * 8 + 6] = e_carry;
            p.prof[blockIdx.x * 8 + 7] = e_zero;
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

bool tc_conv_supported(const ConvGeom& g, int64_t main_ch) {
    Plan pl;
    return make_plan(g, &pl, main_ch);
}

size_t tc_conv_workspace_bytes(const ConvGeom& g, int64_t main_ch) {
    Plan pl;
    if (!make_plan(g, &pl, main_ch)) return 0;
    const size_t tail = pl.tail ? static_cast<size_t>(pl.kgroups) * ceil_div(g.in_ch, pl.cc) * pl.tw_stage_bytes : 0;
    return static_cast<size_t>(pl.kgroups) * static_cast<size_t>(g.in_ch) * pl.b_chan_bytes + ((tail + 255) & ~size_t{255});
}

cudaError_t launch_tc_conv(const uint16_t* in_bf16, const float* wg, float* out, const ConvGeom& g, void* workspace,
                           cudaStream_t stream, int64_t main_ch, bool w_bwd_raw) {
    Plan pl;
    if (!make_plan(g, &pl, main_ch)) return cudaErrorNotSupported;
    auto encode = get_encode_fn();
    if (!encode) return cudaErrorNotSupported;
    uint16_t* img = static_cast<uint16_t*>(workspace);
    const int64_t n_chunks = ceil_div(g.in_ch, pl.cc);
    uint16_t* img_tail = img + static_cast<size_t>(pl.kgroups) * g.in_ch * (pl.b_chan_bytes / 2);
    {
        const int64_t total = static_cast<int64_t>(pl.kgroups) *
                              (g.in_ch * pl.ntot + (pl.tail ? n_chunks * pl.kp : 0)) * kTapsPerBlock;
        const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(total, 256), 4096));
        pack_images_kernel<<<blocks, 256, 0, stream>>>(wg, w_bwd_raw ? 1 : 0, img, img_tail, g.out_ch, g.in_ch, g.taps,
                                                       pl.kp, pl.g, pl.kgroups, pl.cc, pl.tail, n_chunks);
        note_launch();
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    CUtensorMap tmap;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(g.in_w), static_cast<cuuint64_t>(g.n * g.in_ch)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(g.in_stride ? g.in_stride : g.in_w) * 2};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(kSegQ), 1};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<uint16_t*>(in_bf16), dims, strides,
                        box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    CUtensorMap tmap_tail = tmap;  // unused unless pl.tail
    if (pl.tail) {
        // the input as (8 columns, channel, q-chunk, item): element (e, c, u, n) at ((n*C + c)*pitch + 8u + e)
        const int64_t pitch = g.in_stride ? g.in_stride : g.in_w;
        const cuuint64_t d4[4] = {8, static_cast<cuuint64_t>(g.in_ch), static_cast<cuuint64_t>(pitch / 8),
                                  static_cast<cuuint64_t>(g.n)};
        const cuuint64_t s4[3] = {static_cast<cuuint64_t>(pitch) * 2, 16, static_cast<cuuint64_t>(g.in_ch * pitch) * 2};
        const cuuint32_t b4[4] = {8, static_cast<cuuint32_t>(pl.cc), static_cast<cuuint32_t>(pl.tail_chunks), 1};
        const cuuint32_t e4[4] = {1, 1, 1, 1};
        r = encode(&tmap_tail, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<uint16_t*>(in_bf16), d4, s4, b4, e4,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    }
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
    kp.main_ch = main_ch > 0 ? main_ch : g.in_ch;
    kp.pl = pl;
    kp.out = out;
    const int grid = static_cast<int>(std::min<int64_t>(num_sms(), kp.total_tiles));
    static const bool profile = getenv("C1D_PROFILE") != nullptr;
    if (profile) {
        cudaMalloc(&kp.prof, sizeof(unsigned long long) * 8 * grid);
        cudaMemset(kp.prof, 0, sizeof(unsigned long long) * 8 * grid);
    }
    for (int kg = 0; kg < pl.kgroups; ++kg) {
        kp.k_begin = kg * pl.kp;
        kp.bimg = img + static_cast<size_t>(kg) * g.in_ch * (pl.b_chan_bytes / 2);
        kp.bimg_tail = img_tail + static_cast<size_t>(kg) * n_chunks * (pl.tw_stage_bytes / 2);
        tc_conv_kernel<<<grid, kThreads, pl.smem_bytes, stream>>>(tmap, tmap_tail, kp);
        note_launch();
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    if (profile) {
        std::vector<unsigned long long> h(8 * grid);
        cudaMemcpy(h.data(), kp.prof, h.size() * 8, cudaMemcpyDeviceToHost);
        double a[8] = {0};
        for (int b = 0; b < grid; ++b)
            for (int i = 0; i < 8; ++i) a[i] += static_cast<double>(h[b * 8 + i]) / grid;
        fprintf(stderr, "[tc_conv prof] producer wait_empty %.0f / total %.0f | mma wait_full %.0f wait_slot %.0f total %.0f | epilogue store %.0f carry %.0f zero %.0f (cycles, CTA avg)\n",
                a[0], a[1], a[2], a[3], a[4], a[5], a[6], a[7]);
        cudaFree(kp.prof);
    }
    return cudaSuccess;
}

}  // namespace c1d
