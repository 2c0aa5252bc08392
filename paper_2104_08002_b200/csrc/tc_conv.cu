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
__host__ __device__ __forceinline__ int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }

constexpr int kTileQ = 128;      // output columns per tile (MMA M)
constexpr int kSegQ = 256;       // TMA box width in elements
constexpr int kTapsPerBlock = 16;
constexpr int kMaxStages = 6;
constexpr int kMaxStagger = 2;  // trailing chunks of a super-tile issued tile-major (Plan::stagger)

constexpr int kPfRing = 4;  // layer glue: input blocks in flight per epilogue warp
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
    // Expanded-row mode (dilation 1, 2, 4; ConvGeom.xr_rows): the input is the row tensor E (one
    // tap = one 16-B row, 8 output columns = 8/d rows). Each output tile accumulates its G tap
    // blocks directly (one N = KP MMA per (channel, block, tile) at row offset 128t/d + 16g), so
    // there is no carry: the schedule runs with one "block" and T slots per super-tile.
    int xr;          // dilation of the expanded rows (0 = natural rows, d = 8)
    int rows_alloc;  // E rows per channel in a stage (n_box * box_rows)
    int box_rows;    // rows per TMA box
    int n_box;       // boxes per channel
    // inline expansion: the producer loads natural windows (raw_segs 256-column boxes per channel,
    // from a 16-B aligned start) and warps 2-3 write E's rows into the stage
    int xin;
    int rows_stage;       // E rows the MMAs read per channel
    int raw_segs;         // 256-column boxes per channel window
    uint32_t raw_stage_bytes;
    // Resident weights: when the whole B image of a launch is small (narrow layers, e.g. C = K = 15:
    // 30 KB), it is loaded once per CTA into the front of shared memory instead of with every stage
    uint32_t wres_bytes;  // 0 = weights streamed per stage
    // Natural mode: a stage's cc channel windows as ONE 3-D TMA box (256 columns, n_seg segments,
    // cc rows) through an overlapping view whose segment stride is 512 B, instead of cc * n_seg
    // single-row boxes (each TMA box costs the producer ~100 cycles); only for windows inside
    // [0, in_w), since the view's bounds are checked per dimension (edge windows keep the 2-D boxes)
    int xbox3;
    // Weight-stationary main MMAs (tcgen05.mma.ws, B latched in the collector across a channel's
    // tiles): only where the main MMA is N = 64 (KP = 16 narrow layers; sm100.cuh mma_ws_*)
    int ws;
    // Staggered finish (single-buffered carry plans, KP >= 32): the last `stagger` channel chunks of a
    // super-tile are issued tile by tile, each tile committing its own barrier, so the epilogue stores
    // output tile t while the MMAs of tiles t+1.. still run (with all 512 TMEM columns in one
    // super-tile nothing else overlaps the stores). Each accumulator sees its chunks in the same order.
    // The count does not depend on the stage count (every plan has >= 2 stages), so a glued pass,
    // whose epilogue staging leaves fewer stages, accumulates in the same order as the plain pass.
    int stagger;
};

constexpr uint32_t kWresMax = 64 * 1024;

// Resident-weight decision for a plan whose b_chan_bytes / cc are set (stages are sized afterwards)
inline bool want_wres(const ConvGeom& g, uint32_t b_chan_bytes, bool allow) {
    return allow && static_cast<uint64_t>(g.in_ch) * b_chan_bytes <= kWresMax && !dev_switch(DevSwitch::kNoWres);
}
inline void plan_wres(const ConvGeom& g, Plan* p, bool allow) {
    const uint64_t img = static_cast<uint64_t>(g.in_ch) * p->b_chan_bytes;
    p->wres_bytes = want_wres(g, p->b_chan_bytes, allow) ? static_cast<uint32_t>((img + 1023) & ~1023ull) : 0u;
    if (p->wres_bytes) p->w_stage_bytes = 0;
}

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
    // resident image prepacked by the caller (c1d_pack_weights, written before the previous launch
    // on the stream): its bulk load is issued before the PDL wait, overlapping the previous kernel
    int early_w;
    LayerGlue glue;            // mode 0: plain FP32 store of `out`
    // glue outputs through shared-memory staging + TMA stores: slot bits 1 = fp32 A (pre / gsum),
    // 2 = fp32 B (act / gp), 4 = bf16 C (act_bf16 / gp_bf16); 0 = per-lane global stores
    uint32_t tma_slots;
    uint32_t stg_off;    // staging area offset in the aligned dynamic shared memory
    uint32_t stg_bytes;  // one staging buffer (each epilogue warp owns two)
    uint32_t stg_a, stg_b, stg_c;  // slot offsets inside a buffer
    // glue inputs (skip / gadd rows, mask words) prefetched kPfRing blocks ahead with cp.async into
    // per-warp rings: pf_rows / pf_mask = slot has 16 x 32 fp32 rows / 32 mask words
    uint32_t pf_off, pf_slot_bytes, pf_rows, pf_mask;
    uint32_t pf_vec;  // prefetch rows as 16-B pieces (width, column offset and base 16-B compatible)
};

bool make_plan_xr(const ConvGeom& g, Plan* pl, int64_t main_ch, uint32_t reserve, bool allow_wres = true) {
    // d = 8 joins as the inline case whose rows are the natural window itself (no expansion)
    if (g.dil != 1 && g.dil != 2 && g.dil != 4 && !(g.dil == 8 && g.xr_inline)) return false;
    if (g.dil == 8 && g.in_off % 8) return false;
    if (g.n * g.in_ch >= (int64_t{1} << 31) || g.xr_rows >= (int64_t{1} << 31)) return false;
    Plan p{};
    p.xr = static_cast<int>(g.dil);
    // N = KP per MMA here, so wide filter blocks pay: KP = 128 halves the A-tile re-reads per filter
    // and reads E once (one filter group) — single-buffered, 4 tiles per super-tile
    p.kp = g.out_ch <= 16 ? 16 : (g.out_ch <= 32 ? 32 : (g.out_ch <= 64 ? 64 : 128));
    p.kgroups = static_cast<int>(ceil_div(g.out_ch, p.kp));
    p.g = static_cast<int>(ceil_div(g.taps, kTapsPerBlock));
    p.r = static_cast<int>(kTmemCols) / p.kp;
    p.ntot = p.g * p.kp;
    if (p.ntot > 1024) return false;
    p.t = std::min(8, 256 / p.kp);  // no carry: T slots per 256-column region, double-buffered
    p.dbuf = !dev_switch(DevSwitch::kNoDbuf) && p.kp <= 64 ? 1 : 0;
    if (!p.dbuf) p.t = std::min(8, p.r);
    p.acc2 = 0;
    if (main_ch > 0) {  // split FP32: the second 256-column region holds the correction terms
        p.dbuf = 0;
        p.t = std::min(8, 256 / p.kp);
        p.acc2 = 256;
    }
    p.tail = 0;
    // E is read as (64 elements = 8 rows, row octets, item x channel) boxes: 128-B inner box rows
    // keep TMA on its fast path (16-B inner rows run at a third of the rate)
    if (!g.xr_inline && g.xr_rows % 8) return false;
    const int rows_stage = static_cast<int>(ceil_div(p.t * (kTileQ / p.xr) + kTapsPerBlock * p.g, 8) * 8);
    p.rows_stage = rows_stage;
    p.box_rows = std::min(256 * 8, rows_stage);
    p.n_box = static_cast<int>(ceil_div(rows_stage, p.box_rows));
    p.rows_alloc = p.n_box * p.box_rows;
    p.xin = g.xr_inline ? 1 : 0;
    if (p.xin) {
        const int64_t pitch = g.in_stride ? g.in_stride : g.in_w;
        if (pitch % 8 || pitch < g.in_w) return false;
        // window: up to 7 leading columns of alignment + the rows' reach + one 16-B read of slack
        p.raw_segs = static_cast<int>(ceil_div(7 + (rows_stage - 1) * p.xr + 8 + 8, kSegQ));
        p.rows_alloc = p.xr == 8 ? 0 : rows_stage;  // d = 8: the MMAs read the raw window
    }
    p.n_seg = 0;
    p.xw = 0;
    p.b_chan_bytes = static_cast<uint32_t>(p.ntot * kTapsPerBlock * 2);
    const uint32_t raw_chan = p.xin ? static_cast<uint32_t>(p.raw_segs * kSegQ * 2) : 0u;
    const bool wres = want_wres(g, p.b_chan_bytes, allow_wres);
    const uint32_t per_chan = static_cast<uint32_t>(p.rows_alloc * 16) + (wres ? 0u : p.b_chan_bytes) + raw_chan;
    p.cc = static_cast<int>(std::max<uint32_t>(1, std::min<uint32_t>(48 * 1024 / per_chan, 16)));
    p.cc = static_cast<int>(std::min<int64_t>(p.cc, g.in_ch));
    {
        const int64_t nch = ceil_div(g.in_ch, p.cc);
        p.cc = static_cast<int>(ceil_div(g.in_ch, nch));
    }
    p.x_stage_bytes = static_cast<uint32_t>(p.cc * p.rows_alloc * 16);
    p.w_stage_bytes = static_cast<uint32_t>(p.cc) * p.b_chan_bytes;
    p.tx_stage_bytes = p.tw_stage_bytes = 0;
    p.raw_stage_bytes = static_cast<uint32_t>(p.cc) * raw_chan;
    plan_wres(g, &p, allow_wres);
    const uint32_t stage = p.x_stage_bytes + p.w_stage_bytes + p.raw_stage_bytes;
    p.stages = static_cast<int>(std::min<uint32_t>(kMaxStages, (200 * 1024 - reserve - p.wres_bytes) / stage));
    if (p.stages < 2) return p.wres_bytes ? make_plan_xr(g, pl, main_ch, reserve, false) : false;
    p.smem_bytes = p.wres_bytes + static_cast<size_t>(p.stages) * stage + 1024;
    *pl = p;
    return true;
}

bool make_plan(const ConvGeom& g, Plan* pl, int64_t main_ch = 0, uint32_t reserve = 0, bool allow_wres = true) {
    if (g.xr_rows > 0 || g.xr_inline) return make_plan_xr(g, pl, main_ch, reserve, allow_wres);
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
    } else if (std::min(8, 256 / p.kp - (p.g - 1)) >= 4 && !dev_switch(DevSwitch::kNoDbuf)) {
        p.t = std::min(8, 256 / p.kp - (p.g - 1));
        p.dbuf = 1;
    }
    if (p.t < 1) return false;
    p.n_seg = static_cast<int>(ceil_div(p.t * kTileQ + 8 * (kTapsPerBlock - 1), kSegQ));
    p.xw = p.n_seg * kSegQ;
    p.b_chan_bytes = static_cast<uint32_t>(p.ntot * kTapsPerBlock * 2);
    const bool wres = want_wres(g, p.b_chan_bytes, allow_wres);
    const uint32_t per_chan = static_cast<uint32_t>(p.xw * 2) + (wres ? 0u : p.b_chan_bytes);
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
            (!two_regions || main_ch % p.cc == 0) && !dev_switch(DevSwitch::kNoTail)) {
            p.tail = tail;
            p.tail_chunks = 16 * p.t + static_cast<int>(ceil_div(kTapsPerBlock, p.cc));
        }
    }
    p.x_stage_bytes = static_cast<uint32_t>(p.cc * p.xw * 2);
    p.w_stage_bytes = static_cast<uint32_t>(p.cc) * p.b_chan_bytes;
    p.tx_stage_bytes = p.tail ? ((static_cast<uint32_t>(p.tail_chunks * p.cc * 16) + 1023) & ~1023u) : 0;
    p.tw_stage_bytes = p.tail ? static_cast<uint32_t>(p.kp * kTapsPerBlock * 2) : 0;
    plan_wres(g, &p, allow_wres);
    p.ws = (p.tail ? p.g - 1 : p.g) * p.kp == 64 && !dev_switch(DevSwitch::kNoWs) ? 1 : 0;
    const uint32_t stage = p.x_stage_bytes + p.w_stage_bytes + p.tx_stage_bytes + p.tw_stage_bytes;
    p.stages = static_cast<int>(std::min<uint32_t>(kMaxStages, (200 * 1024 - reserve - p.wres_bytes) / stage));
    if (p.stages < 2) return p.wres_bytes ? make_plan(g, pl, main_ch, reserve, false) : false;
    p.smem_bytes = p.wres_bytes + static_cast<size_t>(p.stages) * stage + 1024;
    p.stagger = (!p.dbuf && p.kp >= 32 && !dev_switch(DevSwitch::kNoStagger))
                    ? static_cast<int>(std::min<int64_t>(std::min(kMaxStagger, p.stages), ceil_div(g.in_ch, p.cc)))
                    : 0;
    *pl = p;
    return true;
}

// ---------------------------------------------------------------------------- B image packing
// Weight value (o, i, s) of the forward-shaped problem: from prepped (o, i, s) weights, or straight
// from the caller's KCS weights for backward-data (o = c, i = k, taps reversed; tensor.cpp:23-41)
// so the separate prep launch disappears. BF16 RNE happens in the packing (bf16.hpp:29-40).
template <typename Ix>
__device__ __forceinline__ float wval(const float* __restrict__ w, int bwd_raw, Ix O, Ix I, Ix S, Ix o, Ix i, Ix s) {
    return bwd_raw ? w[(i * O + o) * S + (S - 1 - s)] : w[(o * I + i) * S + s];
}

// One launch packs both images, in the K-major SWIZZLE_NONE core-matrix order
//   element (row, r) at (row/8)*128 + (r/8)*64 + (row%8)*8 + (r%8)   (SBO 256 B, LBO 128 B):
//  main: img[kg][c][row][r], row = b*KP + o, block b holds tap block G-1-b: input tile i0+t then
//        writes output slot t+b (column (t+b)*KP), because tap block g of tile p lands on tile p-g.
//  tail: timg[kg][chunk h][row o][k], k = r*cc + c: tap 16(G-1) + r of channel h*cc + c, zero for
//        k >= tail*cc or past C / K (the tail-tap MMAs, see Plan::tail).
// Index type Ix: 32-bit when every element index fits (always, in practice): 64-bit divisions per
// element made this launch ~7 us for images of ~15k elements.
template <typename Ix>
__global__ void pack_images_kernel(const float* __restrict__ w, int bwd_raw, uint16_t* __restrict__ img,
                                   uint16_t* __restrict__ timg, int64_t out_ch_, int64_t in_ch_, int64_t taps_, int kp,
                                   int g, int kgroups, int cc, int tail, int64_t chunks_) {
    const Ix out_ch = static_cast<Ix>(out_ch_), in_ch = static_cast<Ix>(in_ch_), taps = static_cast<Ix>(taps_);
    const Ix chunks = static_cast<Ix>(chunks_);
    const Ix ntot = static_cast<Ix>(g) * kp;
    const Ix per_chan = ntot * kTapsPerBlock;
    const Ix main_total = static_cast<Ix>(kgroups) * in_ch * per_chan;
    const Ix per_tail = static_cast<Ix>(kp) * kTapsPerBlock;
    const Ix total = main_total + (tail ? static_cast<Ix>(kgroups) * chunks * per_tail : 0);
    pdl_trigger();
    pdl_wait();
    for (Ix e = static_cast<Ix>(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += static_cast<Ix>(gridDim.x) * blockDim.x) {
        if (e < main_total) {
            const Ix r = e % kTapsPerBlock;
            const Ix q16 = e / kTapsPerBlock;
            const Ix row = q16 % ntot;
            const Ix cq = q16 / ntot;  // kg * in_ch + c
            const Ix c = cq % in_ch;
            const Ix blk = row / kp, o = (cq / in_ch) * kp + row % kp, s = (g - 1 - blk) * kTapsPerBlock + r;
            float v = 0.0f;
            if (o < out_ch && s < taps) v = wval(w, bwd_raw, out_ch, in_ch, taps, o, c, s);
            const Ix off = (row / 8) * 128 + (r / 8) * 64 + (row % 8) * 8 + (r % 8);
            img[static_cast<int64_t>(cq) * per_chan + off] = fp32_to_bf16_bits(v);
        } else {
            const Ix f = e - main_total;
            const Ix k = f % kTapsPerBlock;
            const Ix row = (f / kTapsPerBlock) % kp;
            const Ix h = (f / per_tail) % chunks;
            const Ix kg = f / (per_tail * chunks);
            const Ix rr = k / cc, c = h * cc + k % cc, o = kg * kp + row;
            const Ix s = static_cast<Ix>(g - 1) * kTapsPerBlock + rr;
            float v = 0.0f;
            if (rr < tail && c < in_ch && o < out_ch && s < taps) v = wval(w, bwd_raw, out_ch, in_ch, taps, o, c, s);
            const Ix off = (row / 8) * 128 + (k / 8) * 64 + (row % 8) * 8 + (k % 8);
            timg[static_cast<int64_t>(kg * chunks + h) * per_tail + off] = fp32_to_bf16_bits(v);
        }
    }
}

// Several layers' main images in one launch (c1d_pack_weights): job j covers elements [begin_j,
// begin_{j+1}) of the concatenated images; element layout as pack_images_kernel's main image.
struct PackJob {
    const float* w;
    uint16_t* img;
    int32_t bwd_raw, out_ch, in_ch, taps, kp, g, kgroups, pad_;
    int64_t begin;
};
constexpr int kMaxPackJobs = 32;
struct PackJobs {
    PackJob j[kMaxPackJobs];
    int32_t count, pad_;
    int64_t total;
};
__global__ void pack_images_multi_kernel(const PackJobs jobs) {
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < jobs.total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        int ji = 0;
        while (ji + 1 < jobs.count && e >= jobs.j[ji + 1].begin) ++ji;
        const PackJob& jb = jobs.j[ji];
        const int32_t el = static_cast<int32_t>(e - jb.begin);  // < 2^31 (checked on the host)
        const int32_t ntot = jb.g * jb.kp, per_chan = ntot * kTapsPerBlock;
        const int32_t r = el % kTapsPerBlock, q16 = el / kTapsPerBlock;
        const int32_t row = q16 % ntot, cq = q16 / ntot, c = cq % jb.in_ch;
        const int32_t blk = row / jb.kp, o = (cq / jb.in_ch) * jb.kp + row % jb.kp;
        const int32_t s = (jb.g - 1 - blk) * kTapsPerBlock + r;
        float v = 0.0f;
        if (o < jb.out_ch && s < jb.taps) v = wval<int32_t>(jb.w, jb.bwd_raw, jb.out_ch, jb.in_ch, jb.taps, o, c, s);
        const int32_t off = (row / 8) * 128 + (r / 8) * 64 + (row % 8) * 8 + (r % 8);
        jb.img[static_cast<int64_t>(cq) * per_chan + off] = fp32_to_bf16_bits(v);
    }
}

// ---------------------------------------------------------------------------- schedule
// Each CTA owns output tiles [b, e) of the flattened (item, tile) list. For each item segment
// (n, j0..j1) it walks input tiles j0 .. j1+G-1 in super-tiles of up to T tiles. Input tile
// i0+t of a super-tile writes output tiles i0+t-G+1 .. i0+t, which live at TMEM slots t..t+G-1
// (slot j <-> output i0-(G-1)+j, KP columns per slot): every MMA is one contiguous N = G*KP run.
constexpr int kProfSlots = 16;  // C1D_PROFILE counters per CTA

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
    // 32-bit divisions when the tile indices fit (always, in practice): a 64-bit division is a
    // ~70-instruction software routine on every warp role's path to its first tile
    if (c.end < (int64_t{1} << 31) && J < (int64_t{1} << 31)) {
        const uint32_t cur = static_cast<uint32_t>(c.cur), j = static_cast<uint32_t>(J);
        c.n = cur / j;
        c.j0 = cur - static_cast<uint32_t>(c.n) * j;
    } else {
        c.n = c.cur / J;
        c.j0 = c.cur % J;
    }
    const int64_t last = imin64(c.end, (c.n + 1) * J) - 1;
    c.j1 = last - c.n * J;
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

// This CTA's output tiles [b, e). Every item segment a CTA walks costs G-1 warm-up input tiles
// before its first output, so the split is even over "virtual" tiles: each item is G-1 warm-up
// tiles followed by its J output tiles, and a CTA whose range holds an item start gets G-1 fewer
// outputs (an even split of the outputs alone left those CTAs ~6% behind at config 2).
__device__ __forceinline__ void cta_tile_range(const KParams& p, int G, int64_t* b, int64_t* e) {
    if (p.total_tiles < 2 * static_cast<int64_t>(gridDim.x)) {  // about one tile per CTA: plain split
        *b = static_cast<int64_t>(static_cast<uint32_t>(p.total_tiles) * blockIdx.x / gridDim.x);
        *e = static_cast<int64_t>(static_cast<uint32_t>(p.total_tiles) * (blockIdx.x + 1) / gridDim.x);
        return;
    }
    const int64_t J = p.tiles_per_item, W = J + (G - 1);
    const int64_t V = p.n_items * W;
    if (V * static_cast<int64_t>(gridDim.x) < (int64_t{1} << 31)) {  // 32-bit divisions
        const uint32_t w = static_cast<uint32_t>(W), g1 = static_cast<uint32_t>(G - 1), j = static_cast<uint32_t>(J);
        auto real32 = [&](uint32_t v) -> int64_t {
            const uint32_t n = v / w, r = v - n * w;
            return static_cast<int64_t>(n) * j + (r > g1 ? r - g1 : 0u);
        };
        const uint32_t v32 = static_cast<uint32_t>(V);
        *b = real32(v32 * blockIdx.x / gridDim.x);
        *e = real32(v32 * (blockIdx.x + 1) / gridDim.x);
        return;
    }
    auto real = [&](int64_t v) -> int64_t {
        const int64_t n = v / W, r = v - n * W;
        return n * J + (r > G - 1 ? r - (G - 1) : 0);
    };
    *b = real(V * blockIdx.x / gridDim.x);
    *e = real(V * (blockIdx.x + 1) / gridDim.x);
}

__device__ __forceinline__ Cursor make_cursor(const KParams& p) {
    Cursor c{};
    int64_t b, e;
    cta_tile_range(p, p.pl.xr ? 1 : p.pl.g, &b, &e);
    c.cur = b;
    c.end = e;
    c.valid = next_segment(c, p.tiles_per_item);
    return c;
}

// ---------------------------------------------------------------------------- layer glue
// The glue runs on the four epilogue warps, one output column per lane and 16 channel rows per
// TMEM load. It is written for instruction count (the plain store loop is ~50 instructions per 16
// rows; a straightforward glue with per-element optional outputs was ~800 and ran 6x slower):
// every optional output is one guarded loop with a running pointer, the bias comes from shared
// memory, mask words move one per lane (a ballot per row, one store / load per warp), and all
// loads of a block are issued before its stores.

// 16 values -> 8 words of bf16 pairs (rows 2i | 2i+1 << 16), hardware round-to-nearest-even:
// identical to the reference's fp32_to_bf16 (bf16.hpp:29-40) for every non-NaN value, denormals and
// overflow included; NaN becomes the canonical bf16 NaN instead of keeping its payload (a NaN
// activation or gradient stays NaN, and the tensor core canonicalises NaN operands anyway).
__device__ __forceinline__ void pack_bf16_rows(const float (&v)[16], uint32_t (&pk)[8]) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(pk[i]) : "f"(v[2 * i + 1]), "f"(v[2 * i]));
}

// Stage 16 rows x 32 columns of up to three outputs in this warp's shared-memory buffer and write
// them with one TMA store each (rows past the channel count and columns past the width fall
// outside the tensor maps and are dropped, so no per-element predicates). Two buffers per warp:
// lane 0 waits until the older store has read its buffer before the warp refills it.
__device__ __forceinline__ void st_shared_f32(uint32_t a, float v) {
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
// rows 2i and 2i+1 of a bf16 staging tile (64-B rows)
__device__ __forceinline__ void st_shared_bf16_pair(uint32_t a, uint32_t pk) {
    asm volatile("{.reg .b16 l, h; mov.b32 {l, h}, %1; st.shared.b16 [%0], l; st.shared.b16 [%0+64], h;}" ::"r"(a),
                 "r"(pk)
                 : "memory");
}
__device__ __forceinline__ void glue_tma_store(const KParams& p, const uint32_t slots, uint32_t& sbuf, uint32_t wbase,
                                               int lane, const float (&va)[16], const float (&vb)[16],
                                               const uint32_t (&pc)[8], const CUtensorMap* m0,
                                               const CUtensorMap* m1, const CUtensorMap* m2, int32_t col,
                                               int32_t col_c, int32_t row, int32_t item) {
    const uint32_t b = wbase + sbuf * p.stg_bytes;
    if (lane == 0) bulk_wait_read<1>();
    __syncwarp();
    if (slots & 1u) {
        const uint32_t a = b + p.stg_a + static_cast<uint32_t>(lane) * 4u;
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) st_shared_f32(a + jj * 128, va[jj]);
    }
    if (slots & 2u) {
        const uint32_t a = b + p.stg_b + static_cast<uint32_t>(lane) * 4u;
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) st_shared_f32(a + jj * 128, vb[jj]);
    }
    if (slots & 4u) {
        const uint32_t a = b + p.stg_c + static_cast<uint32_t>(lane) * 2u;
#pragma unroll
        for (int i = 0; i < 8; ++i) st_shared_bf16_pair(a + i * 128, pc[i]);
    }
    fence_async_smem();
    __syncwarp();
    if (lane == 0) {
        if (slots & 1u) tma_store_3d(m0, b + p.stg_a, col, row, item);
        if (slots & 2u) tma_store_3d(m1, b + p.stg_b, col, row, item);
        if (slots & 4u) tma_store_3d(m2, b + p.stg_c, col_c, row, item);
        bulk_commit();
    }
    sbuf ^= 1u;
}

// Prefetch the glue inputs of one (tile, 16-row block) into a ring slot: each lane copies its own
// column of the 16 rows (zero-filled outside the tensor) and, for the backward, one mask word
// (lanes 0-15: word w0 of rows 0-15, lanes 16-31: w0 + 1; see glue_backward16).
__device__ __forceinline__ void glue_prefetch(const KParams& p, int64_t n, int64_t o, int kbi, uint32_t slot,
                                              int quarter, int lane) {
    const LayerGlue& gl = p.glue;
    const int64_t x = o * kTileQ + quarter * 32 + lane;
    const int64_t k0 = p.k_begin + kbi * 16;
    const int kvalid = static_cast<int>(imin64(16, p.out_ch - k0));
    const int64_t row0 = n * p.out_ch + k0;
    if (p.pf_rows && p.pf_vec) {
        // 16-B pieces: lane copies columns 4*(lane%8) .. +3 of rows lane/8 + 4i (i < 4). The width
        // and the block's first column are multiples of 4, so a piece is wholly inside or outside.
        const float* base = gl.mode == 1 ? gl.skip : gl.gadd;
        const int64_t w = gl.mode == 1 ? p.out_w : gl.g_q;
        const int64_t c = (gl.mode == 1 ? x : x - gl.g_off) - lane + 4 * (lane & 7);
        const bool cv = c >= 0 && c < w;
        const int r0 = lane >> 3;
        const float* src = base + (row0 + r0) * w + c;
        const uint32_t dst = slot + static_cast<uint32_t>(r0 * 128 + (lane & 7) * 16);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const bool v = cv && r0 + 4 * i < kvalid;
            cp_async16_zfill(dst + i * 512, v ? src : base, v);
            src += 4 * w;
        }
    } else if (p.pf_rows) {
        const float* base = gl.mode == 1 ? gl.skip : gl.gadd;
        const int64_t w = gl.mode == 1 ? p.out_w : gl.g_q;
        const int64_t c = gl.mode == 1 ? x : x - gl.g_off;
        const bool cv = c >= 0 && c < w;
        const float* src = base + row0 * w + c;
        const uint32_t dst = slot + static_cast<uint32_t>(lane) * 4u;
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
            const bool v = cv && jj < kvalid;
            cp_async4_zfill(dst + jj * 128, v ? src : base, v);
            src += w;
        }
    }
    if (p.pf_mask) {
        const int64_t gq = gl.g_q;
        const int64_t xi = x - gl.g_off;
        const bool v = xi >= 0 && xi < gq && kvalid > 0;
        const int64_t kblocks = (p.out_ch + 15) >> 4;
        cp_async4_zfill(slot + (p.pf_rows ? 2048u : 0u) + static_cast<uint32_t>(lane) * 4u,
                        v ? gl.mask_in + (n * kblocks + (k0 >> 4)) * gq + xi : gl.mask_in, v);
    }
}

__device__ __forceinline__ float ld_shared_f32(uint32_t a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t ld_shared_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}

// forward glue for rows k0 .. k0+15 of column q; bias16 = those rows' bias (0 past the channel count)
// kFx: 0 = the glue's outputs from its runtime flags; 1-3 = the config-5 network's layer shapes with
// the flags fixed at compile time (no per-block flag loads / branches in the issue-bound glue):
//   1: bias, ReLU, mask, BF16 activation (TMA slot 4)       -- body layers
//   2: + skip add and FP32 activation (slots 2 | 4)          -- block-output layers
//   3: bias, ReLU, mask, FP32 + BF16 activation, no skip    -- the input layer
//   4: bias, ReLU, mask, skip, FP32 activation only         -- the last block's output (heads input)
template <int kFx>
struct FwdFx {
    static constexpr bool kRelu = true, kMask = true, kBf16 = kFx != 4;
    static constexpr bool kSkip = kFx == 2 || kFx == 4;
    static constexpr uint32_t kSlots = kFx == 1 ? 4u : (kFx == 4 ? 2u : 6u);  // slot 2: the FP32 activation
};
template <int kFx>
__device__ __forceinline__ void glue_forward16(const KParams& p, const uint32_t (&v)[16], int64_t n, int64_t q,
                                               int64_t k0, int lane, const float (&bias16)[16], uint32_t& sbuf,
                                               uint32_t wbase, const CUtensorMap* m0, const CUtensorMap* m1,
                                               const CUtensorMap* m2, uint32_t pf_slot) {
    const LayerGlue& gl = p.glue;
    using F = FwdFx<kFx>;
    const int64_t out_w = p.out_w;
    const bool qv = q < out_w;
    const int kvalid = static_cast<int>(imin64(16, p.out_ch - k0));
    const int64_t row0 = n * p.out_ch + k0;
    float x[16], a[16];
    const bool relu = kFx ? F::kRelu : gl.relu != 0;
    const bool has_mask = kFx ? F::kMask : gl.mask_out != nullptr;
    const bool has_skip = kFx ? F::kSkip : gl.skip != nullptr;
    const bool has_bf16 = kFx ? F::kBf16 : gl.act_bf16 != nullptr;
    const uint32_t slots = kFx ? F::kSlots : p.tma_slots;
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) {
        x[jj] = __uint_as_float(v[jj]) + bias16[jj];
        a[jj] = (relu && !(x[jj] > 0.0f)) ? 0.0f : x[jj];
    }
    // mask word (bit jj = x[jj] > 0) from integer ops: with ReLU, a[jj] is +0 or x[jj] > 0 (NaN -> 0),
    // so bit = (bits(a) != 0) = (bits(a) + 0x7fffffff) >> 31, accumulated MSB-first; the float
    // compare form compiled to ~100 predicate-juggling instructions per block
    uint32_t mword = 0;
    if (has_mask) {
        if (relu) {
#pragma unroll
            for (int jj = 15; jj >= 0; --jj) mword = (mword << 1) | ((__float_as_uint(a[jj]) + 0x7fffffffu) >> 31);
        } else {
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) mword |= (x[jj] > 0.0f ? 1u : 0u) << jj;
        }
    }
    if (has_skip) {  // prefetched rows (zero outside the tensor)
        const uint32_t src = pf_slot + static_cast<uint32_t>(lane) * 4u;
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) a[jj] += ld_shared_f32(src + jj * 128);
    }
    if (has_mask) {  // one word per column and 16-channel block: bit jj = row k0 + jj
        const int64_t kblocks = (p.out_ch + 15) >> 4;
        if (qv && kvalid > 0) gl.mask_out[(n * kblocks + (k0 >> 4)) * out_w + q] = mword;
    }
    uint32_t pc[8];
    if (has_bf16) pack_bf16_rows(a, pc);
    if (slots) {
        glue_tma_store(p, slots, sbuf, wbase, lane, x, a, pc, m0, m1, m2, static_cast<int32_t>(q - lane),
                       static_cast<int32_t>(gl.act_off + q - lane), static_cast<int32_t>(k0), static_cast<int32_t>(n));
        return;
    }
    if (!qv) return;
    if (gl.pre) {
        float* d = gl.pre + row0 * out_w + q;
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
            if (jj < kvalid) *d = x[jj];
            d += out_w;
        }
    }
    if (gl.act) {
        float* d = gl.act + row0 * out_w + q;
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
            if (jj < kvalid) *d = a[jj];
            d += out_w;
        }
    }
    if (gl.act_bf16) {
        const int64_t pitch = gl.act_pitch;
        uint16_t* d = gl.act_bf16 + row0 * pitch + gl.act_off + q;
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
            if (jj < kvalid) *d = static_cast<uint16_t>(pc[jj / 2] >> (16 * (jj & 1)));
            d += pitch;
        }
    }
}

// backward glue for rows k0 .. k0+15 of padded column x (the glued layer's column xi = x - g_off)
// kFx: 0 = runtime flags; 1 = ReLU mask + BF16 gradient + bias gradient, per-lane stores (body
// layers); 2 = 1 + skip gradient added (gadd) and the sum stored (gsum) (block-input layers);
// 3 = 1 + gadd without gsum (the first block's input layer)
template <int kFx>
__device__ __forceinline__ void glue_backward16(const KParams& p, const uint32_t (&v)[16], int64_t n, int64_t x,
                                                int64_t k0, int lane, float (&bs)[16], uint32_t& sbuf,
                                                uint32_t wbase, const CUtensorMap* m0, const CUtensorMap* m1,
                                                const CUtensorMap* m2, uint32_t pf_slot) {
    const LayerGlue& gl = p.glue;
    const bool has_mask = kFx ? true : gl.mask_in != nullptr;
    const bool has_gadd = kFx ? kFx >= 2 : gl.gadd != nullptr;
    const bool has_gsum = kFx ? kFx == 2 : gl.gsum != nullptr;
    const bool has_gp = kFx ? false : gl.gp != nullptr;
    const bool has_gpb = kFx ? true : gl.gp_bf16 != nullptr;
    const uint32_t slots = kFx ? 0u : p.tma_slots;
    const int64_t gq = gl.g_q;
    const int64_t xi = x - gl.g_off;
    const bool xv = xi >= 0 && xi < gq;
    const int kvalid = static_cast<int>(imin64(16, p.out_ch - k0));
    const int64_t row0 = n * p.out_ch + k0;
    // ReLU mask: this column's word for the 16-row block (prefetched; bit jj = row k0 + jj)
    const uint32_t mword = has_mask ? ld_shared_u32(pf_slot + (has_gadd ? 2048u : 0u) + static_cast<uint32_t>(lane) * 4u)
                                    : 0xffffu;
    float g[16];
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) g[jj] = __uint_as_float(v[jj]);
    if (has_gadd) {  // prefetched rows (zero outside the window)
        const uint32_t src = pf_slot + static_cast<uint32_t>(lane) * 4u;
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) g[jj] += ld_shared_f32(src + jj * 128);
    }
    float gp[16];
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) gp[jj] = (mword & (1u << jj)) ? g[jj] : 0.0f;
    if (xv) {
#pragma unroll
        for (int jj = 0; jj < 16; ++jj)
            if (jj < kvalid) bs[jj] += gp[jj];
    }
    uint32_t pc[8];
    if (has_gpb) pack_bf16_rows(gp, pc);
    // TMA stores need a non-negative start column: the warp straddling the glued window's left
    // edge (once per item) takes the per-lane path
    const int64_t col = xi - lane;
    if (slots && col >= 0) {
        glue_tma_store(p, slots, sbuf, wbase, lane, g, gp, pc, m0, m1, m2, static_cast<int32_t>(col),
                       static_cast<int32_t>(col), static_cast<int32_t>(k0), static_cast<int32_t>(n));
        return;
    }
    if (!xv) return;
    const int64_t e = row0 * gq + xi;
    if (has_gsum) {
        float* d = gl.gsum + e;
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
            if (jj < kvalid) *d = g[jj];
            d += gq;
        }
    }
    if (has_gp) {
        float* d = gl.gp + e;
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
            if (jj < kvalid) *d = gp[jj];
            d += gq;
        }
    }
    if (has_gpb) {
        uint16_t* d = gl.gp_bf16 + e;
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
            if (jj < kvalid) *d = static_cast<uint16_t>(pc[jj / 2] >> (16 * (jj & 1)));
            d += gq;
        }
    }
}

// Inline E rows: rows r0 .. r0+RG-1 of one channel from its natural window (element e of row r =
// window[K0 + D*r + e], K0 = the window's alignment offset, uniform per super-tile). A group's
// window words are loaded once; every index is compile-time (one instantiation per D, K0).
template <int D, int K0>
__device__ __forceinline__ void expand_group_rows(uint32_t rc, uint32_t xc, int rows, int et) {
    constexpr int RG = D == 4 ? 4 : 8;                 // rows per group
    constexpr int NW = ((K0 + D * (RG - 1) + 8 + 7) / 8) * 4;  // 32-bit words loaded
    for (int r0 = et * RG; r0 < rows; r0 += 64 * RG) {
        const uint32_t src = rc + static_cast<uint32_t>(D * r0 * 2);  // 16-B aligned (D*r0 % 8 == 0)
        uint32_t w[NW];
#pragma unroll
        for (int i = 0; i < NW; i += 4)
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(w[i]), "=r"(w[i + 1]), "=r"(w[i + 2]), "=r"(w[i + 3])
                         : "r"(src + static_cast<uint32_t>(i * 4)));
#pragma unroll
        for (int j = 0; j < RG; ++j) {
            const int o = K0 + D * j;  // element offset of the row in the loaded words
            uint32_t v[4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
                v[i] = (o & 1) ? __funnelshift_r(w[(o >> 1) + i], w[(o >> 1) + i + 1], 16) : w[(o >> 1) + i];
            asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(xc + static_cast<uint32_t>((r0 + j) * 16)),
                         "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3])
                         : "memory");
        }
    }
}

template <int D>
__device__ __forceinline__ void expand_rows_d(uint32_t rc, uint32_t xc, int rows, int et, int off) {
    switch (off) {
        case 0: expand_group_rows<D, 0>(rc, xc, rows, et); break;
        case 1: expand_group_rows<D, 1>(rc, xc, rows, et); break;
        case 2: expand_group_rows<D, 2>(rc, xc, rows, et); break;
        case 3: expand_group_rows<D, 3>(rc, xc, rows, et); break;
        case 4: expand_group_rows<D, 4>(rc, xc, rows, et); break;
        case 5: expand_group_rows<D, 5>(rc, xc, rows, et); break;
        case 6: expand_group_rows<D, 6>(rc, xc, rows, et); break;
        default: expand_group_rows<D, 7>(rc, xc, rows, et); break;
    }
}

// The main MMAs of a stage: for each channel, its NT consecutive input tiles as one straight-line
// run. Tile t reads A at +256 B per tile and accumulates at column dcol + t*KP; every descriptor and
// column is an independent add from the channel base (a dependent uniform-register chain between
// MMAs throttled the issuing thread to ~70 cycles per MMA). With ws, the channel's B block is
// latched in the collector by its first MMA and re-used by the others (tcgen05.mma.ws).
struct IssueArgs {
    uint32_t dcol, kp, acc2;
    uint64_t adesc, bdesc;
    uint32_t idesc, a_chan_bytes, b_chan_bytes;
    int ccn, c_split;  // channels of the stage; channels >= c_split accumulate at +acc2
    int ws;
};
template <int NT>
__device__ __forceinline__ void issue_channels(const IssueArgs& ia) {
    uint64_t adesc = ia.adesc, bdesc = ia.bdesc;
    for (int c = 0; c < ia.ccn; ++c) {
        const uint32_t dcol = ia.dcol + (c >= ia.c_split ? ia.acc2 : 0u);
        if (ia.ws && NT >= 2) {
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const uint64_t a = adesc + static_cast<uint64_t>(t * (kTileQ * 2 / 16));
                const uint32_t d = dcol + static_cast<uint32_t>(t) * ia.kp;
                if (t == 0) mma_ws_fill(d, a, bdesc, ia.idesc, 1);
                else if (t == NT - 1) mma_ws_lastuse(d, a, bdesc, ia.idesc, 1);
                else mma_ws_use(d, a, bdesc, ia.idesc, 1);
            }
        } else {
#pragma unroll
            for (int t = 0; t < NT; ++t)
                mma_bf16_ss(dcol + static_cast<uint32_t>(t) * ia.kp, adesc + static_cast<uint64_t>(t * (kTileQ * 2 / 16)),
                            bdesc, ia.idesc, 1);
        }
        adesc = desc_advance(adesc, ia.a_chan_bytes);
        bdesc = desc_advance(bdesc, ia.b_chan_bytes);
    }
}

// kMode: 0 plain FP32 store, 1 forward glue, 2 backward glue (p.glue.mode); kKPB (modes 1-2): 16-channel
// blocks per filter group (KP/16), so the per-lane bias values / bias-gradient sums live in registers. One instantiation per
// mode keeps each kernel's code small: the epilogue warps share the instruction cache with the MMA
// and TMA warps, and an all-modes kernel (~30k instructions) ran the epilogue 6x slower.
// kLean 1: the plan is a natural-row, single-buffered carry plan with streamed weights and one
// accumulator region (config 3); kLean 2 and the fixed-flag glue kernels (kFx): a natural-row,
// double-buffered, one-region plan with weight-stationary N = 64 MMAs (config 2, the network's
// layers). Those plan fields are
// compile-time constants there, which drops the other paths' code from the three roles' hot loops
// (they share the instruction cache).
template <int kMode, int kKPB, int kEG = 1, int kFx = 0, int kLean = 0>
__global__ void __launch_bounds__(128 + 128 * kEG, 1)
    tc_conv_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap tmap_tail,
                   const __grid_constant__ CUtensorMap om0, const __grid_constant__ CUtensorMap om1,
                   const __grid_constant__ CUtensorMap om2, const KParams p) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint64_t stage_full[kMaxStages], stage_empty[kMaxStages];
    __shared__ uint64_t raw_full[kMaxStages];  // inline expansion: natural windows landed
    // double-buffered TMEM: tmem_empty / tmem_empty2 release region 0 / 1 (stores done, non-carry
    // slots zeroed); carry_full publishes the G-1 carried slots of the next super-tile
    __shared__ uint64_t tmem_full, tmem_empty, tmem_empty2, carry_full, wres_full;
    __shared__ uint64_t tile_full[8];  // staggered finish: output slot t of the super-tile is complete
    __shared__ uint32_t tmem_base_s;
    __shared__ float bias_red[8 * 64];  // layer glue: per-epilogue-warp bias-gradient sums

    Plan plv = p.pl;
    if constexpr (kLean == 1) {
        plv.xr = plv.xin = plv.dbuf = plv.ws = 0;
        plv.wres_bytes = 0;
        plv.acc2 = 0;
        plv.raw_segs = plv.rows_alloc = plv.n_box = plv.box_rows = 0;
        plv.raw_stage_bytes = 0;
    }
    if constexpr (kFx != 0 || kLean == 2) {
        // the fixed-flag glue kernels (the network's narrow layers) only take natural-row,
        // double-buffered, one-region plans (launch_tc_conv checks)
        plv.xr = plv.xin = plv.tail = plv.stagger = 0;
        plv.dbuf = plv.ws = 1;
        plv.acc2 = 0;
        plv.raw_segs = plv.rows_alloc = plv.n_box = plv.box_rows = 0;
        plv.raw_stage_bytes = plv.tx_stage_bytes = plv.tw_stage_bytes = 0;
    }
    const Plan& pl = plv;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    const uint32_t wres_s = smem_u32(smem);  // resident weights (pl.wres_bytes), then the stages
    uint8_t* xs_base = smem + pl.wres_bytes;
    uint8_t* ws_base = xs_base + static_cast<size_t>(pl.stages) * pl.x_stage_bytes;
    uint8_t* tx_base = ws_base + static_cast<size_t>(pl.stages) * pl.w_stage_bytes;
    uint8_t* tw_base = tx_base + static_cast<size_t>(pl.stages) * pl.tx_stage_bytes;
    uint8_t* raw_base = tw_base + static_cast<size_t>(pl.stages) * pl.tw_stage_bytes;
    // G: tap blocks the schedule carries between tiles (1 in expanded-row mode: no carry)
    const int G = pl.xr ? 1 : pl.g, T = pl.t, KP = pl.kp;
    const int64_t J = p.tiles_per_item;
    const int n_chunks = static_cast<int>(ceil_div(p.in_ch, pl.cc));

    if (threadIdx.x == 0) {
        for (int s = 0; s < pl.stages; ++s) {
            mbar_init(&stage_full[s], pl.xin && pl.xr != 8 ? 2 : 1);  // + the expanders' arrival
            mbar_init(&raw_full[s], 1);
            mbar_init(&stage_empty[s], 1);
        }
        mbar_init(&tmem_full, 1);
        mbar_init(&tmem_empty, 4);  // one arrival per epilogue warp
        mbar_init(&tmem_empty2, 4);
        mbar_init(&carry_full, 4);
        mbar_init(&wres_full, 1);
        for (int t = 0; t < 8; ++t) mbar_init(&tile_full[t], 1);
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc<kTmemCols>(&tmem_base_s);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_s;
    if (p.early_w && threadIdx.x == 0) {
        const uint32_t wbytes = static_cast<uint32_t>(p.in_ch) * pl.b_chan_bytes;
        mbar_arrive_expect_tx(smem_u32(&wres_full), wbytes);
        for (uint32_t o = 0; o < wbytes; o += 32768u)
            bulk_g2s(wres_s + o, p.bimg + o / 2, wbytes - o < 32768u ? wbytes - o : 32768u, smem_u32(&wres_full));
    }
    // PDL: everything above overlapped the previous kernel; global memory only from here on (the
    // prepacked weight image excepted: it was complete before the previous kernel was launched)
    pdl_trigger();
    pdl_wait();
    if (p.prof && threadIdx.x == 0) {
        p.prof[blockIdx.x * kProfSlots + 8] = globaltimer_ns();
        p.prof[blockIdx.x * kProfSlots + 10] = clock64();
    }

    if (warp == 0) {
        // ------------------------------------------------------------------ TMA producer
        if (lane == 0) {
            prefetch_tmap(&tmap);
            if (pl.tail || pl.xbox3) prefetch_tmap(&tmap_tail);
            long long t_wait = 0;
            const long long t_begin = clock64();
            Cursor cur = make_cursor(p);
            int stage = 0;
            uint32_t phase = 0;
            Super su;
            const uint32_t wchan = pl.wres_bytes ? 0u : pl.b_chan_bytes;  // weight bytes per channel and stage
            if (pl.wres_bytes && !p.early_w) {
                const uint32_t wbytes = static_cast<uint32_t>(p.in_ch) * pl.b_chan_bytes;
                mbar_arrive_expect_tx(smem_u32(&wres_full), wbytes);
                for (uint32_t o = 0; o < wbytes; o += 32768u)
                    bulk_g2s(wres_s + o, p.bimg + o / 2, wbytes - o < 32768u ? wbytes - o : 32768u, smem_u32(&wres_full));
            }
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
                    if (pl.xin) {
                        // natural windows from a 16-B aligned start into the raw area (the expanders
                        // build the E rows), the weights straight into the stage
                        // (d = 8: the window is the A operand itself, so it completes the stage barrier)
                        const uint32_t rf = pl.xr == 8 ? full : smem_u32(&raw_full[stage]);
                        mbar_arrive_expect_tx(rf, static_cast<uint32_t>(ccn * pl.raw_segs * kSegQ * 2) +
                                                      (pl.xr == 8 ? static_cast<uint32_t>(ccn) * wchan : 0u));
                        const int32_t x_al = x_start - (((x_start % 8) + 8) % 8);
                        const uint32_t raw = smem_u32(raw_base + static_cast<size_t>(stage) * pl.raw_stage_bytes);
                        for (int c = 0; c < ccn; ++c) {
                            const int32_t row = static_cast<int32_t>(su.n * p.in_ch + c0 + c);
                            for (int sg = 0; sg < pl.raw_segs; ++sg)
                                tma_load_2d(raw + static_cast<uint32_t>((c * pl.raw_segs + sg) * kSegQ * 2), &tmap,
                                            x_al + sg * kSegQ, row, rf);
                        }
                        if (pl.xr != 8) mbar_arrive_expect_tx(full, static_cast<uint32_t>(ccn) * wchan);
                        if (wchan) {
                            const uint32_t wsm = smem_u32(ws_base + static_cast<size_t>(stage) * pl.w_stage_bytes);
                            bulk_g2s(wsm, p.bimg + static_cast<size_t>(c0) * (pl.b_chan_bytes / 2),
                                     static_cast<uint32_t>(ccn) * pl.b_chan_bytes, full);
                        }
                        if (++stage == pl.stages) {
                            stage = 0;
                            phase ^= 1;
                        }
                        continue;
                    }
                    const bool box3 = pl.xbox3 && x_start >= 0 && x_start + pl.xw <= p.in_w;
                    const uint32_t xbytes = pl.xr ? static_cast<uint32_t>(pl.rows_alloc * 16) : static_cast<uint32_t>(nseg * kSegQ * 2);
                    const uint32_t bytes = (box3 ? static_cast<uint32_t>(pl.cc * pl.xw * 2) + static_cast<uint32_t>(ccn) * wchan
                                                 : static_cast<uint32_t>(ccn) * (xbytes + wchan)) +
                                           (pl.tail ? pl.tail_chunks * pl.cc * 16u + pl.tw_stage_bytes : 0u);
                    mbar_arrive_expect_tx(full, bytes);
                    const uint32_t xs = smem_u32(xs_base + static_cast<size_t>(stage) * pl.x_stage_bytes);
                    if (pl.xr) {  // E rows [128 i0 / d, ...) of each channel, n_box boxes
                        const int32_t r0 = static_cast<int32_t>(su.i0 * (kTileQ / pl.xr));
                        for (int c = 0; c < ccn; ++c) {
                            const int32_t row = static_cast<int32_t>(su.n * p.in_ch + c0 + c);
                            for (int b = 0; b < pl.n_box; ++b)
                                tma_load_3d(xs + static_cast<uint32_t>((c * pl.rows_alloc + b * pl.box_rows) * 16), &tmap,
                                            0, (r0 + b * pl.box_rows) / 8, row, full);
                        }
                    } else if (box3) {
                        tma_load_3d(xs, &tmap_tail, x_start, 0, static_cast<int32_t>(su.n * p.in_ch + c0), full);
                    } else {
                        for (int c = 0; c < ccn; ++c) {
                            const int32_t row = static_cast<int32_t>(su.n * p.in_ch + c0 + c);
                            for (int sg = 0; sg < nseg; ++sg)
                                tma_load_2d(xs + static_cast<uint32_t>((c * pl.xw + sg * kSegQ) * 2), &tmap,
                                            x_start + sg * kSegQ, row, full);
                        }
                    }
                    if (wchan) {
                        const uint32_t wsm = smem_u32(ws_base + static_cast<size_t>(stage) * pl.w_stage_bytes);
                        bulk_g2s(wsm, p.bimg + static_cast<size_t>(c0) * (pl.b_chan_bytes / 2),
                                 static_cast<uint32_t>(ccn) * pl.b_chan_bytes, full);
                    }
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
                p.prof[blockIdx.x * kProfSlots + 0] = t_wait;
                p.prof[blockIdx.x * kProfSlots + 1] = clock64() - t_begin;
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------------ MMA issuer
        // The whole warp walks the schedule (warp-uniform control flow keeps descriptors in
        // uniform registers); one elected lane issues each tcgen05 instruction.
        long long t_full = 0, t_tmem = 0, t_full_first = -1, n_super = 0, t_issue = 0;
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
        uint32_t rphase[2] = {0u, 0u}, cphase = 0;
        if (pl.wres_bytes) {
            mbar_wait(smem_u32(&wres_full), 0);
            tc_fence_after();
        }
        bool first_super = true;
        Super su;
        while (next_super(cur, J, G, T, &su)) {
            const long long ts0 = clock64();
            if (pl.dbuf) {
                const int ri = region ? 1 : 0;
                mbar_wait(smem_u32(ri ? &tmem_empty2 : &tmem_empty), rphase[ri]);
                rphase[ri] ^= 1u;
            } else {
                mbar_wait(smem_u32(&tmem_empty), tphase);
                tphase ^= 1;
            }
            t_tmem += clock64() - ts0;
            tc_fence_after();
            // double buffering: tiles t >= G-1 do not touch the carried slots 0..G-2, so the first
            // stage issues them before waiting for the epilogue's carry (the carry overlaps MMAs)
            bool need_carry = pl.dbuf && G > 1 && !first_super;
            first_super = false;
            const uint32_t rtmem = tmem + region;
            int sg_stage[kMaxStagger] = {0, 0};
            for (int ch = 0; ch < n_chunks; ++ch) {
                const int c0 = ch * pl.cc;
                const int ccn = static_cast<int>(imin64(pl.cc, p.in_ch - c0));
                const long long tf0 = clock64();
                mbar_wait(smem_u32(&stage_full[stage]), phase);
                t_full += clock64() - tf0;
                tc_fence_after();
                if constexpr (kKPB != 1) {
                    if (ch >= n_chunks - pl.stagger) {  // staggered finish: issued tile-major below
                        sg_stage[ch - (n_chunks - pl.stagger)] = stage;
                        if (++stage == pl.stages) {
                            stage = 0;
                            phase ^= 1;
                        }
                        continue;
                    }
                }
                const uint32_t xs = smem_u32(xs_base + static_cast<size_t>(stage) * pl.x_stage_bytes);
                const uint32_t wsm = pl.wres_bytes ? wres_s + static_cast<uint32_t>(c0) * pl.b_chan_bytes
                                                   : smem_u32(ws_base + static_cast<size_t>(stage) * pl.w_stage_bytes);
                const uint64_t a0 = make_smem_desc(xs, 128, 16, kLayoutNone);
                const uint64_t b0 = make_smem_desc(wsm + main_brow, 128, 256, kLayoutNone);
                if (pl.xr) {
                    // expanded rows: A = E rows (16 B, one tap each), M groups 128/d B apart;
                    // tile t, block g at row 128t/d + 16g; B block g = image block G-1-g
                    if (elect_one()) {
                        const uint32_t tile_bytes = static_cast<uint32_t>((kTileQ / pl.xr) * 16);
                        const uint32_t idesc_x = make_idesc(128, static_cast<uint32_t>(KP), kFmtBF16, 1, 0);
                        // d = 8 (inline): A is the raw window (its start is 16-B aligned, so no shift)
                        const uint32_t a_base =
                            pl.xr == 8 ? smem_u32(raw_base + static_cast<size_t>(stage) * pl.raw_stage_bytes) : xs;
                        const uint32_t a_chan = pl.xr == 8 ? static_cast<uint32_t>(pl.raw_segs * kSegQ * 2)
                                                           : static_cast<uint32_t>(pl.rows_alloc * 16);
                        uint64_t achan = make_smem_desc(a_base, 128, static_cast<uint32_t>(128 / pl.xr), kLayoutNone);
                        uint64_t bchan = make_smem_desc(wsm, 128, 256, kLayoutNone);
                        for (int c = 0; c < ccn; ++c) {
                            // image block b (ascending) holds tap block gb = G-1-b (A rows 16 gb)
                            uint64_t ablk = desc_advance(achan, static_cast<uint32_t>((pl.g - 1) * kTapsPerBlock * 16));
                            uint64_t bblk = bchan;
                            const uint32_t dbase = rtmem + ((c0 + c >= p.main_ch) ? pl.acc2 : 0u);
                            for (int b = 0; b < pl.g; ++b) {
                                uint64_t adesc = ablk;
                                uint32_t dcol = dbase;
                                for (int t = 0; t < su.tcur; ++t) {
                                    mma_bf16_ss(dcol, adesc, bblk, idesc_x, 1);
                                    adesc = desc_advance(adesc, tile_bytes);
                                    dcol += static_cast<uint32_t>(KP);
                                }
                                ablk -= static_cast<uint64_t>(kTapsPerBlock);  // 16 rows x 16 B, in 16-B units
                                bblk = desc_advance(bblk, static_cast<uint32_t>(KP * 32));
                            }
                            achan = desc_advance(achan, a_chan);
                            bchan = desc_advance(bchan, pl.b_chan_bytes);
                        }
                    }
                } else {
                    const int tsplit = need_carry ? (su.tcur < G - 1 ? su.tcur : G - 1) : 0;
                    // main MMAs of input tiles [t0, t1) for every channel of the stage
                    auto issue_tiles = [&](int t0, int t1) {
                        if constexpr (kKPB == 1) {
                            // KP = 16 (own instantiation): straight-line runs per channel, B latched in
                            // the collector (ws); the wider plans keep the loop below, which keeps
                            // their kernels' code small (straight-line runs there cost config 3 ~4%)
                            const uint64_t a_t0 = desc_advance(a0, static_cast<uint32_t>(t0 * kTileQ * 2));
                            const uint32_t dchan = rtmem + main_slot + static_cast<uint32_t>(t0 * KP);
                            const int c_split = static_cast<int>(imin64(ccn, imax64(0, p.main_ch - c0)));
                            const IssueArgs ia{dchan, static_cast<uint32_t>(KP), pl.acc2, a_t0, b0, idesc,
                                               static_cast<uint32_t>(pl.xw * 2), pl.b_chan_bytes, ccn, c_split, pl.ws};
                            switch (t1 - t0) {
                                case 1: issue_channels<1>(ia); break;
                                case 2: issue_channels<2>(ia); break;
                                case 3: issue_channels<3>(ia); break;
                                case 4: issue_channels<4>(ia); break;
                                case 5: issue_channels<5>(ia); break;
                                case 6: issue_channels<6>(ia); break;
                                case 7: issue_channels<7>(ia); break;
                                case 8: issue_channels<8>(ia); break;
                                default: break;
                            }
                            return;
                        }
                        uint64_t bdesc = b0;
                        uint64_t achan = desc_advance(a0, static_cast<uint32_t>(t0 * kTileQ * 2));
                        for (int c = 0; c < ccn; ++c) {
                            uint64_t adesc = achan;
                            uint32_t dcol = rtmem + ((c0 + c >= p.main_ch) ? pl.acc2 : 0u) + main_slot +
                                            static_cast<uint32_t>(t0 * KP);
                            for (int t = t0; t < t1; ++t) {
                                mma_bf16_ss(dcol, adesc, bdesc, idesc, 1);
                                adesc = desc_advance(adesc, static_cast<uint32_t>(kTileQ * 2));
                                dcol += static_cast<uint32_t>(KP);
                            }
                            bdesc = desc_advance(bdesc, pl.b_chan_bytes);
                            achan = desc_advance(achan, static_cast<uint32_t>(pl.xw * 2));
                        }
                    };
                    const long long ti0 = clock64();
                    if (elect_one()) issue_tiles(tsplit, su.tcur);
                    __syncwarp();
                    t_issue += clock64() - ti0;
                    if (need_carry) {
                        const long long tc0 = clock64();
                        mbar_wait(smem_u32(&carry_full), cphase);
                        cphase ^= 1u;
                        t_tmem += clock64() - tc0;
                        tc_fence_after();
                        need_carry = false;
                        const long long ti1 = clock64();
                        if (elect_one()) issue_tiles(0, tsplit);
                        __syncwarp();
                        t_issue += clock64() - ti1;
                    }
                    if (pl.tail && elect_one()) {
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
            bool staggered = false;
            if constexpr (kKPB != 1) {
                if (pl.stagger) {
                    // the deferred chunks, tile by tile: slot t is complete after tile t (input tile t
                    // is the last to write it), so each tile commits its own barrier
                    staggered = true;
                    const long long ti0 = clock64();
                    if (elect_one()) {
                        for (int t = 0; t < su.tcur; ++t) {
                            for (int i = 0; i < pl.stagger; ++i) {
                                const int c0 = (n_chunks - pl.stagger + i) * pl.cc;
                                const int ccn = static_cast<int>(imin64(pl.cc, p.in_ch - c0));
                                const size_t st = static_cast<size_t>(sg_stage[i]);
                                const uint32_t wsm = pl.wres_bytes ? wres_s + static_cast<uint32_t>(c0) * pl.b_chan_bytes
                                                                   : smem_u32(ws_base + st * pl.w_stage_bytes);
                                uint64_t adesc = desc_advance(make_smem_desc(smem_u32(xs_base + st * pl.x_stage_bytes), 128, 16, kLayoutNone),
                                                              static_cast<uint32_t>(t * kTileQ * 2));
                                uint64_t bdesc = make_smem_desc(wsm + main_brow, 128, 256, kLayoutNone);
                                for (int c = 0; c < ccn; ++c) {
                                    mma_bf16_ss(rtmem + ((c0 + c >= p.main_ch) ? pl.acc2 : 0u) + main_slot + static_cast<uint32_t>(t * KP),
                                                adesc, bdesc, idesc, 1);
                                    bdesc = desc_advance(bdesc, pl.b_chan_bytes);
                                    adesc = desc_advance(adesc, static_cast<uint32_t>(pl.xw * 2));
                                }
                                if (pl.tail) {
                                    const uint32_t tx = smem_u32(tx_base + st * pl.tx_stage_bytes);
                                    const uint32_t tw = smem_u32(tw_base + st * pl.tw_stage_bytes);
                                    mma_bf16_ss(rtmem + ((c0 >= p.main_ch) ? pl.acc2 : 0u) + static_cast<uint32_t>(t * KP),
                                                desc_advance(make_smem_desc(tx, 128, static_cast<uint32_t>(pl.cc * 16), kLayoutNone),
                                                             static_cast<uint32_t>(t * 16 * pl.cc * 16)),
                                                make_smem_desc(tw, 128, 256, kLayoutNone), idesc_tail, 1);
                                }
                            }
                            mma_commit(smem_u32(&tile_full[t]));
                        }
                        for (int i = 0; i < pl.stagger; ++i) mma_commit(smem_u32(&stage_empty[sg_stage[i]]));
                    }
                    __syncwarp();
                    t_issue += clock64() - ti0;
                }
            }
            if (!staggered && elect_one()) mma_commit(smem_u32(&tmem_full));
            __syncwarp();
            if (pl.dbuf) region ^= 256u;
            if (t_full_first < 0) t_full_first = t_full + t_tmem;
            ++n_super;
        }
        if (p.prof && lane == 0) {
            p.prof[blockIdx.x * kProfSlots + 2] = t_full;
            p.prof[blockIdx.x * kProfSlots + 3] = t_tmem;
            p.prof[blockIdx.x * kProfSlots + 4] = clock64() - t_begin;
            p.prof[blockIdx.x * kProfSlots + 12] = t_full_first;
            p.prof[blockIdx.x * kProfSlots + 13] = n_super;
            p.prof[blockIdx.x * kProfSlots + 14] = t_issue;
        }
    } else if (warp == 2 || warp == 3) {
        // ------------------------------------------------------------------ E-row expanders
        // (inline expanded-row mode) row r of a channel = 8 elements from column x_start + d*r
        // of its natural window: two aligned 16-B reads, a funnel shift, one 16-B write
        if (pl.xin && pl.xr != 8) {
            const int et = threadIdx.x - 64;
            const int d = pl.xr;
            const uint32_t raw_chan = static_cast<uint32_t>(pl.raw_segs * kSegQ * 2);
            Cursor cur = make_cursor(p);
            int stage = 0;
            uint32_t phase = 0;
            Super su;
            while (next_super(cur, J, G, T, &su)) {
                const int64_t x_start = su.i0 * kTileQ + p.in_off;
                const int off = static_cast<int>(((x_start % 8) + 8) % 8);
                for (int ch = 0; ch < n_chunks; ++ch) {
                    const int ccn = static_cast<int>(imin64(pl.cc, p.in_ch - ch * pl.cc));
                    mbar_wait(smem_u32(&raw_full[stage]), phase);
                    const uint32_t raw = smem_u32(raw_base + static_cast<size_t>(stage) * pl.raw_stage_bytes);
                    const uint32_t xs = smem_u32(xs_base + static_cast<size_t>(stage) * pl.x_stage_bytes);
                    for (int c = 0; c < ccn; ++c) {
                        const uint32_t rc = raw + static_cast<uint32_t>(c) * raw_chan;
                        const uint32_t xc = xs + static_cast<uint32_t>(c * pl.rows_alloc * 16);
                        if (d == 1)
                            expand_rows_d<1>(rc, xc, pl.rows_stage, et, off);
                        else if (d == 2)
                            expand_rows_d<2>(rc, xc, pl.rows_stage, et, off);
                        else
                            expand_rows_d<4>(rc, xc, pl.rows_stage, et, off);
                    }
                    fence_async_smem();  // generic-proxy rows -> the tensor core's async proxy
                    asm volatile("bar.sync 2, 64;" ::: "memory");
                    if (et == 0) mbar_arrive(smem_u32(&stage_full[stage]));
                    if (++stage == pl.stages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp >= 4) {
        // ------------------------------------------------------------------ epilogue
        // kEG groups of four warps (the glue variants with narrow filter blocks run two: the glue
        // is issue-bound); group g stores the CTA's output tiles t with (t - first) % kEG == g, and
        // group 0 alone carries / zeroes TMEM and signals the MMA warp
        const int ew = warp - 4;         // epilogue warp 0 .. 4*kEG-1
        const int egrp = ew >> 2;        // epilogue group
        const int quarter = ew & 3;      // TMEM lanes 32*quarter .. +31
        const uint32_t lane_base = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
        uint32_t z[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) z[j] = 0;
        if (egrp == 0) {
            for (uint32_t col = 0; col < kTmemCols; col += 16) tmem_st16(lane_base + col, z);
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(smem_u32(&tmem_empty));
                if (pl.dbuf) mbar_arrive(smem_u32(&tmem_empty2));  // both regions start zeroed
            }
        }
        Cursor cur = make_cursor(p);
        uint32_t tphase = 0;
        Super su;
        long long e_store = 0, e_carry = 0, e_zero = 0;  // C1D_PROFILE counters
        constexpr int kBR = kMode == 1 ? kKPB : 1;
        float bias_r[kBR][16];  // layer glue (mode 1): this filter group's bias, 0 past the channels
#pragma unroll
        for (int a = 0; a < kBR; ++a)
#pragma unroll
            for (int b = 0; b < 16; ++b) {
                const int64_t k = p.k_begin + a * 16 + b;
                bias_r[a][b] = (kMode == 1 && p.glue.bias && k < p.out_ch) ? __ldg(p.glue.bias + k) : 0.0f;
            }
        // layer glue input prefetch: this warp's blocks are (tile, kbi) for the CTA's tiles [cta_b, cta_e)
        // in order (the super-tile walk emits every output tile once, in increasing order)
        constexpr int kB = kKPB > 0 ? kKPB : 1;
        int64_t cta_b, cta_e;
        cta_tile_range(p, G, &cta_b, &cta_e);
        const int64_t cta_tiles = cta_e - cta_b;
        const int64_t nblk = (cta_tiles > egrp ? (cta_tiles - egrp + kEG - 1) / kEG : 0) * kB;  // this group's blocks
        const bool pf_on = kMode != 0 && (p.pf_rows | p.pf_mask) != 0;
        const uint32_t pf_base = smem_u32(smem) + p.pf_off + static_cast<uint32_t>(ew * kPfRing) * p.pf_slot_bytes;
        int64_t blk = 0, pf_next = 0;
        int64_t pf_n = (cta_b + egrp) / p.tiles_per_item, pf_o = (cta_b + egrp) % p.tiles_per_item;  // block pf_next
        int pf_kbi = 0;
        auto pf_issue = [&]() {
            if (pf_next < nblk) {
                glue_prefetch(p, pf_n, pf_o, pf_kbi, pf_base + static_cast<uint32_t>(pf_next & (kPfRing - 1)) * p.pf_slot_bytes,
                              quarter, lane);
                if (++pf_kbi == kB) {
                    pf_kbi = 0;
                    for (int e = 0; e < kEG; ++e) {
                        if (++pf_o == p.tiles_per_item) {
                            pf_o = 0;
                            ++pf_n;
                        }
                    }
                }
            }
            cp_async_commit();
            ++pf_next;
        };
        if (pf_on)
            for (int i = 0; i < kPfRing - 1; ++i) pf_issue();
        // the slot of the next block, once its copies have landed
        auto pf_take = [&]() -> uint32_t {
            uint32_t slot = 0;
            if (pf_on) {
                pf_issue();
                cp_async_wait_group<kPfRing - 1>();
                slot = pf_base + static_cast<uint32_t>(blk & (kPfRing - 1)) * p.pf_slot_bytes;
            }
            ++blk;
            return slot;
        };
        uint32_t sbuf = 0;  // layer glue: this warp's staging buffer (0/1) and its shared-memory base
        const uint32_t wbase = smem_u32(smem) + p.stg_off + static_cast<uint32_t>(ew) * 2u * p.stg_bytes;
        constexpr int kBS = kMode == 2 ? kKPB : 1;
        float bsum[kBS][16];  // layer glue (mode 2): this lane's bias-gradient sums per channel
#pragma unroll
        for (int a = 0; a < kBS; ++a)
#pragma unroll
            for (int b = 0; b < 16; ++b) bsum[a][b] = 0.0f;
        uint32_t region = 0;  // mirrors the MMA warp's double-buffer region
        const uint32_t used_cols = static_cast<uint32_t>((T + G - 1) * KP);
        // output tile o of item n belongs to this epilogue group?
        auto mine = [&](int64_t n, int64_t o) -> bool {
            return kEG == 1 || (((n * J + o - cta_b) & (kEG - 1)) == egrp);
        };
        // carry the G-1 partial slots (tcur..tcur+G-2) of `src` into slots 0..G-2 of `dst` (or zero
        // them at a segment end) and zero dst's remaining used slots: dst is then ready
        auto prepare = [&](uint32_t src, uint32_t dst, const Super& s2) {
            for (uint32_t reg = 0; reg <= pl.acc2; reg += (pl.acc2 ? pl.acc2 : 1u)) {
                // the carried run (G-1 slots) is contiguous in both places; two 16-column loads in
                // flight per round trip (the MMA warp waits for this pass)
                const uint32_t run = static_cast<uint32_t>((G - 1) * KP);
                const uint32_t from = lane_base + src + reg + static_cast<uint32_t>(s2.tcur * KP);
                const uint32_t to = lane_base + dst + reg;
                if (!s2.last_in_segment) {
                    uint32_t col = 0;
                    for (; col + 32 <= run; col += 32) {
                        uint32_t va[16], vb[16];
                        tmem_ld16(from + col, va);
                        tmem_ld16(from + col + 16, vb);
                        tmem_ld_wait();
                        tmem_st16(to + col, va);
                        tmem_st16(to + col + 16, vb);
                    }
                    for (; col < run; col += 16) {
                        uint32_t v[16];
                        tmem_ld16(from + col, v);
                        tmem_ld_wait();
                        tmem_st16(to + col, v);
                    }
                } else if (dst != src) {
                    for (uint32_t col = 0; col < run; col += 16) tmem_st16(to + col, z);
                }
                for (uint32_t col = run; col < used_cols; col += 16) tmem_st16(lane_base + dst + reg + col, z);
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&tmem_empty));
        };
        // double buffering: carry the G-1 partial slots of `region` into slots 0..G-2 of the other
        // region (zeros at a segment end) and publish them; the other region's remaining slots were
        // zeroed when it was released
        auto carry_out = [&](const Super& s2) {
            for (int j = 0; j < G - 1; ++j) {
                for (int kb = 0; kb < KP; kb += 16) {
                    uint32_t v[16];
                    if (!s2.last_in_segment) {
                        tmem_ld16(lane_base + region + static_cast<uint32_t>((s2.tcur + j) * KP + kb), v);
                        tmem_ld_wait();
                        tmem_st16(lane_base + (region ^ 256u) + static_cast<uint32_t>(j * KP + kb), v);
                    } else {
                        tmem_st16(lane_base + (region ^ 256u) + static_cast<uint32_t>(j * KP + kb), z);
                    }
                }
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&carry_full));
        };
        // double buffering: zero the non-carry slots of `region` after its stores, then release it
        auto release = [&]() {
            for (uint32_t col = static_cast<uint32_t>((G - 1) * KP); col < used_cols; col += 16)
                tmem_st16(lane_base + region + col, z);
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(region ? &tmem_empty2 : &tmem_empty));
        };
        uint32_t tfph = 0;  // staggered finish: parity bit of each tile_full barrier
        auto tile_wait = [&](int j) {
            if (kKPB != 1 && pl.stagger) {
                mbar_wait_sleep(smem_u32(&tile_full[j]), (tfph >> j) & 1u, 64);
                tfph ^= 1u << j;
                tc_fence_after();
            }
        };
        while (next_super(cur, J, G, T, &su)) {
            if (kKPB == 1 || !pl.stagger) {
                mbar_wait_sleep(smem_u32(&tmem_full), tphase, 256);
                tphase ^= 1;
                tc_fence_after();
            }
            const long long e0 = clock64();
            if (pl.dbuf && egrp == 0) carry_out(su);  // the next super-tile's carry-dependent tiles may start
            const long long e1 = clock64();
            // store the completed outputs (slots 0..tcur-1)
            const int64_t out_w = p.out_w;
            float* const out_item = p.out + su.n * p.out_ch * out_w;
            if constexpr (kMode == 1) {  // fused forward glue instead of the plain store
                for (int j = 0; j < su.tcur; ++j) {
                    tile_wait(j);
                    const int64_t o = su.i0 - (G - 1) + j;
                    if (o < su.j0 || o > su.j1 || !mine(su.n, o)) continue;
                    const int64_t q = o * kTileQ + quarter * 32 + lane;
#pragma unroll
                    for (int kbi = 0; kbi < kKPB; ++kbi) {
                        uint32_t v[16];
                        tmem_ld16(lane_base + region + static_cast<uint32_t>(j * KP + kbi * 16), v);
                        tmem_ld_wait();
                        if (pl.acc2) {
                            uint32_t v2[16];
                            tmem_ld16(lane_base + pl.acc2 + static_cast<uint32_t>(j * KP + kbi * 16), v2);
                            tmem_ld_wait();
#pragma unroll
                            for (int jj = 0; jj < 16; ++jj) v[jj] = __float_as_uint(__uint_as_float(v[jj]) + __uint_as_float(v2[jj]));
                        }
                        const uint32_t slot = pf_take();
                        glue_forward16<kFx>(p, v, su.n, q, p.k_begin + kbi * 16, lane, bias_r[kbi], sbuf, wbase, &om0,
                                       &om1, &om2, slot);
                    }
                }
            } else if constexpr (kMode == 2) {  // fused backward glue
                for (int j = 0; j < su.tcur; ++j) {
                    tile_wait(j);
                    const int64_t o = su.i0 - (G - 1) + j;
                    if (o < su.j0 || o > su.j1 || !mine(su.n, o)) continue;
                    const int64_t q = o * kTileQ + quarter * 32 + lane;
#pragma unroll
                    for (int kbi = 0; kbi < kKPB; ++kbi) {
                        uint32_t v[16];
                        tmem_ld16(lane_base + region + static_cast<uint32_t>(j * KP + kbi * 16), v);
                        tmem_ld_wait();
                        if (pl.acc2) {
                            uint32_t v2[16];
                            tmem_ld16(lane_base + pl.acc2 + static_cast<uint32_t>(j * KP + kbi * 16), v2);
                            tmem_ld_wait();
#pragma unroll
                            for (int jj = 0; jj < 16; ++jj) v[jj] = __float_as_uint(__uint_as_float(v[jj]) + __uint_as_float(v2[jj]));
                        }
                        const uint32_t slot = pf_take();
                        glue_backward16<kFx>(p, v, su.n, q, p.k_begin + kbi * 16, lane, bsum[kbi], sbuf, wbase, &om0,
                                        &om1, &om2, slot);
                    }
                }
            } else
            for (int j = 0; j < su.tcur; ++j) {
                tile_wait(j);
                const int64_t o = su.i0 - (G - 1) + j;
                if (o < su.j0 || o > su.j1 || !mine(su.n, o)) continue;  // phantom (warm-up / beyond the segment)
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
            // both groups are done with this region before group 0 overwrites it (next prepare)
            if (kEG > 1) asm volatile("bar.sync 4, %0;" ::"n"(128 * kEG) : "memory");
            if (!pl.dbuf) {
                if (egrp == 0) prepare(0, 0, su);  // in place: carry down, zero the rest, release
                e_carry += clock64() - e2;
            } else {
                if (egrp == 0) release();
                e_carry += e1 - e0;
                e_zero += clock64() - e2;
                region ^= 256u;
            }
        }
        if (kMode != 0 && p.tma_slots && lane == 0) bulk_wait<0>();
        if (kMode == 2 && p.glue.part) {
            // fixed-order CTA partial per channel: warp butterfly, then quarters 0..3 in order
#pragma unroll
            for (int kbi = 0; kbi < kBS; ++kbi) {
#pragma unroll
                for (int jj = 0; jj < 16; ++jj) {
                    float t = bsum[kbi][jj];
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
                    if (lane == 0) bias_red[ew * 64 + kbi * 16 + jj] = t;
                }
            }
            asm volatile("bar.sync 1, %0;" ::"n"(128 * kEG) : "memory");  // all epilogue warps
            const int c = threadIdx.x - 128;
            if (c < KP && p.k_begin + c < p.out_ch) {
                float t = 0.0f;
                for (int w = 0; w < 4 * kEG; ++w) t += bias_red[w * 64 + c];  // fixed order
                p.glue.part[(p.k_begin + c) * p.glue.part_stride + blockIdx.x] = t;
            }
        }
        if (p.prof && threadIdx.x == 128) {
            p.prof[blockIdx.x * kProfSlots + 5] = e_store;
            p.prof[blockIdx.x * kProfSlots + 6] = e_carry;
            p.prof[blockIdx.x * kProfSlots + 7] = e_zero;
            p.prof[blockIdx.x * kProfSlots + 9] = globaltimer_ns();
            p.prof[blockIdx.x * kProfSlots + 11] = clock64();
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


// Tensor maps of the glue outputs for the TMA-store epilogue: (width, channel rows, items) with a
// 32 x 16 x 1 box. Every requested output must be 16-B aligned with 16-B row pitches and start at
// a column that is a multiple of 8 (the tiles start at multiples of 32); otherwise the epilogue
// uses per-lane global stores for the whole launch.
struct GlueMaps {
    CUtensorMap m[3];
    uint32_t slots = 0, stg_bytes = 0, a = 0, b = 0, c = 0;
};
bool glue_maps(const ConvGeom& g, const LayerGlue& gl, PFN_cuTensorMapEncodeTiled_v12000 encode, GlueMaps* out) {
    const bool fwd = gl.mode == 1;
    const int64_t width = fwd ? g.out_w : gl.g_q;
    void* ptr[3] = {fwd ? static_cast<void*>(gl.pre) : static_cast<void*>(gl.gsum),
                    fwd ? static_cast<void*>(gl.act) : static_cast<void*>(gl.gp),
                    fwd ? static_cast<void*>(gl.act_bf16) : static_cast<void*>(gl.gp_bf16)};
    const int64_t pitch[3] = {width, width, fwd ? gl.act_pitch : width};
    const int64_t dim0[3] = {width, width, fwd ? gl.act_off + width : width};
    const int64_t col_off = fwd ? gl.act_off : gl.g_off;
    if (col_off % 8) return false;
    GlueMaps r;
    uint32_t off = 0;
    for (int i = 0; i < 3; ++i) {
        if (!ptr[i]) continue;
        const int64_t esz = i == 2 ? 2 : 4;
        if ((reinterpret_cast<uintptr_t>(ptr[i]) & 15u) || (pitch[i] * esz) % 16) return false;
        const cuuint64_t dims[3] = {static_cast<cuuint64_t>(dim0[i]), static_cast<cuuint64_t>(g.out_ch),
                                    static_cast<cuuint64_t>(g.n)};
        const cuuint64_t strides[2] = {static_cast<cuuint64_t>(pitch[i] * esz),
                                       static_cast<cuuint64_t>(pitch[i] * esz * g.out_ch)};
        const cuuint32_t box[3] = {32, 16, 1};
        const cuuint32_t estr[3] = {1, 1, 1};
        if (encode(&r.m[i], i == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, ptr[i], dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return false;
        r.slots |= 1u << i;
        (i == 0 ? r.a : i == 1 ? r.b : r.c) = off;
        off += static_cast<uint32_t>(32 * 16 * esz);
    }
    r.stg_bytes = off;
    *out = r;
    return true;
}

}  // namespace

int64_t tc_conv_xr_rows(const ConvGeom& g) {
    if (g.dil != 1 && g.dil != 2 && g.dil != 4) return 0;
    return ceil_div(g.out_w, kTileQ) * (kTileQ / g.dil) + kTapsPerBlock * ceil_div(g.taps, kTapsPerBlock) + 8;
}

int tc_conv_carry_tiles(const ConvGeom& g, int64_t main_ch) {
    Plan pl;
    ConvGeom gc = g;
    gc.xr_inline = false;
    gc.xr_rows = 0;
    return make_plan(gc, &pl, main_ch) ? pl.t : 0;
}

int pl_probe_kp(const ConvGeom& g, int64_t main_ch) {
    Plan pl;
    return make_plan(g, &pl, main_ch) ? pl.kp : 0;
}

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

// Prepacked images (c1d_pack_weights): plans whose main image is the whole B operand (no tail
// image, natural rows, one accumulator region); the layout depends only on (KP, G, filter groups, C).
size_t tc_conv_prepack_bytes(const ConvGeom& g) {
    Plan pl;
    if (g.xr_rows > 0 || g.xr_inline || !make_plan(g, &pl)) return 0;
    if (pl.tail || pl.kp > 32) return 0;
    if (static_cast<int64_t>(pl.kgroups) * g.in_ch * pl.ntot * kTapsPerBlock >= (int64_t{1} << 31)) return 0;
    if (g.out_ch * g.in_ch * g.taps >= (int64_t{1} << 31)) return 0;
    return static_cast<size_t>(pl.kgroups) * static_cast<size_t>(g.in_ch) * pl.b_chan_bytes;
}

cudaError_t launch_pack_images_multi(int count, const ConvGeom* gs, const float* const* w, const int* bwd_raw,
                                     void* const* images, cudaStream_t stream) {
    for (int j0 = 0; j0 < count; j0 += kMaxPackJobs) {
        PackJobs jobs{};
        int64_t total = 0;
        for (int j = j0; j < count && j - j0 < kMaxPackJobs; ++j) {
            Plan pl;
            if (!tc_conv_prepack_bytes(gs[j]) || !make_plan(gs[j], &pl)) return cudaErrorInvalidValue;
            PackJob& jb = jobs.j[jobs.count++];
            jb.w = w[j];
            jb.img = static_cast<uint16_t*>(images[j]);
            jb.bwd_raw = bwd_raw[j];
            jb.out_ch = static_cast<int32_t>(gs[j].out_ch);
            jb.in_ch = static_cast<int32_t>(gs[j].in_ch);
            jb.taps = static_cast<int32_t>(gs[j].taps);
            jb.kp = pl.kp;
            jb.g = pl.g;
            jb.kgroups = pl.kgroups;
            jb.begin = total;
            total += static_cast<int64_t>(pl.kgroups) * gs[j].in_ch * pl.ntot * kTapsPerBlock;
        }
        jobs.total = total;
        const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(total, 256), 4096));
        if (blocks > 0) {
            // a plain launch (no PDL trigger): the next kernel starts after this one completes, so
            // the images are complete before any conv that loads them early
            pack_images_multi_kernel<<<blocks, 256, 0, stream>>>(jobs);
            note_launch();
            const cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) return e;
        }
    }
    return cudaSuccess;
}

cudaError_t launch_tc_conv(const uint16_t* in_bf16, const float* wg, float* out, const ConvGeom& g, void* workspace,
                           cudaStream_t stream, int64_t main_ch, bool w_bwd_raw, const LayerGlue* glue,
                           const uint16_t* prepacked) {
    auto encode = get_encode_fn();
    if (!encode) return cudaErrorNotSupported;
    GlueMaps gm;
    static const bool no_glue_tma = getenv("C1D_NO_GLUE_TMA") != nullptr;  // dev A/B switch
    // TMA-store staging for the forward glue only: the backward glue's per-lane stores measured
    // faster (config-5 body layer with gadd + gsum: 173 vs 187 us; without: 139 vs 141 us)
    static const bool bwd_glue_tma = getenv("C1D_BWD_GLUE_TMA") != nullptr;  // dev A/B switch
    if (glue && glue->mode != 0 && !no_glue_tma && (glue->mode == 1 || bwd_glue_tma) &&
        !glue_maps(g, *glue, encode, &gm))
        gm = GlueMaps{};
    const int mode = glue ? glue->mode : 0;
    // glue epilogue groups: two for narrow filter blocks (<= 32 filters per launch, the network's
    // layers), whose glue is issue-bound; one otherwise (register budget at 384 threads)
    static const bool one_group = getenv("C1D_GLUE_EG1") != nullptr;  // dev A/B switch
    int eg = (mode != 0 && g.out_ch <= 32 && !one_group) ? 2 : 1;
    if (mode != 0 && pl_probe_kp(g, main_ch) > 64) return cudaErrorNotSupported;  // glue: KP <= 64
    const uint32_t pf_rows = (mode == 1 && glue->skip) || (mode == 2 && glue->gadd);
    const uint32_t pf_mask = mode == 2 && glue->mask_in;
    const uint32_t pf_slot = pf_rows * 2048u + pf_mask * 128u;  // rows: 16 x 32 fp32, mask: 32 words
    // staging (epilogue warps x 2 buffers) and prefetch rings scale with the epilogue warps; a
    // second group that leaves too few pipeline stages falls back to one
    uint32_t stg_total = 0, pf_total = 0, extra = 0;
    Plan pl;
    for (;; eg = 1) {
        stg_total = 4u * eg * 2u * gm.stg_bytes;
        pf_total = 4u * eg * kPfRing * pf_slot;
        extra = stg_total + pf_total;
        if (make_plan(g, &pl, main_ch, extra ? extra + 1024 : 0)) break;
        if (eg == 1) return cudaErrorNotSupported;
    }
    uint32_t stg_off = 0, pf_off = 0;
    if (extra) {
        const uint32_t stage =
            pl.x_stage_bytes + pl.w_stage_bytes + pl.tx_stage_bytes + pl.tw_stage_bytes + pl.raw_stage_bytes;
        stg_off = (pl.wres_bytes + static_cast<uint32_t>(pl.stages) * stage + 127u) & ~127u;
        pf_off = stg_off + stg_total;
        pl.smem_bytes = pf_off + pf_total + 1024;
    }
    uint16_t* img = prepacked ? const_cast<uint16_t*>(prepacked) : static_cast<uint16_t*>(workspace);
    const int64_t n_chunks = ceil_div(g.in_ch, pl.cc);
    uint16_t* img_tail = img + static_cast<size_t>(pl.kgroups) * g.in_ch * (pl.b_chan_bytes / 2);
    if (prepacked && (pl.tail || pl.xr || pl.kp > 32 || main_ch > 0)) return cudaErrorInvalidValue;
    if (!prepacked) {
        const int64_t total = static_cast<int64_t>(pl.kgroups) *
                              (g.in_ch * pl.ntot + (pl.tail ? n_chunks * pl.kp : 0)) * kTapsPerBlock;
        const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(total, 256), 4096));
        note_launch();
        const bool i32 = total + 256 * 4096 < (int64_t{1} << 31) &&
                         static_cast<int64_t>(g.out_ch) * g.in_ch * g.taps < (int64_t{1} << 31);
        cudaError_t e = i32 ? launch_pdl(pack_images_kernel<int32_t>, dim3(blocks), dim3(256), 0, stream, wg,
                                         w_bwd_raw ? 1 : 0, img, img_tail, static_cast<int64_t>(g.out_ch),
                                         static_cast<int64_t>(g.in_ch), static_cast<int64_t>(g.taps), pl.kp, pl.g,
                                         pl.kgroups, pl.cc, pl.tail, n_chunks)
                            : launch_pdl(pack_images_kernel<int64_t>, dim3(blocks), dim3(256), 0, stream, wg,
                                         w_bwd_raw ? 1 : 0, img, img_tail, static_cast<int64_t>(g.out_ch),
                                         static_cast<int64_t>(g.in_ch), static_cast<int64_t>(g.taps), pl.kp, pl.g,
                                         pl.kgroups, pl.cc, pl.tail, n_chunks);
        if (e != cudaSuccess) return e;
    }
    CUtensorMap tmap;
    CUresult r;
    if (pl.xr && !pl.xin) {  // the row tensor E: (8 elements, rows, item x channel)
        const cuuint64_t dims[3] = {64, static_cast<cuuint64_t>(g.xr_rows / 8), static_cast<cuuint64_t>(g.n * g.in_ch)};
        const cuuint64_t strides[2] = {128, static_cast<cuuint64_t>(g.xr_rows) * 16};
        const cuuint32_t box[3] = {64, static_cast<cuuint32_t>(pl.box_rows / 8), 1};
        const cuuint32_t estr[3] = {1, 1, 1};
        r = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<uint16_t*>(in_bf16), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
        const cuuint64_t dims[2] = {static_cast<cuuint64_t>(g.in_w), static_cast<cuuint64_t>(g.n * g.in_ch)};
        const cuuint64_t strides[1] = {static_cast<cuuint64_t>(g.in_stride ? g.in_stride : g.in_w) * 2};
        const cuuint32_t box[2] = {static_cast<cuuint32_t>(kSegQ), 1};
        const cuuint32_t estr[2] = {1, 1};
        r = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<uint16_t*>(in_bf16), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    CUtensorMap tmap_tail = tmap;  // unused unless pl.tail / pl.xbox3
    pl.xbox3 = 0;
    static const bool no_box3 = getenv("C1D_NO_BOX3") != nullptr;  // dev A/B switch
    if (!pl.tail && !pl.xr && !no_box3 && pl.n_seg * kSegQ == pl.xw) {
        // overlapping view: element (i, j, row) at row*pitch + i + 256 j (see Plan::xbox3)
        const int64_t pitch = g.in_stride ? g.in_stride : g.in_w;
        const cuuint64_t d3[3] = {static_cast<cuuint64_t>(g.in_w), static_cast<cuuint64_t>(pl.n_seg),
                                  static_cast<cuuint64_t>(g.n * g.in_ch)};
        const cuuint64_t s3[2] = {static_cast<cuuint64_t>(kSegQ) * 2, static_cast<cuuint64_t>(pitch) * 2};
        const cuuint32_t b3[3] = {static_cast<cuuint32_t>(kSegQ), static_cast<cuuint32_t>(pl.n_seg),
                                  static_cast<cuuint32_t>(pl.cc)};
        const cuuint32_t e3[3] = {1, 1, 1};
        if (pl.cc * pl.xw * 2 <= static_cast<int>(pl.x_stage_bytes) &&
            encode(&tmap_tail, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<uint16_t*>(in_bf16), d3, s3, b3, e3,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
            pl.xbox3 = 1;
        else
            tmap_tail = tmap;
    }
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
    // KP = 16 plans get their own instantiation (kKPB = 1) with the straight-line narrow issue
    auto kernel = pl.kp == 16 ? tc_conv_kernel<0, 1, 1> : tc_conv_kernel<0, 0, 1>;
    if (mode == 1)
        kernel = pl.kp == 16 ? (eg == 2 ? tc_conv_kernel<1, 1, 2> : tc_conv_kernel<1, 1, 1>)
               : (pl.kp == 32 ? (eg == 2 ? tc_conv_kernel<1, 2, 2> : tc_conv_kernel<1, 2, 1>) : tc_conv_kernel<1, 4, 1>);
    if (mode == 2)
        kernel = pl.kp == 16 ? (eg == 2 ? tc_conv_kernel<2, 1, 2> : tc_conv_kernel<2, 1, 1>)
               : (pl.kp == 32 ? (eg == 2 ? tc_conv_kernel<2, 2, 2> : tc_conv_kernel<2, 2, 1>) : tc_conv_kernel<2, 4, 1>);
    // the network's layer shapes with their glue flags fixed at compile time (glue_forward16 /
    // glue_backward16 kFx): narrow filter blocks, two epilogue groups
    static const bool no_fx = getenv("C1D_NO_GLUE_FX") != nullptr;  // dev A/B switch
    if (mode != 0 && pl.kp == 16 && eg == 2 && !no_fx && !pl.xr && !pl.xin && pl.dbuf && !pl.acc2 && !pl.tail &&
        !pl.stagger && pl.ws) {
        const LayerGlue& gl = *glue;
        if (mode == 1 && gl.relu && gl.mask_out && gl.act_bf16 && !gl.pre) {
            if (!gl.skip && !gl.act && gm.slots == 4u) kernel = tc_conv_kernel<1, 1, 2, 1>;
            else if (gl.skip && gl.act && gm.slots == 6u) kernel = tc_conv_kernel<1, 1, 2, 2>;
            else if (!gl.skip && gl.act && gm.slots == 6u) kernel = tc_conv_kernel<1, 1, 2, 3>;
        } else if (mode == 1 && gl.relu && gl.mask_out && !gl.act_bf16 && !gl.pre && gl.skip && gl.act &&
                   gm.slots == 2u) {
            kernel = tc_conv_kernel<1, 1, 2, 4>;
        } else if (mode == 2 && gl.mask_in && gl.gp_bf16 && !gl.gp && gm.slots == 0u) {
            if (!gl.gadd && !gl.gsum) kernel = tc_conv_kernel<2, 1, 2, 1>;
            else if (gl.gadd && gl.gsum) kernel = tc_conv_kernel<2, 1, 2, 2>;
            else if (gl.gadd && !gl.gsum) kernel = tc_conv_kernel<2, 1, 2, 3>;
        }
    }
    static const bool no_lean = getenv("C1D_NO_LEAN") != nullptr;  // dev A/B switch
    if (mode == 0 && pl.kp != 16 && !pl.xr && !pl.xin && !pl.dbuf && !pl.ws && !pl.wres_bytes && !pl.acc2 && !no_lean)
        kernel = tc_conv_kernel<0, 0, 1, 0, 1>;
    // kLean 2: the plain KP = 16 kernel on a natural-row, double-buffered, one-region plan (config 2)
    if (mode == 0 && pl.kp == 16 && !pl.xr && !pl.xin && pl.dbuf && !pl.acc2 && !pl.tail && !pl.stagger && pl.ws &&
        !no_lean)
        kernel = tc_conv_kernel<0, 1, 1, 0, 2>;
    const int threads = 128 + 128 * eg;
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
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
    kp.early_w = prepacked && pl.wres_bytes ? 1 : 0;
    kp.tma_slots = gm.slots;
    kp.stg_off = stg_off;
    kp.stg_bytes = gm.stg_bytes;
    kp.stg_a = gm.a;
    kp.stg_b = gm.b;
    kp.stg_c = gm.c;
    kp.pf_off = pf_off;
    kp.pf_slot_bytes = pf_slot;
    kp.pf_rows = pf_rows;
    kp.pf_mask = pf_mask;
    if (glue && pf_rows) {
        const int64_t w = mode == 1 ? g.out_w : glue->g_q;
        const float* rows = mode == 1 ? glue->skip : glue->gadd;
        kp.pf_vec = w % 4 == 0 && (mode == 1 || glue->g_off % 4 == 0) && (reinterpret_cast<uintptr_t>(rows) & 15u) == 0;
    }
    const int grid = static_cast<int>(std::min<int64_t>(num_sms(), kp.total_tiles));
    if (glue && glue->mode != 0) {
        kp.glue = *glue;
        kp.glue.part_stride = grid;
        if (glue->mode == 2 && glue->bias_grad && !glue->part) return cudaErrorInvalidValue;
    }
    static const bool profile = getenv("C1D_PROFILE") != nullptr;
    if (profile) {
        cudaMalloc(&kp.prof, sizeof(unsigned long long) * kProfSlots * grid);
        cudaMemset(kp.prof, 0, sizeof(unsigned long long) * kProfSlots * grid);
    }
    for (int kg = 0; kg < pl.kgroups; ++kg) {
        kp.k_begin = kg * pl.kp;
        kp.bimg = img + static_cast<size_t>(kg) * g.in_ch * (pl.b_chan_bytes / 2);
        kp.bimg_tail = img_tail + static_cast<size_t>(kg) * n_chunks * (pl.tw_stage_bytes / 2);
        e = launch_pdl(kernel, dim3(grid), dim3(threads), pl.smem_bytes, stream, tmap, tmap_tail,
                       gm.slots & 1u ? gm.m[0] : tmap, gm.slots & 2u ? gm.m[1] : tmap, gm.slots & 4u ? gm.m[2] : tmap, kp);
        note_launch();
        if (e != cudaSuccess) return e;
    }
    if (kp.glue.mode == 2 && kp.glue.bias_grad) {
        e = launch_bias_grad_reduce(kp.glue.part, kp.glue.bias_grad, 1, g.out_ch, grid, stream);
        if (e != cudaSuccess) return e;
    }
    if (profile) {
        std::vector<unsigned long long> h(kProfSlots * grid);
        cudaMemcpy(h.data(), kp.prof, h.size() * 8, cudaMemcpyDeviceToHost);
        double a[8] = {0}, mma_max = 0;
        unsigned long long t0 = ~0ull, t1 = 0, t1_min = ~0ull;
        double mhz = 0, cta_us = 0, first = 0, nsup = 0, issue = 0;
        for (int b = 0; b < grid; ++b) {
            for (int i = 0; i < 8; ++i) a[i] += static_cast<double>(h[b * kProfSlots + i]) / grid;
            mma_max = std::max(mma_max, static_cast<double>(h[b * kProfSlots + 4]));
            t0 = std::min(t0, h[b * kProfSlots + 8]);
            t1 = std::max(t1, h[b * kProfSlots + 9]);
            t1_min = std::min(t1_min, h[b * kProfSlots + 9]);
            const double dt = static_cast<double>(h[b * kProfSlots + 9] - h[b * kProfSlots + 8]);
            mhz += static_cast<double>(h[b * kProfSlots + 11] - h[b * kProfSlots + 10]) / dt * 1e3 / grid;
            cta_us += dt * 1e-3 / grid;
            first += static_cast<double>(h[b * kProfSlots + 12]) / grid;
            nsup += static_cast<double>(h[b * kProfSlots + 13]) / grid;
            issue += static_cast<double>(h[b * kProfSlots + 14]) / grid;
        }
        fprintf(stderr, "[tc_conv prof] producer wait_empty %.0f / total %.0f | mma wait_full %.0f wait_slot %.0f total %.0f (max %.0f) | epilogue store %.0f carry %.0f zero %.0f (cycles, CTA avg) | span %.1f us, first CTA done %.1f us, CTA avg %.1f us at %.0f MHz | mma waits in super-tile 1: %.0f, super-tiles %.1f, issue %.0f\n",
                a[0], a[1], a[2], a[3], a[4], mma_max, a[5], a[6], a[7], (t1 - t0) * 1e-3, (t1_min - t0) * 1e-3, cta_us, mhz, first, nsup, issue);
        cudaFree(kp.prof);
    }
    return cudaSuccess;
}

}  // namespace c1d
