// c1d_api.cu — the C ABI (include/c1d.h): validation, workspace, kernel selection, dispatch.
//
// Validation mirrors the reference's checks and error classes:
//   validate_params (positivity, BF16 even dims)  proj/src/conv.cpp:33-50  -> SHAPE_MISMATCH / ODD_DIMS
//   check_bf16_widths                             proj/src/conv.cpp:52-57  -> ODD_DIMS (strict mode)
//   output_width / TooNarrow                      proj/src/conv.cpp:142-151
#include <atomic>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/c1d.h"
#include "common.cuh"
#include "kernels.h"

namespace c1d {

static std::atomic<uint64_t> g_launches{0};
void note_launch(int n) { g_launches.fetch_add(static_cast<uint64_t>(n), std::memory_order_relaxed); }

namespace {
thread_local std::string t_last_error;
}
void set_last_error(const char* msg) { t_last_error = msg; }

namespace {
thread_local bool t_exact = false;
}
bool exact_accum() { return t_exact; }
ExactAccumScope::ExactAccumScope(bool on) : saved(t_exact) { t_exact = on; }
ExactAccumScope::~ExactAccumScope() { t_exact = saved; }

int num_sms() {
    static int sms = [] {
        int dev = 0, v = 148;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v > 0 ? v : 148;
    }();
    return sms;
}

namespace {

c1d_status fail(c1d_status st, const std::string& msg) {
    t_last_error = msg;
    return st;
}

c1d_status cuda_fail(cudaError_t e, const char* where) {
    return fail(C1D_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

// Internal workspace (used when the caller passes workspace == NULL): one lazily grown buffer per
// (device, stream), so calls on different streams never share scratch memory; calls on one stream
// are ordered by the stream itself. A buffer that is outgrown is RETIRED, not freed: CUDA graphs
// captured earlier on that stream keep its address, so it stays allocated until the caller
// releases the stream's buffers (c1d_release_workspace). Growing never synchronises, so it is legal
// during stream capture (the allocation itself runs in relaxed capture mode).
struct DeviceWorkspace {
    void* ptr = nullptr;
    size_t bytes = 0;
    std::vector<void*> retired;
};
std::mutex g_ws_mutex;
std::map<std::pair<int, cudaStream_t>, DeviceWorkspace> g_ws;

cudaError_t internal_workspace(size_t need, cudaStream_t stream, void** out) {
    *out = nullptr;
    if (need == 0) return cudaSuccess;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(g_ws_mutex);
    DeviceWorkspace& w = g_ws[{dev, stream}];
    if (w.bytes < need) {
        const size_t grow = need + need / 4;
        void* p = nullptr;
        cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
        cudaThreadExchangeStreamCaptureMode(&mode);
        e = cudaMalloc(&p, grow);
        cudaThreadExchangeStreamCaptureMode(&mode);
        if (e != cudaSuccess) return e;
        if (w.ptr) w.retired.push_back(w.ptr);
        w.ptr = p;
        w.bytes = grow;
    }
    *out = w.ptr;
    return cudaSuccess;
}

// Frees the internal buffers of (current device, stream) after the stream drains. The caller
// guarantees that no captured graph which used them will be replayed again.
cudaError_t release_internal_workspace(cudaStream_t stream) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(g_ws_mutex);
    auto it = g_ws.find({dev, stream});
    if (it == g_ws.end()) return cudaSuccess;
    e = stream ? cudaStreamSynchronize(stream) : cudaDeviceSynchronize();
    if (e != cudaSuccess) return e;
    for (void* p : it->second.retired) cudaFree(p);
    if (it->second.ptr) cudaFree(it->second.ptr);
    g_ws.erase(it);
    return cudaSuccess;
}

bool is_bf16(const c1d_desc& d) { return d.precision == C1D_PRECISION_BF16; }
// FP32 precision always caps its accumulation chains (the reference's 1e-5 bound); BF16 on request
bool exact_for(const c1d_desc& d) { return !is_bf16(d) || (d.flags & C1D_FLAG_EXACT_ACCUM); }

c1d_status validate(const c1d_desc* desc, int64_t* q_out) {
    if (!desc) return fail(C1D_ERR_INVALID_ARGUMENT, "desc is NULL");
    const c1d_desc& d = *desc;
    if (d.c < 1 || d.k < 1 || d.s < 1 || d.d < 1) {
        return fail(C1D_ERR_SHAPE_MISMATCH, "conv params must be positive: C=" + std::to_string(d.c) +
                                                " K=" + std::to_string(d.k) + " S=" + std::to_string(d.s) +
                                                " d=" + std::to_string(d.d));
    }
    if (d.n < 0 || d.w_in < 0) return fail(C1D_ERR_SHAPE_MISMATCH, "negative batch or width");
    if (d.precision != C1D_PRECISION_FP32 && d.precision != C1D_PRECISION_BF16)
        return fail(C1D_ERR_INVALID_ARGUMENT, "unknown precision");
    if (d.in_dtype != C1D_DTYPE_F32 && d.in_dtype != C1D_DTYPE_BF16)
        return fail(C1D_ERR_INVALID_ARGUMENT, "unknown in_dtype");
    if (d.algo < C1D_ALGO_AUTO || d.algo > C1D_ALGO_BF16X3) return fail(C1D_ERR_INVALID_ARGUMENT, "unknown algo");
    const int64_t receptive = d.d * (d.s - 1);
    if (d.w_in <= receptive) {
        return fail(C1D_ERR_TOO_NARROW, "padded width " + std::to_string(d.w_in) +
                                            " does not cover the receptive field d*(S-1) = " +
                                            std::to_string(receptive));
    }
    const int64_t q = d.w_in - receptive;
    if ((d.flags & C1D_FLAG_STRICT_BF16_DIMS) && is_bf16(d)) {
        if (d.c % 2 != 0 || d.k % 2 != 0)
            return fail(C1D_ERR_ODD_DIMS, "bf16 conv needs even channels and filters, got C=" + std::to_string(d.c) +
                                              " K=" + std::to_string(d.k));
        if (d.block_w > 0 && d.block_w % 2 != 0)
            return fail(C1D_ERR_ODD_DIMS, "bf16 conv needs an even width tile, got " + std::to_string(d.block_w));
        if (d.w_in % 2 != 0 || q % 2 != 0)
            return fail(C1D_ERR_ODD_DIMS, "bf16 conv needs even tensor widths, got input " + std::to_string(d.w_in) +
                                              ", output " + std::to_string(q));
    }
    if (d.n > (int64_t{1} << 31) || d.c * d.s > (int64_t{1} << 31) || d.k * d.s > (int64_t{1} << 31))
        return fail(C1D_ERR_UNSUPPORTED, "dimensions too large");
    *q_out = q;
    return C1D_OK;
}

ConvGeom fwd_geom(const c1d_desc& d, int64_t q) {
    return ConvGeom{d.n, d.c, d.w_in, d.k, q, d.s, d.d, 0};
}
ConvGeom bwd_geom(const c1d_desc& d, int64_t q) {
    return ConvGeom{d.n, d.k, q, d.c, d.w_in, d.s, d.d, -d.d * (d.s - 1)};
}

// Dilations other than 8 on the dilation-8 tensor-core kernels (relayout.cu):
//   phases (d < 8, 8 % d == 0): m = 8/d phase channels read with a column shift, S' = ceil(S/m)
//   planes (d = 8m): chunk planes, N*m items of width W/m
struct DilPlan {
    enum Kind { kNative, kPhases, kPlanes, kNone } kind = kNone;
    int64_t m = 1, p = 1, sp = 0;  // factor, phase count min(m, S), taps per phase (ceil(S/m))
};
DilPlan dil_plan(const c1d_desc& d, int64_t q) {
    DilPlan r;
    if (d.d == 8) {
        r.kind = DilPlan::kNative;
    } else if (d.d < 8 && 8 % d.d == 0) {
        r.kind = DilPlan::kPhases;
        r.m = 8 / d.d;
        r.p = std::min<int64_t>(r.m, d.s);
        r.sp = ceil_div(d.s, r.m);
    } else if (d.d % 8 == 0 && q % d.d == 0 && d.w_in % d.d == 0) {
        r.kind = DilPlan::kPlanes;
        r.m = d.d / 8;
    }
    return r;
}
int64_t round8(int64_t v) { return (v + 7) / 8 * 8; }
// Phase copies of a forward-shaped pass: out[n][b*I + i][j] = in[n][i][j + base + b*d] with
// `base` chosen so the conv's remaining column offset is a non-negative multiple of 8 (aligned
// TMA starts); zero columns on the left stand in for the original negative offset's zero fill.
struct PhaseCopy {
    int64_t base, w_out;
};
PhaseCopy phase_copy(const ConvGeom& g) {
    const int64_t fb = ((g.in_off % 8) + 8) % 8;
    const int64_t off1 = g.in_off - fb;  // multiple of 8
    const int64_t padl = off1 < 0 ? -off1 : 0;
    return PhaseCopy{fb - padl, round8(g.in_w + padl)};
}
// geometry of the dilation-8 conv over the phase copies: P*I channels, S' taps
ConvGeom phase_geom(const ConvGeom& g, const DilPlan& dp) {
    const PhaseCopy pc = phase_copy(g);
    ConvGeom r = g;
    r.in_ch = dp.p * g.in_ch;
    r.in_w = pc.w_out;
    r.in_off = g.in_off - pc.base;  // = original offset + left padding - fraction: >= 0, multiple of 8
    r.taps = dp.sp;
    r.dil = 8;
    r.in_stride = 0;
    return r;
}
// plane geometry: N*m items, widths / m, dilation 8 (in_off scales with the width)
ConvGeom plane_geom(const ConvGeom& g, const DilPlan& dp) {
    ConvGeom r = g;
    r.n = g.n * dp.m;
    r.in_w = g.in_w / dp.m;
    r.out_w = g.out_w / dp.m;
    r.dil = 8;
    r.in_off = g.in_off / dp.m;
    return r;
}
// Input rows whose pitch is not a multiple of 8 elements (the 16-B TMA / cp.async granule) go
// through a zero-padded bf16 copy with pitch round8(width).
ConvGeom pitched(ConvGeom g) {
    if (g.in_w % 8) g.in_stride = round8(g.in_w);
    return g;
}
// Expanded-row geometry (d = 1, 2, 4): the conv runs on the row tensor E (launch_expand_rows),
// which absorbs the column offset, so in_off becomes 0.
ConvGeom xr_geom(ConvGeom g) {
    g.xr_rows = tc_conv_xr_rows(g);
    return g;
}
bool xr_ok(const ConvGeom& g) { return (g.dil == 1 || g.dil == 2 || g.dil == 4) && tc_conv_supported(xr_geom(g)); }
// the same mode with E's rows built in shared memory from natural bf16 rows (pitch padded to 8)
ConvGeom xr_inline_geom(const ConvGeom& g) {
    ConvGeom r = pitched(g);
    r.xr_inline = true;
    return r;
}
// Inline pays when the MMAs per expanded row are many enough to hide the expanders' shared-memory
// work: 128/(d*G) rows per (tile, block) MMA <= 32. With few taps at d = 1, 2 the TMA-fed row
// tensor is faster (measured: C = 16, S = 3, d = 1: 60 vs 85 us; C = 64, S = 51, d = 1 bwd-d:
// 327 vs 259 us).
bool xr_inline_ok(const ConvGeom& g) {
    if (g.dil != 1 && g.dil != 2 && g.dil != 4) return false;
    if (g.dil * ceil_div(g.taps, 16) < 4) return false;
    return tc_conv_supported(xr_inline_geom(g));
}
// d = 8 on the carry-free direct mode (the expanded-row mode over the natural rows) for more than
// 64 filters: one 128-wide filter block instead of two carry-mode filter groups that each stream the
// input (measured, N = 16, Q = 20000: C = K = 128, S = 51 fwd 558 -> 499 us, S = 9 292 -> 181 us;
// at K <= 64 the carry mode's N = 192-256 MMAs win: config 3 638 vs 938 us)
bool native_direct(const ConvGeom& g, int64_t main_ch = 0) {
    if (dev_switch(DevSwitch::kD8Carry)) return false;  // dev A/B switch
    if (g.out_ch <= 64 && main_ch == 0) return false;
    // split FP32 (two TMEM regions): only when the carry mode would run tiny super-tiles (FP32
    // config 1, C = K = 15, keeps 8 tiles per super-tile in the carry mode: 99 vs 144 us)
    if (g.out_ch <= 64 && main_ch > 0 && tc_conv_carry_tiles(g, main_ch) >= 4) return false;
    ConvGeom gi = g;
    gi.xr_inline = true;
    return tc_conv_supported(gi, main_ch);
}
// BF16 reduction chains: the tensor core's FP32 accumulation into one TMEM accumulator drifts by
// ~1.2e-9 (norm-relative) per accumulated product, always toward zero (measured: got/true - 1 =
// -6.4e-5 for both signs at 52k products), so a chain of C_in*S products much past ~4k leaves 1e-5
// (C = 160, S = 51: 1.07e-5; the reference's RN FP32 accumulation gives 2.5e-6 there). Under
// C1D_FLAG_EXACT_ACCUM longer reductions run as two chains: the channel halves accumulate in two
// TMEM regions that the epilogue adds in FP32 (the split-FP32 machinery's main_ch).
constexpr int64_t kMaxBf16Chain = 4096;
struct ChainPlan {
    ConvGeom g;
    int64_t main_ch;
};
// native d = 8, no glue: carry mode, or the carry-free direct mode for > 64 filters or two chains
ChainPlan native_choice(const ConvGeom& gq) {
    if (exact_accum() && gq.in_ch * gq.taps > kMaxBf16Chain) {
        const int64_t half = (gq.in_ch + 1) / 2;
        ConvGeom gd = gq;
        gd.xr_inline = native_direct(gq, half);
        if (tc_conv_supported(gd, half)) return ChainPlan{gd, half};
    }
    ConvGeom gk = gq;
    gk.xr_inline = native_direct(gq);
    return ChainPlan{gk, 0};
}
// expanded-row geometries (d < 8): the same mode with two chains when the reduction is long
int64_t xr_main_ch(const ConvGeom& gx) {
    if (!exact_accum() || gx.in_ch * gx.taps <= kMaxBf16Chain) return 0;
    const int64_t half = (gx.in_ch + 1) / 2;
    return tc_conv_supported(gx, half) ? half : 0;
}

// backward-weight on expanded rows (d = 1, 2, 4): one tc_wgrad launch over E (rows of x at every
// d-column start) instead of one launch per phase
int64_t xr_wgrad_rows(const c1d_desc& d, int64_t q_pad) { return ceil_div(q_pad + d.d * (d.s - 1), d.d) + 16; }
// Loader-built rows vs the HBM row tensor for backward-weight (measured, N = 16, Q = 20000): the
// loaders win at C = 16 (d = 1: 48 vs 82 us) and tie at d = 1 for C = 64, 128 (the ring, 8 rows per
// 8 columns, limits both to one K-step per stage); at d = 2, 4 with C >= 64 the row tensor's
// pipelined cp.async stream is faster (C = 128, d = 2: 2286 vs 3501 us).
bool xin_wgrad_preferred(const c1d_desc& d) { return d.c <= 32 || d.d == 1; }
bool xr_wgrad_ok(const c1d_desc& d, int64_t q_pad) {
    return (d.d == 1 || d.d == 2 || d.d == 4) && tc_wgrad_v3_supported(d.n, d.c, d.k, d.s, d.d, q_pad);
}
// backward-weight on channel-octet streams (any d != 8 up to 64; tc_wgrad.cu W2Plan::xt): X relaid
// once as XT[n][C/8][rows][8], every tap shift a descriptor offset: no expanded rows, no phase
// copies, no chunk planes
bool xt_wgrad_ok(const c1d_desc& d, int64_t q_pad) {
    static const bool off = getenv("C1D_NO_XT") != nullptr;     // dev A/B switches
    static const bool at_d8 = getenv("C1D_XT_D8") != nullptr;
    // (d = 4 with <= 32 channels: the expanded-row loaders measured slightly faster, 31.5 vs 34.5 us
    // at C = 16, S = 3)
    if (off || (d.d == 4 && d.c <= 32) || d.d > 64) return false;
    int64_t cp = 16;
    while (cp < d.c) cp *= 2;
    const int64_t t = 128 / cp;  // tap copies stacked on M
    // d = 8: the native plan (P dY copies, N = 256) wins except at T = 1 with long filters
    // (C = K = 128, N = 16, Q = 20000: S = 51 475 vs 560 us, S = 25 276 vs 307, S = 9 158 vs 150)
    if (d.d == 8 && !at_d8 && (t > 1 || d.s < 16)) return false;
    // d = 8m also runs as chunk planes at dilation 8; the octet streams win there only while the
    // copies reach little: measured (config-4 sweep, d = 16) T = 1 or T*d*S <= 600 (C = 32, S = 9:
    // 47 vs 60 us; C = 32, S = 25: 114 vs 69 us)
    if (d.d % 8 == 0 && d.d != 8 && t > 1 && t * d.d * d.s > 600) return false;
    return d.n * ((d.c + 7) / 8) <= 65535 && tc_wgrad_xt_supported(d.n, d.c, d.k, d.s, d.d, q_pad);
}
// the FP32 split's backward-weight problem (2C channels x 2K filters, BF16) and whether it runs
// as one octet-stream launch per split pass (else: the BF16 block passes, the phase / plane plans)
c1d_desc split_wgrad_desc(const c1d_desc& d) {
    c1d_desc d2 = d;
    d2.c = 2 * d.c;
    d2.k = 2 * d.k;
    return d2;
}
bool split_wgrad_xt_ok(const c1d_desc& d, int64_t q) {
    return d.c * 2 <= 128 && d.k * 2 <= 128 && q % 8 == 0 && xt_wgrad_ok(split_wgrad_desc(d), q);
}
int64_t xt_rows(const c1d_desc& d, int64_t q_pad) {
    return std::max<int64_t>(d.w_in, q_pad + d.d * (d.s - 1)) + tc_wgrad_xt_pad_rows(d.n, d.c, d.k, d.s, d.d, q_pad);
}
// backward-weight: Q is padded to a multiple of 8 (zero dY columns add nothing) and x gets a
// zero-padded pitch covering Q_pad + d(S-1) when either width is unaligned.
struct WgradPad {
    bool pad;
    int64_t q_pad, x_pitch;
};
WgradPad wgrad_pad(const c1d_desc& d, int64_t q) {
    WgradPad r;
    r.pad = (d.w_in % 8) || (q % 8);
    r.q_pad = round8(q);
    r.x_pitch = r.pad ? round8(std::max<int64_t>(d.w_in, r.q_pad + d.d * (d.s - 1))) : d.w_in;
    return r;
}
// backward-weight phases: one shifted x copy at a time, pitch covering every phase's reads
int64_t phase_x_pitch(const c1d_desc& d, const WgradPad& wp, const DilPlan& dp) {
    return round8(std::max<int64_t>(d.w_in, wp.q_pad + 8 * (dp.sp - 1)));
}
bool phase_wgrad_ok(const c1d_desc& d, int64_t q, const DilPlan& dp) {
    const int64_t qp = wgrad_pad(d, q).q_pad;
    for (int64_t b = 0; b < dp.p; ++b)
        if (!tc_wgrad_supported(d.n, d.c, d.k, ceil_div(d.s - b, dp.m), 8, qp)) return false;
    return true;
}
// The row-tap kernels put 16 taps of one channel in an MMA's K; a phase carries ceil(S/m) taps, so
// few taps x few channels leave the tensor core mostly idle and the FFMA kernels win. Measured on
// B200 (config-4 sweep): the phase path pays off once taps-per-phase x input channels >= 96.
bool phases_pay_off(const DilPlan& dp, int64_t in_ch) { return dp.sp * in_ch >= 96; }

// FP32 split path (split.cu) composed with the dilation plans: the split multiplies channels
// (4x for conv-shaped passes: [hi|lo|hi|lo] inputs against [hi|hi|lo|lo] weights, main term =
// the first block; 2C x 2K for backward-weight) and is applied after the phase copies / before the
// plane relayout, so every rewrite feeds the same dilation-8 kernels.
struct SplitConv {
    ConvGeom gs;      // geometry the tensor-core kernel runs
    int64_t main_ch;  // channels accumulating in the main TMEM region
};
SplitConv split_conv_geom(const c1d_desc& d, c1d_pass pass, int64_t q, const DilPlan& dp) {
    ConvGeom g = pass == C1D_PASS_FORWARD ? fwd_geom(d, q) : bwd_geom(d, q);
    if (dp.kind == DilPlan::kPhases && (g.dil == 1 || g.dil == 2 || g.dil == 4)) {
        // expanded rows of the split channels: built in shared memory from the natural split rows
        // (the split quadruples the channels, so a row tensor in HBM would be 4 * 8/d x the input),
        // else the row tensor
        ConvGeom g4 = g;
        g4.in_ch *= kSplitBlocks;
        ConvGeom gi = pitched(g4);  // the split rows get an 8-element pitch
        gi.xr_inline = true;
        if (tc_conv_supported(gi, g.in_ch)) return SplitConv{gi, g.in_ch};
        g4 = xr_geom(g4);
        if (tc_conv_supported(g4, g.in_ch)) return SplitConv{g4, g.in_ch};
    }
    if (dp.kind == DilPlan::kNative) {
        // two TMEM regions leave the carry mode 256/KP - (G-1) tiles per super-tile (1 at KP = 64,
        // S = 51), so the carry-free direct mode (4 tiles) runs the split
        ConvGeom g4 = pitched(g);
        g4.in_ch *= kSplitBlocks;
        if (native_direct(g4, g.in_ch)) {
            g4.xr_inline = true;
            return SplitConv{g4, g.in_ch};
        }
    }
    if (dp.kind == DilPlan::kPlanes) g = plane_geom(g, dp);
    if (dp.kind == DilPlan::kPhases) g = phase_geom(g, dp);
    SplitConv r{g, g.in_ch};
    r.gs.in_ch *= kSplitBlocks;
    return r;
}

// FP32 split: main-term products per TMEM accumulation chain (error model in resolve())
constexpr int64_t kMaxSplitTerms = 3300;
bool split_wgrad_blocks(const c1d_desc& d);

// FP32 crossover between the FFMA sliding-window kernels (direct.cu) and the BF16 operand split,
// measured on the BASELINE config-4 sweep (N = 16, Q = 20000, C = K in {16, 32, 64, 128}, S in
// {3, 9, 25, 51}; forced-algorithm sweeps): the split's per-call floor
// (split / pack / sum launches) dominates small problems.
//   forward / backward-data: FFMA while C_in * S is at most a per-dilation limit (the split's
//   d != 8 plans spend more tensor-core work per product than the native one);
//   backward-weight: FFMA while C * K * S (products per output column) is at most 24000 at
//   d = 1, 2, 4 (the split runs on channel-octet streams there) and 3000 otherwise.
int64_t ffma_fp32_limit(c1d_pass pass, int64_t dil) {
    if (pass == C1D_PASS_BACKWARD_WEIGHT) return dil == 1 || dil == 2 || dil == 4 ? 24000 : 3000;
    switch (dil) {
        case 1: return 1000;
        case 2: return 450;
        case 4: return 200;
        case 8: return 150;
        default: return 400;
    }
}
bool ffma_beats_split(const c1d_desc& d, c1d_pass pass) {
    if (pass == C1D_PASS_BACKWARD_WEIGHT) return d.c * d.k * d.s <= ffma_fp32_limit(pass, d.d);
    const int64_t width = pass == C1D_PASS_FORWARD ? d.c : d.k;
    return width * d.s <= ffma_fp32_limit(pass, d.d);
}

// Resolve AUTO.
c1d_algo resolve(const c1d_desc& d, c1d_pass pass, int64_t q) {
    const bool tc_ok = [&] {
        if (!is_bf16(d)) return false;
        const DilPlan dp = dil_plan(d, q);
        if (pass == C1D_PASS_BACKWARD_WEIGHT && xt_wgrad_ok(d, wgrad_pad(d, q).q_pad)) return true;  // any d
        if (dp.kind == DilPlan::kNone) return false;
        if (pass == C1D_PASS_BACKWARD_WEIGHT) {
            const WgradPad wp = wgrad_pad(d, q);
            if (dp.kind == DilPlan::kNative) return tc_wgrad_supported(d.n, d.c, d.k, d.s, 8, wp.q_pad);
            if (dp.kind == DilPlan::kPhases)
                return xr_wgrad_ok(d, wp.q_pad) ||
                       ((d.algo == C1D_ALGO_TCGEN05 || phases_pay_off(dp, d.c)) && phase_wgrad_ok(d, q, dp));
            return tc_wgrad_supported(d.n * dp.m, d.c, d.k, d.s, 8, q / dp.m);
        }
        const ConvGeom g = pitched(pass == C1D_PASS_FORWARD ? fwd_geom(d, q) : bwd_geom(d, q));
        if (dp.kind == DilPlan::kNative) return tc_conv_supported(g);
        if (dp.kind == DilPlan::kPhases) {
            if (xr_ok(g)) return true;
            return (d.algo == C1D_ALGO_TCGEN05 || phases_pay_off(dp, g.in_ch)) && tc_conv_supported(phase_geom(g, dp));
        }
        return tc_conv_supported(plane_geom(g, dp));
    }();
    const bool split_ok = [&] {
        if (is_bf16(d) || d.in_dtype != C1D_DTYPE_F32) return false;
        if (d.algo == C1D_ALGO_AUTO && ffma_beats_split(d, pass)) return false;
        const DilPlan dp = dil_plan(d, q);
        if (pass == C1D_PASS_BACKWARD_WEIGHT && split_wgrad_xt_ok(d, q)) return true;  // any d
        if (dp.kind == DilPlan::kNone) return false;
        if (pass == C1D_PASS_BACKWARD_WEIGHT) {
            // small problems at d < 8 (few taps per phase x channels) stay on the sliding-window FFMA
            // kernel (direct.cu): faster there than the split's expanded rows
            if (split_wgrad_blocks(d))
                return dp.kind != DilPlan::kPhases || d.algo == C1D_ALGO_BF16X3 || phases_pay_off(dp, d.c);
            if (dp.kind == DilPlan::kPlanes) return tc_wgrad_supported(d.n * dp.m, 2 * d.c, 2 * d.k, d.s, 8, q / dp.m);
            if (dp.kind == DilPlan::kPhases && d.algo != C1D_ALGO_BF16X3 && !phases_pay_off(dp, d.c)) return false;
            if (dp.kind == DilPlan::kPhases && q % 8 == 0 && (d.d == 1 || d.d == 2 || d.d == 4) &&
                tc_wgrad_v3_supported(d.n, 2 * d.c, 2 * d.k, d.s, d.d, q))
                return true;  // expanded rows
            if (d.w_in % 8 || q % 8) return false;
            if (dp.kind == DilPlan::kNative) return tc_wgrad_supported(d.n, 2 * d.c, 2 * d.k, d.s, 8, q);
            if (d.algo != C1D_ALGO_BF16X3 && !phases_pay_off(dp, d.c)) return false;
            for (int64_t b = 0; b < dp.p; ++b)
                if (!tc_wgrad_supported(d.n, 2 * d.c, 2 * d.k, ceil_div(d.s - b, dp.m), 8, q)) return false;
            return true;
        }
        // Error model: each product carries <= 2*2^-18 relative representation error (dropped
        // residuals of the two-level split), and the tensor core's FP32 accumulation adds
        // ~1.5e-9 norm-relative per accumulated main-term product (measured); the correction
        // terms accumulate in their own TMEM region, so only the C_in*S main products form the
        // long chain. Keep C_in*S <= kMaxSplitTerms (<= ~6e-6 + 7.6e-6 worst case, 1e-5 bound);
        // longer reductions run on FFMA.
        const int64_t cin = pass == C1D_PASS_FORWARD ? d.c : d.k;
        if (cin * d.s > 2 * kMaxSplitTerms) return false;  // longer chains: FFMA (up to 2x: two channel halves)
        // Small FP32 problems stay on FFMA (exact FP32 products, smooth in the inputs: the reference's
        // finite-difference acceptance checks at eps 1e-3 resolve the split's 1e-6-level error).
        if (dp.kind == DilPlan::kPhases && d.algo != C1D_ALGO_BF16X3 && !phases_pay_off(dp, cin)) return false;
        const SplitConv sc = split_conv_geom(d, pass, q, dp);
        // the halves read channel subsets through split_channels (not the phase-copy fallback)
        if (cin * d.s > kMaxSplitTerms && dp.kind == DilPlan::kPhases && sc.gs.xr_rows == 0 && !sc.gs.xr_inline)
            return false;
        return tc_conv_supported(sc.gs, sc.main_ch);
    }();
    if (d.algo == C1D_ALGO_AUTO) return tc_ok ? C1D_ALGO_TCGEN05 : (split_ok ? C1D_ALGO_BF16X3 : C1D_ALGO_DIRECT);
    if (d.algo == C1D_ALGO_TCGEN05 && !tc_ok) return static_cast<c1d_algo>(-1);
    if (d.algo == C1D_ALGO_BF16X3 && !split_ok) return static_cast<c1d_algo>(-1);
    return static_cast<c1d_algo>(d.algo);
}

size_t align_up(size_t v) { return (v + 255) & ~size_t{255}; }

size_t split_workspace(const c1d_desc& d, c1d_pass pass, int64_t q);  // dry run of the split paths

size_t workspace_for(const c1d_desc& d, c1d_pass pass, int64_t q, c1d_algo algo) {
    const size_t wbytes = align_up(sizeof(float) * static_cast<size_t>(d.k * d.c * d.s));
    if (algo == C1D_ALGO_BF16X3) return split_workspace(d, pass, q);
    if (algo == C1D_ALGO_DIRECT) {
        if (pass == C1D_PASS_BACKWARD_WEIGHT) return align_up(direct_wgrad_workspace_bytes(d.n, d.c, d.k, d.s, d.d, q));
        return wbytes;
    }
    // tensor-core paths: BF16 copies of FP32 inputs + kernel workspace
    const bool conv_in_f32 = d.in_dtype == C1D_DTYPE_F32;
    const DilPlan dp = dil_plan(d, q);
    if (pass == C1D_PASS_BACKWARD_WEIGHT && xt_wgrad_ok(d, wgrad_pad(d, q).q_pad)) {
        const WgradPad wpd = wgrad_pad(d, q);
        return align_up(sizeof(uint16_t) * static_cast<size_t>(d.n * d.k * wpd.q_pad)) +
               align_up(sizeof(uint16_t) * 8 * static_cast<size_t>(d.n * ((d.c + 7) / 8) * xt_rows(d, wpd.q_pad))) +
               align_up(tc_wgrad_xt_workspace_bytes(d.n, d.c, d.k, d.s, d.d, wpd.q_pad));
    }
    if (pass == C1D_PASS_BACKWARD_WEIGHT && dp.kind == DilPlan::kPhases && xr_wgrad_ok(d, wgrad_pad(d, q).q_pad) &&
        xin_wgrad_preferred(d) && tc_wgrad_xin_supported(d.n, d.c, d.k, d.s, d.d, wgrad_pad(d, q).q_pad)) {
        const WgradPad wpd = wgrad_pad(d, q);
        return align_up(sizeof(uint16_t) * static_cast<size_t>(d.n * d.k * wpd.q_pad)) +
               align_up(sizeof(uint16_t) * static_cast<size_t>(d.n * d.c * round8(d.w_in))) +
               align_up(tc_wgrad_xin_workspace_bytes(d.n, d.c, d.k, d.s, d.d, wpd.q_pad));
    }
    if (pass == C1D_PASS_BACKWARD_WEIGHT && dp.kind == DilPlan::kPhases && xr_wgrad_ok(d, wgrad_pad(d, q).q_pad)) {
        const WgradPad wpd = wgrad_pad(d, q);
        return align_up(sizeof(uint16_t) * static_cast<size_t>(d.n * d.k * wpd.q_pad)) +
               align_up(sizeof(uint16_t) * 8 * static_cast<size_t>(d.n * d.c * xr_wgrad_rows(d, wpd.q_pad))) +
               align_up(tc_wgrad_workspace_bytes(d.n, d.c, d.k, d.s, d.d, wpd.q_pad));
    }
    if (pass == C1D_PASS_BACKWARD_WEIGHT && dp.kind != DilPlan::kPlanes) {
        const WgradPad wpd = wgrad_pad(d, q);
        size_t b = 0;
        if (wpd.pad)
            b += align_up(sizeof(uint16_t) * static_cast<size_t>(d.n * d.c * wpd.x_pitch)) +
                 align_up(sizeof(uint16_t) * static_cast<size_t>(d.n * d.k * wpd.q_pad));
        else if (conv_in_f32)
            b += align_up(sizeof(uint16_t) * static_cast<size_t>(d.n * d.c * d.w_in)) +
                 align_up(sizeof(uint16_t) * static_cast<size_t>(d.n * d.k * q));
        if (dp.kind == DilPlan::kPhases) {
            size_t kws = 0;
            for (int64_t ph = 0; ph < dp.p; ++ph)
                kws = std::max(kws, tc_wgrad_workspace_bytes(d.n, d.c, d.k, ceil_div(d.s - ph, dp.m), 8, wpd.q_pad));
            return b + align_up(sizeof(uint16_t) * static_cast<size_t>(d.n * d.c * phase_x_pitch(d, wpd, dp))) +
                   align_up(sizeof(float) * static_cast<size_t>(d.k * dp.p * d.c * dp.sp)) + align_up(kws);
        }
        return b + align_up(tc_wgrad_workspace_bytes(d.n, d.c, d.k, d.s, 8, wpd.q_pad));
    }
    if (dp.kind == DilPlan::kPhases && xr_inline_ok(pass == C1D_PASS_FORWARD ? fwd_geom(d, q) : bwd_geom(d, q))) {
        const ConvGeom g = xr_inline_geom(pass == C1D_PASS_FORWARD ? fwd_geom(d, q) : bwd_geom(d, q));
        size_t b = wbytes + align_up(std::max(tc_conv_workspace_bytes(g), tc_conv_workspace_bytes(g, xr_main_ch(g))));
        if (g.in_stride || conv_in_f32)
            b += align_up(sizeof(uint16_t) * static_cast<size_t>(g.n * g.in_ch * (g.in_stride ? g.in_stride : g.in_w)));
        return b;
    }
    if (dp.kind == DilPlan::kPhases && xr_ok(pass == C1D_PASS_FORWARD ? fwd_geom(d, q) : bwd_geom(d, q))) {
        const ConvGeom g = xr_geom(pass == C1D_PASS_FORWARD ? fwd_geom(d, q) : bwd_geom(d, q));
        return wbytes + align_up(std::max(tc_conv_workspace_bytes(g), tc_conv_workspace_bytes(g, xr_main_ch(g)))) +
               align_up(sizeof(uint16_t) * 8 * static_cast<size_t>(g.n * g.in_ch * g.xr_rows));
    }
    if (dp.kind == DilPlan::kPhases) {
        const ConvGeom g = phase_geom(pass == C1D_PASS_FORWARD ? fwd_geom(d, q) : bwd_geom(d, q), dp);
        return wbytes + align_up(tc_conv_workspace_bytes(g)) +
               align_up(sizeof(float) * static_cast<size_t>(g.out_ch * g.in_ch * dp.sp)) +
               align_up(sizeof(uint16_t) * static_cast<size_t>(g.n * g.in_ch * g.in_w));
    }
    if (dp.kind == DilPlan::kNative) {
        const ConvGeom g = pitched(pass == C1D_PASS_FORWARD ? fwd_geom(d, q) : bwd_geom(d, q));
        // conv_pass runs the carry mode (glued calls) or native_choice's plan: size for the larger
        const ChainPlan cp = native_choice(g);
        const size_t kws = std::max(tc_conv_workspace_bytes(g), tc_conv_workspace_bytes(cp.g, cp.main_ch));
        size_t b = wbytes + align_up(kws);
        if (g.in_stride || conv_in_f32)
            b += align_up(sizeof(uint16_t) * static_cast<size_t>(g.n * g.in_ch * (g.in_stride ? g.in_stride : g.in_w)));
        return b;
    }
    if (dp.kind == DilPlan::kPlanes) {
        const size_t px = align_up(sizeof(uint16_t) * static_cast<size_t>(d.n * d.c * d.w_in));
        const size_t pdy = align_up(sizeof(uint16_t) * static_cast<size_t>(d.n * d.k * q));
        if (pass == C1D_PASS_BACKWARD_WEIGHT)
            return px + pdy + align_up(tc_wgrad_workspace_bytes(d.n * dp.m, d.c, d.k, d.s, 8, q / dp.m));
        const ConvGeom g = plane_geom(pass == C1D_PASS_FORWARD ? fwd_geom(d, q) : bwd_geom(d, q), dp);
        const size_t pout = align_up(sizeof(float) * static_cast<size_t>(g.n * g.out_ch * g.out_w));
        return wbytes + (pass == C1D_PASS_FORWARD ? px : pdy) + pout + align_up(tc_conv_workspace_bytes(g));
    }
    return wbytes;  // no tensor-core plan (resolve() never selects one)
}

struct Bump {
    char* p;
    size_t left;
    bool dry = false;  // sizing pass: only count (used by workspace_for for the composed paths)
    size_t used = 0;
    bool overflow = false;  // a take() did not fit: the plan's sizing and its run disagree
    template <typename T>
    T* take(size_t bytes) {
        bytes = align_up(bytes);
        used += bytes;
        if (dry) return reinterpret_cast<T*>(alignof(T));  // never dereferenced
        if (bytes > left) {
            overflow = true;
            return nullptr;
        }
        T* r = reinterpret_cast<T*>(p);
        p += bytes;
        left -= bytes;
        return r;
    }
};

c1d_status acquire_workspace(void* user, size_t user_bytes, size_t need, Bump* out, cudaStream_t stream) {
    if (user) {
        if (user_bytes < need)
            return fail(C1D_ERR_WORKSPACE, "workspace of " + std::to_string(user_bytes) + " bytes, need " +
                                               std::to_string(need));
        *out = Bump{static_cast<char*>(user), user_bytes};
        return C1D_OK;
    }
    void* p = nullptr;
    cudaError_t e = internal_workspace(need, stream, &p);
    if (e != cudaSuccess) return cuda_fail(e, "internal workspace");
    *out = Bump{static_cast<char*>(p), need};
    return C1D_OK;
}

// a bump.take() of a running plan did not fit the workspace its sizing pass computed
c1d_status workspace_overflow() {
    return fail(C1D_ERR_WORKSPACE, "workspace too small for the selected plan (internal sizing mismatch)");
}

c1d_status check_device() {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    int major = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    if (major < 10) return fail(C1D_ERR_NO_DEVICE, "needs an sm_100 (B200) device");
    return C1D_OK;
}

// FP32 split path of a conv-shaped pass under its dilation plan (see split_conv_geom). With a dry
// bump only the workspace is sized.
cudaError_t split_conv_run(const c1d_desc& d, c1d_pass pass, int64_t q, const void* in, const float* w_kcs,
                           float* out, Bump& bump, cudaStream_t stream, int64_t in_item_stride = 0) {
    const DilPlan dp = dil_plan(d, q);
    const ConvGeom g = pass == C1D_PASS_FORWARD ? fwd_geom(d, q) : bwd_geom(d, q);
    const SplitConv sc = split_conv_geom(d, pass, q, dp);
    const bool run = !bump.dry;
    const size_t kcs = static_cast<size_t>(d.k * d.c * d.s);
    const int mode = pass == C1D_PASS_FORWARD ? kWeightsForward : kWeightsBackwardData;
    cudaError_t e = cudaSuccess;
    auto step = [&](auto&& launch) {
        if (run && e == cudaSuccess) e = bump.overflow ? cudaErrorInvalidValue : launch();
    };
    if (dp.kind != DilPlan::kPhases || sc.gs.xr_rows > 0 || sc.gs.xr_inline) {
        float* w4 = bump.take<float>(kSplitBlocks * sizeof(float) * kcs);
        float* wg4 = bump.take<float>(kSplitBlocks * sizeof(float) * kcs);
        if (pass == C1D_PASS_FORWARD) {  // c-blocks of the weight parts (kSplitW)
            step([&] { return launch_split_weights(w_kcs, w4, d.k, d.c, d.s, 1, kSplitBlocks, kSplitW, stream); });
            step([&] { return launch_prep_weights(w4, wg4, d.k, kSplitBlocks * d.c, d.s, kWeightsForward, false, stream); });
        } else {  // k-blocks of the weight parts, then the bwd-d transpose
            step([&] { return launch_split_weights(w_kcs, w4, d.k, d.c, d.s, kSplitBlocks, 1, kSplitW, stream); });
            step([&] {
                return launch_prep_weights(w4, wg4, kSplitBlocks * d.k, d.c, d.s, kWeightsBackwardData, false, stream);
            });
        }
        const int64_t x4_pitch = sc.gs.xr_inline && sc.gs.in_stride ? sc.gs.in_stride : g.in_w;
        const size_t n4 = static_cast<size_t>(g.n * kSplitBlocks * g.in_ch * x4_pitch);
        uint16_t* x4 = bump.take<uint16_t>(sizeof(uint16_t) * n4);
        step([&] {
            return launch_split_channels(static_cast<const float*>(in), x4, g.n, g.in_ch, g.in_w, kSplitBlocks, kSplitX, stream, x4_pitch,
                                         in_item_stride);
        });
        if (dp.kind == DilPlan::kPlanes) {
            uint16_t* p4 = bump.take<uint16_t>(sizeof(uint16_t) * n4);
            float* pout = bump.take<float>(sizeof(float) * static_cast<size_t>(sc.gs.n * sc.gs.out_ch * sc.gs.out_w));
            void* kws = bump.take<char>(tc_conv_workspace_bytes(sc.gs, sc.main_ch));
            step([&] { return launch_to_planes(x4, C1D_DTYPE_BF16, p4, g.n, kSplitBlocks * g.in_ch, g.in_w, dp.m, stream); });
            step([&] { return launch_tc_conv(p4, wg4, pout, sc.gs, kws, stream, sc.main_ch); });
            step([&] { return launch_from_planes(pout, out, g.n, g.out_ch, g.out_w, dp.m, stream); });
            return e;
        }
        if (sc.gs.xr_inline) {  // d < 8: expanded rows built in the kernel from the split rows
            void* kws = bump.take<char>(tc_conv_workspace_bytes(sc.gs, sc.main_ch));
            step([&] { return launch_tc_conv(x4, wg4, out, sc.gs, kws, stream, sc.main_ch); });
            return e;
        }
        if (sc.gs.xr_rows > 0) {  // d < 8: expanded rows of the split channels
            uint16_t* ex = bump.take<uint16_t>(sizeof(uint16_t) * 8 * static_cast<size_t>(g.n * kSplitBlocks * g.in_ch * sc.gs.xr_rows));
            void* kws = bump.take<char>(tc_conv_workspace_bytes(sc.gs, sc.main_ch));
            step([&] {
                return launch_expand_rows(x4, C1D_DTYPE_BF16, ex, g.n * kSplitBlocks * g.in_ch, g.in_w, g.dil, g.in_off, sc.gs.xr_rows,
                                          stream);
            });
            step([&] { return launch_tc_conv(ex, wg4, out, sc.gs, kws, stream, sc.main_ch); });
            return e;
        }
        void* kws = bump.take<char>(tc_conv_workspace_bytes(sc.gs, sc.main_ch));
        step([&] { return launch_tc_conv(x4, wg4, out, sc.gs, kws, stream, sc.main_ch); });
        return e;
    }
    // phases: weights prep -> phase split -> hi/lo split; input fp32 phase copies -> hi/lo split
    const int64_t O = g.out_ch, I = g.in_ch, PI = dp.p * g.in_ch;
    float* wg = bump.take<float>(sizeof(float) * kcs);
    float* wph = bump.take<float>(sizeof(float) * static_cast<size_t>(O * PI * dp.sp));
    float* wg4 = bump.take<float>(kSplitBlocks * sizeof(float) * static_cast<size_t>(O * PI * dp.sp));
    step([&] { return launch_prep_weights(w_kcs, wg, d.k, d.c, d.s, mode, false, stream); });
    step([&] { return launch_phase_split_weights(wg, wph, O, I, d.s, dp.m, dp.p, stream); });
    step([&] { return launch_split_weights(wph, wg4, O, PI, dp.sp, 1, kSplitBlocks, kSplitW, stream); });
    const PhaseCopy pc = phase_copy(g);
    const int64_t W2 = sc.gs.in_w;
    float* cp = bump.take<float>(sizeof(float) * static_cast<size_t>(g.n * PI * W2));
    uint16_t* x4 = bump.take<uint16_t>(sizeof(uint16_t) * static_cast<size_t>(g.n * kSplitBlocks * PI * W2));
    void* kws = bump.take<char>(tc_conv_workspace_bytes(sc.gs, sc.main_ch));
    step([&] {
        return launch_shift_copies_f32(static_cast<const float*>(in), cp, g.n, I, g.in_w, dp.p, pc.base, d.d, W2, stream);
    });
    step([&] { return launch_split_channels(cp, x4, g.n, PI, W2, kSplitBlocks, kSplitX, stream); });
    step([&] { return launch_tc_conv(x4, wg4, out, sc.gs, kws, stream, sc.main_ch); });
    return e;
}

// FP32 split conv whose main chain C_in*S exceeds kMaxSplitTerms (native d = 8): the reduction
// channels in two halves (separate launches, hence separate TMEM chains); the second half is added
// to the first in FP32.
cudaError_t split_conv_any(const c1d_desc& d, c1d_pass pass, int64_t q, const void* in, const float* w_kcs,
                           float* out, Bump& bump, cudaStream_t stream) {
    const bool fwd = pass == C1D_PASS_FORWARD;
    const int64_t cin = fwd ? d.c : d.k;
    if (cin * d.s <= kMaxSplitTerms) return split_conv_run(d, pass, q, in, w_kcs, out, bump, stream);
    const bool run = !bump.dry;
    const int64_t h0 = (cin + 1) / 2;
    const int64_t w_in = d.w_in;
    const int64_t in_w = fwd ? w_in : q;  // width of the reduction-channel rows
    const int64_t out_elems = fwd ? d.n * d.k * q : d.n * d.c * w_in;
    float* tmp = bump.take<float>(sizeof(float) * static_cast<size_t>(out_elems));
    float* wsub = bump.take<float>(sizeof(float) * static_cast<size_t>(d.k * d.c * d.s));
    cudaError_t e = cudaSuccess;
    for (int h = 0; h < 2 && e == cudaSuccess; ++h) {
        const int64_t c0 = h ? h0 : 0, nh = h ? cin - h0 : h0;
        c1d_desc dh = d;
        if (fwd)
            dh.c = nh;
        else
            dh.k = nh;
        const float* wh = w_kcs + (fwd ? 0 : c0 * d.c * d.s);
        if (fwd && run)  // channels [c0, c0 + nh) of every filter: a compact [K][nh][S] copy
            e = cudaMemcpy2DAsync(wsub, sizeof(float) * nh * d.s, w_kcs + c0 * d.s, sizeof(float) * d.c * d.s,
                                  sizeof(float) * nh * d.s, d.k, cudaMemcpyDeviceToDevice, stream);
        if (fwd) wh = wsub;
        const float* inh = run ? static_cast<const float*>(in) + c0 * in_w : nullptr;
        if (e == cudaSuccess)
            e = split_conv_run(dh, pass, q, inh, wh, h ? tmp : out, bump, stream, cin * in_w);
        if (e == cudaSuccess && h == 1 && run) e = launch_add_into(out, tmp, out_elems, stream);
    }
    return e;
}

// FP32 split backward-weight in three BF16 block passes when [x_hi | x_lo] / [dy_hi | dy_lo] (2C, 2K
// channels) exceed the single-launch kernels (v3: C, K <= 128) but the BF16 pass runs on (C, K)
bool split_wgrad_blocks(const c1d_desc& d) {
    if (d.c * 2 <= 128 && d.k * 2 <= 128) return false;
    int64_t q = 0;
    if (validate(&d, &q) != C1D_OK) return false;
    c1d_desc d16 = d;
    d16.precision = C1D_PRECISION_BF16;
    d16.in_dtype = C1D_DTYPE_BF16;
    d16.algo = C1D_ALGO_TCGEN05;
    d16.flags = 0;
    return resolve(d16, C1D_PASS_BACKWARD_WEIGHT, q) == C1D_ALGO_TCGEN05;
}

// FP32 split path of backward-weight, three-level split v = hi + mid + lo (split.cu): two launches
// of the (2C, 2K) problem under the dilation plan,
//   A: x' = [x_hi | x_mid], dy' = [dy_hi | dy_mid]      B: x' = [x_hi | x_lo], dy' = [dy_lo | dy_hi]
// whose 2x2 block results combine as hh + (hm + (mh + (hl + (lh + (mm + ll))))) (sum_split3). Under the
// dilation plans the split operands are relaid out exactly as the BF16 ones.
cudaError_t split_wgrad_run(const c1d_desc& d, int64_t q, const void* x, const void* dy, float* dw, Bump& bump,
                            cudaStream_t stream) {
    const DilPlan dp = dil_plan(d, q);
    const bool run = !bump.dry;
    cudaError_t e = cudaSuccess;
    auto step = [&](auto&& launch) {
        if (run && e == cudaSuccess) e = bump.overflow ? cudaErrorInvalidValue : launch();
    };
    const size_t nx = static_cast<size_t>(2 * d.n * d.c * d.w_in), ng = static_cast<size_t>(2 * d.n * d.k * q);
    const size_t kcs = static_cast<size_t>(d.k * d.c * d.s);
    if (split_wgrad_blocks(d)) {
        // 2C or 2K too wide for one launch: six BF16 block passes (dy part x x part: hh, hm, mh, hl,
        // lh, mm) on separate part tensors through the BF16 tensor-core path (any dilation plan),
        // summed in a fixed order
        c1d_desc d16 = d;
        d16.precision = C1D_PRECISION_BF16;
        d16.in_dtype = C1D_DTYPE_BF16;
        d16.algo = C1D_ALGO_TCGEN05;
        d16.flags = C1D_FLAG_EXACT_ACCUM;  // the FP32 result keeps its capped chains
        uint16_t* xp[3];
        uint16_t* gp[3];
        for (int i = 0; i < 3; ++i) xp[i] = bump.take<uint16_t>(sizeof(uint16_t) * nx / 2);
        for (int i = 0; i < 3; ++i) gp[i] = bump.take<uint16_t>(sizeof(uint16_t) * ng / 2);
        float* part = bump.take<float>(6 * sizeof(float) * kcs);
        const size_t inner = workspace_for(d16, C1D_PASS_BACKWARD_WEIGHT, q, C1D_ALGO_TCGEN05);
        char* iws = bump.take<char>(inner);
        for (unsigned i = 0; i < 3; ++i) {
            step([&] { return launch_split_channels(static_cast<const float*>(x), xp[i], d.n, d.c, d.w_in, 1, i, stream); });
            step([&] { return launch_split_channels(static_cast<const float*>(dy), gp[i], d.n, d.k, q, 1, i, stream); });
        }
        const int pairs[6][2] = {{0, 0}, {0, 1}, {1, 0}, {0, 2}, {2, 0}, {1, 1}};  // (dy part, x part)
        for (int b = 0; b < 6; ++b)
            step([&] {
                const c1d_status st = c1d_backward_weight(&d16, xp[pairs[b][1]], gp[pairs[b][0]], part + b * kcs, iws,
                                                          inner, reinterpret_cast<c1d_stream_t>(stream));
                return st == C1D_OK ? cudaSuccess : cudaErrorUnknown;
            });
        step([&] { return launch_sum6(part, dw, static_cast<int64_t>(kcs), stream); });
        return e;
    }
    uint16_t* x2 = bump.take<uint16_t>(sizeof(uint16_t) * nx);
    uint16_t* g2 = bump.take<uint16_t>(sizeof(uint16_t) * ng);
    const unsigned pat_x[2] = {kSplitHM, kSplitHL3}, pat_g[2] = {kSplitHM, kSplitL3H};
    auto split_pass = [&](int pass) {
        step([&] { return launch_split_channels(static_cast<const float*>(x), x2, d.n, d.c, d.w_in, 2, pat_x[pass], stream); });
        step([&] { return launch_split_channels(static_cast<const float*>(dy), g2, d.n, d.k, q, 2, pat_g[pass], stream); });
    };
    // both split passes' operands from one read of x and one of dy (pass 1's into x2b / g2b)
    auto split_both = [&](uint16_t* x2b, uint16_t* g2b) {
        step([&] {
            return launch_split_channels(static_cast<const float*>(x), x2, d.n, d.c, d.w_in, 2, pat_x[0], stream, 0, 0,
                                         x2b, pat_x[1]);
        });
        step([&] {
            return launch_split_channels(static_cast<const float*>(dy), g2, d.n, d.k, q, 2, pat_g[0], stream, 0, 0, g2b,
                                         pat_g[1]);
        });
    };
    const c1d_desc d2 = split_wgrad_desc(d);
    if (split_wgrad_xt_ok(d, q)) {
        // channel-octet streams of the split x, one launch per split pass
        const int64_t rows = xt_rows(d2, q);
        uint16_t* xt = bump.take<uint16_t>(sizeof(uint16_t) * 8 * static_cast<size_t>(d.n * ((d2.c + 7) / 8) * rows));
        float* dw4[2] = {bump.take<float>(4 * sizeof(float) * kcs), bump.take<float>(4 * sizeof(float) * kcs)};
        void* kws = bump.take<char>(tc_wgrad_xt_workspace_bytes(d.n, d2.c, d2.k, d.s, d.d, q));
        uint16_t* x2b = bump.take<uint16_t>(sizeof(uint16_t) * nx);
        uint16_t* g2b = bump.take<uint16_t>(sizeof(uint16_t) * ng);
        split_both(x2b, g2b);
        const uint16_t* xsrc[2] = {x2, x2b};
        const uint16_t* gsrc[2] = {g2, g2b};
        for (int ps = 0; ps < 2; ++ps) {
            step([&] { return launch_to_octets(xsrc[ps], C1D_DTYPE_BF16, xt, d.n, d2.c, d.w_in, rows, stream); });
            step([&] { return launch_tc_wgrad_xt(xt, rows, gsrc[ps], dw4[ps], kws, d.n, d2.c, d2.k, d.s, d.d, q, stream); });
        }
        step([&] { return launch_sum_split3(dw4[0], dw4[1], dw, d.k, d.c, d.s, stream); });
        return e;
    }
    if (dp.kind == DilPlan::kPhases && (d.d == 1 || d.d == 2 || d.d == 4) &&
        tc_wgrad_v3_supported(d.n, 2 * d.c, 2 * d.k, d.s, d.d, q)) {
        // expanded rows of the split x, one launch per split pass
        const int64_t rows = xr_wgrad_rows(d, q);
        uint16_t* ex = bump.take<uint16_t>(sizeof(uint16_t) * 8 * static_cast<size_t>(2 * d.n * d.c * rows));
        float* dw4[2] = {bump.take<float>(4 * sizeof(float) * kcs), bump.take<float>(4 * sizeof(float) * kcs)};
        void* kws = bump.take<char>(tc_wgrad_workspace_bytes(d.n, 2 * d.c, 2 * d.k, d.s, d.d, q));
        for (int ps = 0; ps < 2; ++ps) {
            split_pass(ps);
            step([&] { return launch_expand_rows(x2, C1D_DTYPE_BF16, ex, 2 * d.n * d.c, d.w_in, d.d, 0, rows, stream); });
            step([&] { return launch_tc_wgrad(ex, g2, dw4[ps], kws, d.n, 2 * d.c, 2 * d.k, d.s, d.d, q, stream, rows * 8); });
        }
        step([&] { return launch_sum_split3(dw4[0], dw4[1], dw, d.k, d.c, d.s, stream); });
        return e;
    }
    if (dp.kind == DilPlan::kPhases) {
        const int64_t pitch = round8(std::max<int64_t>(d.w_in, q + 8 * (dp.sp - 1)));
        uint16_t* xs[2] = {bump.take<uint16_t>(sizeof(uint16_t) * static_cast<size_t>(2 * d.n * d.c * pitch)),
                           bump.take<uint16_t>(sizeof(uint16_t) * static_cast<size_t>(2 * d.n * d.c * pitch))};
        uint16_t* g2b = bump.take<uint16_t>(sizeof(uint16_t) * ng);  // pass B's dy split (pass A's stays in g2)
        float* dw4b[2] = {bump.take<float>(4 * sizeof(float) * static_cast<size_t>(d.k * d.c * dp.sp)),
                          bump.take<float>(4 * sizeof(float) * static_cast<size_t>(d.k * d.c * dp.sp))};
        float* dwb = bump.take<float>(sizeof(float) * static_cast<size_t>(d.k * d.c * dp.sp));
        size_t kb = 0;
        for (int64_t b = 0; b < dp.p; ++b)
            kb = std::max(kb, tc_wgrad_workspace_bytes(d.n, 2 * d.c, 2 * d.k, ceil_div(d.s - b, dp.m), 8, q));
        void* kws = bump.take<char>(kb);
        // both splits of dy once; x's two splits are re-shifted per phase
        step([&] {
            return launch_split_channels(static_cast<const float*>(dy), g2, d.n, d.k, q, 2, pat_g[0], stream, 0, 0, g2b,
                                         pat_g[1]);
        });
        const uint16_t* gsrc[2] = {g2, g2b};
        for (int64_t b = 0; b < dp.p; ++b) {
            const int64_t sb = ceil_div(d.s - b, dp.m);
            for (int ps = 0; ps < 2; ++ps) {
                step([&] {
                    return launch_split_channels(static_cast<const float*>(x), x2, d.n, d.c, d.w_in, 2, pat_x[ps], stream);
                });
                step([&] { return launch_shift_copies(x2, C1D_DTYPE_BF16, xs[ps], d.n, 2 * d.c, d.w_in, 1, b * d.d, 0, pitch, stream); });
                step([&] { return launch_tc_wgrad(xs[ps], gsrc[ps], dw4b[ps], kws, d.n, 2 * d.c, 2 * d.k, sb, 8, q, stream, pitch); });
            }
            step([&] { return launch_sum_split3(dw4b[0], dw4b[1], dwb, d.k, d.c, sb, stream); });
            step([&] { return launch_scatter_phase_wgrad(dwb, dw, d.k, d.c, d.s, dp.m, b, stream); });
        }
        return e;
    }
    float* dw4[2] = {bump.take<float>(4 * sizeof(float) * kcs), bump.take<float>(4 * sizeof(float) * kcs)};
    if (dp.kind == DilPlan::kPlanes) {
        uint16_t* px = bump.take<uint16_t>(sizeof(uint16_t) * nx);
        uint16_t* pg = bump.take<uint16_t>(sizeof(uint16_t) * ng);
        void* kws = bump.take<char>(tc_wgrad_workspace_bytes(d.n * dp.m, 2 * d.c, 2 * d.k, d.s, 8, q / dp.m));
        for (int ps = 0; ps < 2; ++ps) {
            split_pass(ps);
            step([&] { return launch_to_planes(x2, C1D_DTYPE_BF16, px, d.n, 2 * d.c, d.w_in, dp.m, stream); });
            step([&] { return launch_to_planes(g2, C1D_DTYPE_BF16, pg, d.n, 2 * d.k, q, dp.m, stream); });
            step([&] { return launch_tc_wgrad(px, pg, dw4[ps], kws, d.n * dp.m, 2 * d.c, 2 * d.k, d.s, 8, q / dp.m, stream); });
        }
    } else {
        uint16_t* x2b = bump.take<uint16_t>(sizeof(uint16_t) * nx);
        uint16_t* g2b = bump.take<uint16_t>(sizeof(uint16_t) * ng);
        void* kws = bump.take<char>(tc_wgrad_workspace_bytes(d.n, 2 * d.c, 2 * d.k, d.s, 8, q));
        split_both(x2b, g2b);
        const uint16_t* xsrc[2] = {x2, x2b};
        const uint16_t* gsrc[2] = {g2, g2b};
        for (int ps = 0; ps < 2; ++ps)
            step([&] { return launch_tc_wgrad(xsrc[ps], gsrc[ps], dw4[ps], kws, d.n, 2 * d.c, 2 * d.k, d.s, 8, q, stream); });
    }
    step([&] { return launch_sum_split3(dw4[0], dw4[1], dw, d.k, d.c, d.s, stream); });
    return e;
}

size_t split_workspace(const c1d_desc& d, c1d_pass pass, int64_t q) {
    Bump dry{nullptr, 0, true};
    if (pass == C1D_PASS_BACKWARD_WEIGHT)
        split_wgrad_run(d, q, nullptr, nullptr, nullptr, dry, nullptr);
    else
        split_conv_any(d, pass, q, nullptr, nullptr, nullptr, dry, nullptr);
    return dry.used;
}

// Conv-shaped pass (forward or backward-data).
// glue (optional): layer glue fused into the tensor-core epilogue; only for glue_fusable() passes,
// and `out` may then be NULL.
// C1D_FLAG_PREPACKED_WEIGHTS: BF16 on the native dilation-8 tensor-core path, one accumulator
// chain (the carry plan), and a plan whose image tc_conv_prepack_bytes describes
bool prepack_ok(const c1d_desc& d, c1d_pass pass, int64_t q, c1d_algo algo) {
    if (pass == C1D_PASS_BACKWARD_WEIGHT || algo != C1D_ALGO_TCGEN05 || !is_bf16(d)) return false;
    if (dil_plan(d, q).kind != DilPlan::kNative) return false;
    const ConvGeom g = pitched(pass == C1D_PASS_FORWARD ? fwd_geom(d, q) : bwd_geom(d, q));
    return tc_conv_prepack_bytes(g) > 0;
}

c1d_status conv_pass(const c1d_desc* desc, c1d_pass pass, const void* in, const float* w_kcs, float* out,
                     void* ws, size_t ws_bytes, cudaStream_t stream, const LayerGlue* glue = nullptr) {
    t_last_error.clear();
    int64_t q = 0;
    c1d_status st = validate(desc, &q);
    if (st != C1D_OK) return st;
    const ExactAccumScope exact_scope(exact_for(*desc));
    const c1d_desc& d = *desc;
    if (d.n == 0) return C1D_OK;
    if (!in || !w_kcs || (!out && !glue)) return fail(C1D_ERR_INVALID_ARGUMENT, "NULL tensor pointer");
    st = check_device();
    if (st != C1D_OK) return st;
    const c1d_algo algo = resolve(d, pass, q);
    if (static_cast<int>(algo) < 0) return fail(C1D_ERR_UNSUPPORTED, "requested algo cannot run this shape");
    const ConvGeom g = pass == C1D_PASS_FORWARD ? fwd_geom(d, q) : bwd_geom(d, q);
    const bool prepacked = (d.flags & C1D_FLAG_PREPACKED_WEIGHTS) != 0;
    if (prepacked && !prepack_ok(d, pass, q, algo))
        return fail(C1D_ERR_UNSUPPORTED, "C1D_FLAG_PREPACKED_WEIGHTS: this pass's plan packs its own weights");
    Bump bump{};
    st = acquire_workspace(ws, ws_bytes, workspace_for(d, pass, q, algo), &bump, stream);
    if (st != C1D_OK) return st;
    if (algo == C1D_ALGO_BF16X3) {
        // FP32 via split BF16 operands (split.cu), composed with the dilation plans
        const cudaError_t e = split_conv_any(d, pass, q, in, w_kcs, out, bump, stream);
        if (bump.overflow) return workspace_overflow();
        if (e != cudaSuccess) return cuda_fail(e, "tc_conv (bf16x3)");
        return C1D_OK;
    }
    const bool bf16 = is_bf16(d);
    const DilPlan dp = dil_plan(d, q);
    // (o, i, s) weights for the FFMA / relayout paths; the native tensor-core path packs straight
    // from the caller's KCS weights (one launch fewer)
    float* wg = bump.take<float>(sizeof(float) * static_cast<size_t>(d.k * d.c * d.s));
    cudaError_t e = cudaSuccess;
    const bool use_xr = algo == C1D_ALGO_TCGEN05 && dp.kind == DilPlan::kPhases && xr_ok(g);
    if (bump.overflow) return workspace_overflow();
    if (algo == C1D_ALGO_DIRECT || (dp.kind != DilPlan::kNative && !use_xr))
        e = launch_prep_weights(w_kcs, wg, d.k, d.c, d.s,
                                pass == C1D_PASS_FORWARD ? kWeightsForward : kWeightsBackwardData, bf16, stream);
    if (e != cudaSuccess) return cuda_fail(e, "prep_weights");
    if (algo == C1D_ALGO_DIRECT) {
        if (bump.overflow) return workspace_overflow();
        e = launch_direct_conv(in, d.in_dtype, bf16 && d.in_dtype == C1D_DTYPE_F32, wg, out, g, stream);
        if (e != cudaSuccess) return cuda_fail(e, "direct_conv");
        return C1D_OK;
    }
    if (dp.kind == DilPlan::kPlanes) {
        // d = 8m: de-interleave the input into chunk planes, run dilation 8, re-interleave
        const ConvGeom gp = plane_geom(g, dp);
        uint16_t* pin = bump.take<uint16_t>(sizeof(uint16_t) * static_cast<size_t>(g.n * g.in_ch * g.in_w));
        float* pout = bump.take<float>(sizeof(float) * static_cast<size_t>(gp.n * gp.out_ch * gp.out_w));
        if (bump.overflow) return workspace_overflow();
        e = launch_to_planes(in, d.in_dtype, pin, g.n, g.in_ch, g.in_w, dp.m, stream);
        if (e != cudaSuccess) return cuda_fail(e, "to_planes");
        void* kws = bump.take<char>(tc_conv_workspace_bytes(gp));
        if (bump.overflow) return workspace_overflow();
        e = launch_tc_conv(pin, wg, pout, gp, kws, stream);
        if (e == cudaSuccess) e = launch_from_planes(pout, out, g.n, g.out_ch, g.out_w, dp.m, stream);
        if (e != cudaSuccess) return cuda_fail(e, "tc_conv (planes)");
        return C1D_OK;
    }
    if (use_xr && xr_inline_ok(g)) {
        // d < 8: expanded rows built in shared memory from the natural bf16 rows
        const ConvGeom gi = xr_inline_geom(g);
        const uint16_t* in_b = static_cast<const uint16_t*>(in);
        if (gi.in_stride) {
            uint16_t* tmp = bump.take<uint16_t>(sizeof(uint16_t) * static_cast<size_t>(g.n * g.in_ch * gi.in_stride));
            if (bump.overflow) return workspace_overflow();
            e = launch_pad_rows(in, d.in_dtype, tmp, g.n * g.in_ch, g.in_w, gi.in_stride, stream);
            if (e != cudaSuccess) return cuda_fail(e, "pad_rows");
            in_b = tmp;
        } else if (d.in_dtype == C1D_DTYPE_F32) {
            const int64_t count = g.n * g.in_ch * g.in_w;
            uint16_t* tmp = bump.take<uint16_t>(sizeof(uint16_t) * static_cast<size_t>(count));
            if (bump.overflow) return workspace_overflow();
            e = launch_round_bf16(static_cast<const float*>(in), tmp, count, stream);
            if (e != cudaSuccess) return cuda_fail(e, "round_bf16");
            in_b = tmp;
        }
        const int64_t mc = glue ? 0 : xr_main_ch(gi);
        void* kws = bump.take<char>(tc_conv_workspace_bytes(gi, mc));
        if (bump.overflow) return workspace_overflow();
        e = launch_tc_conv(in_b, w_kcs, out, gi, kws, stream, mc, pass == C1D_PASS_BACKWARD_DATA, glue);
        if (e != cudaSuccess) return cuda_fail(e, "tc_conv (expanded rows, inline)");
        return C1D_OK;
    }
    if (use_xr) {
        // d < 8: expanded rows (E = 8-element rows at every d-column start), 16 taps per MMA
        const ConvGeom gx = xr_geom(g);
        uint16_t* ex = bump.take<uint16_t>(sizeof(uint16_t) * 8 * static_cast<size_t>(gx.n * gx.in_ch * gx.xr_rows));
        if (bump.overflow) return workspace_overflow();
        e = launch_expand_rows(in, d.in_dtype, ex, g.n * g.in_ch, g.in_w, g.dil, g.in_off, gx.xr_rows, stream);
        if (e != cudaSuccess) return cuda_fail(e, "expand_rows");
        const int64_t mc = glue ? 0 : xr_main_ch(gx);
        void* kws = bump.take<char>(tc_conv_workspace_bytes(gx, mc));
        if (bump.overflow) return workspace_overflow();
        e = launch_tc_conv(ex, w_kcs, out, gx, kws, stream, mc, pass == C1D_PASS_BACKWARD_DATA, glue);
        if (e != cudaSuccess) return cuda_fail(e, "tc_conv (expanded rows)");
        return C1D_OK;
    }
    if (dp.kind == DilPlan::kPhases) {
        // d < 8: shifted phase copies (P*I channels) against phase-split weights, dilation 8
        const ConvGeom gp = phase_geom(g, dp);
        const PhaseCopy pc = phase_copy(g);
        uint16_t* cp = bump.take<uint16_t>(sizeof(uint16_t) * static_cast<size_t>(gp.n * gp.in_ch * gp.in_w));
        float* wph = bump.take<float>(sizeof(float) * static_cast<size_t>(gp.out_ch * gp.in_ch * dp.sp));
        if (bump.overflow) return workspace_overflow();
        e = launch_shift_copies(in, d.in_dtype, cp, g.n, g.in_ch, g.in_w, dp.p, pc.base, d.d, gp.in_w, stream);
        if (e == cudaSuccess) e = launch_phase_split_weights(wg, wph, g.out_ch, g.in_ch, d.s, dp.m, dp.p, stream);
        if (e != cudaSuccess) return cuda_fail(e, "phase copies");
        void* kws = bump.take<char>(tc_conv_workspace_bytes(gp));
        if (bump.overflow) return workspace_overflow();
        e = launch_tc_conv(cp, wph, out, gp, kws, stream, 0, false, glue);
        if (e != cudaSuccess) return cuda_fail(e, "tc_conv (phases)");
        return C1D_OK;
    }
    const ConvGeom gq = pitched(g);
    const uint16_t* in_b = static_cast<const uint16_t*>(in);
    if (gq.in_stride) {  // unaligned row pitch: zero-padded bf16 copy (rounds FP32 storage too)
        uint16_t* tmp = bump.take<uint16_t>(sizeof(uint16_t) * static_cast<size_t>(g.n * g.in_ch * gq.in_stride));
        if (bump.overflow) return workspace_overflow();
        e = launch_pad_rows(in, d.in_dtype, tmp, g.n * g.in_ch, g.in_w, gq.in_stride, stream);
        if (e != cudaSuccess) return cuda_fail(e, "pad_rows");
        in_b = tmp;
    } else if (d.in_dtype == C1D_DTYPE_F32) {
        const int64_t count = g.n * g.in_ch * g.in_w;
        uint16_t* tmp = bump.take<uint16_t>(sizeof(uint16_t) * static_cast<size_t>(count));
        if (bump.overflow) return workspace_overflow();
        e = launch_round_bf16(static_cast<const float*>(in), tmp, count, stream);
        if (e != cudaSuccess) return cuda_fail(e, "round_bf16");
        in_b = tmp;
    }
    // glued calls keep the carry mode; otherwise native_choice (carry / direct / two chains)
    const ChainPlan cp = glue || prepacked ? ChainPlan{gq, 0} : native_choice(gq);
    void* kws = bump.take<char>(tc_conv_workspace_bytes(cp.g, cp.main_ch));
    if (bump.overflow) return workspace_overflow();
    e = launch_tc_conv(in_b, w_kcs, out, cp.g, kws, stream, cp.main_ch, pass == C1D_PASS_BACKWARD_DATA, glue,
                       prepacked ? reinterpret_cast<const uint16_t*>(w_kcs) : nullptr);
    if (e != cudaSuccess) return cuda_fail(e, "tc_conv");
    return C1D_OK;
}


// ---- layer-glued conv passes (c1d_forward_glued / c1d_backward_data_glued) ----
// Fused: the glue runs in the tcgen05 conv epilogue (native dilation 8 and the phase rewrite, whose
// output layout is the caller's). Otherwise the conv writes an FP32 scratch tensor and one
// layer.cu glue pass follows.
bool glue_fusable(const c1d_desc& d, c1d_pass pass, int64_t q, c1d_algo algo) {
    if (algo != C1D_ALGO_TCGEN05) return false;
    const DilPlan dp = dil_plan(d, q);
    // the glue epilogue handles filter blocks of up to 64 (the expanded-row mode takes KP = 128 above)
    // native d = 8 keeps the carry mode under glue (any filter count, groups of <= 64); the expanded-row
    // mode's glue needs filter blocks of <= 64 (it takes 128-wide blocks above)
    return dp.kind == DilPlan::kNative || (dp.kind == DilPlan::kPhases && (pass == C1D_PASS_FORWARD ? d.k : d.c) <= 64);
}
struct GlueSizes {
    bool fused;
    size_t conv, scratch, part;
    size_t total() const { return conv + scratch + part; }
};
GlueSizes glue_sizes(const c1d_desc& d, c1d_pass pass, int64_t q, c1d_algo algo, int64_t glue_q) {
    GlueSizes r{};
    r.fused = glue_fusable(d, pass, q, algo);
    r.conv = align_up(workspace_for(d, pass, q, algo));
    const bool fwd = pass == C1D_PASS_FORWARD;
    const int64_t out_elems = fwd ? d.n * d.k * q : d.n * d.c * d.w_in;
    r.scratch = r.fused ? 0 : align_up(sizeof(float) * static_cast<size_t>(out_elems));
    if (!fwd) {
        const int64_t parts = r.fused ? d.c * num_sms() : d.n * d.c * layer_bias_blocks(glue_q);
        r.part = align_up(sizeof(float) * static_cast<size_t>(parts));
    }
    return r;
}

}  // namespace
}  // namespace c1d

using namespace c1d;

extern "C" {

int c1d_api_version(void) { return C1D_API_VERSION; }

const char* c1d_strerror(c1d_status status) {
    switch (status) {
        case C1D_OK: return "ok";
        case C1D_ERR_SHAPE_MISMATCH: return "shape mismatch";
        case C1D_ERR_ODD_DIMS: return "bf16 conv needs even dimensions";
        case C1D_ERR_TOO_NARROW: return "input narrower than the receptive field";
        case C1D_ERR_INVALID_ARGUMENT: return "invalid argument";
        case C1D_ERR_WORKSPACE: return "workspace too small";
        case C1D_ERR_UNSUPPORTED: return "unsupported shape for the requested algorithm";
        case C1D_ERR_CUDA: return "CUDA error";
        case C1D_ERR_NO_DEVICE: return "no sm_100 device";
    }
    return "unknown status";
}

const char* c1d_last_error_message(void) { return t_last_error.c_str(); }

c1d_status c1d_output_width(const c1d_desc* desc, int64_t* q_out) {
    t_last_error.clear();
    if (!q_out) return fail(C1D_ERR_INVALID_ARGUMENT, "q_out is NULL");
    return validate(desc, q_out);
}

int64_t c1d_conv_flops(const c1d_desc* desc) {
    int64_t q = 0;
    if (validate(desc, &q) != C1D_OK) return -1;
    return int64_t{2} * desc->n * desc->k * desc->c * desc->s * q;
}

c1d_status c1d_selected_algo(const c1d_desc* desc, c1d_pass pass, c1d_algo* algo) {
    t_last_error.clear();
    int64_t q = 0;
    c1d_status st = validate(desc, &q);
    if (st != C1D_OK) return st;
    const c1d_algo a = resolve(*desc, pass, q);
    if (static_cast<int>(a) < 0) return fail(C1D_ERR_UNSUPPORTED, "requested algo cannot run this shape");
    if (algo) *algo = a;
    return C1D_OK;
}

c1d_status c1d_workspace_size(const c1d_desc* desc, c1d_pass pass, size_t* bytes) {
    t_last_error.clear();
    int64_t q = 0;
    c1d_status st = validate(desc, &q);
    if (st != C1D_OK) return st;
    const ExactAccumScope exact_scope(exact_for(*desc));
    const c1d_algo a = resolve(*desc, pass, q);
    if (static_cast<int>(a) < 0) return fail(C1D_ERR_UNSUPPORTED, "requested algo cannot run this shape");
    if (bytes) *bytes = workspace_for(*desc, pass, q, a);
    return C1D_OK;
}

c1d_status c1d_packed_weights_size(const c1d_desc* desc, c1d_pass pass, size_t* bytes) {
    t_last_error.clear();
    int64_t q = 0;
    c1d_status st = validate(desc, &q);
    if (st != C1D_OK) return st;
    const ExactAccumScope exact_scope(exact_for(*desc));
    const c1d_algo a = resolve(*desc, pass, q);
    if (static_cast<int>(a) < 0 || !prepack_ok(*desc, pass, q, a))
        return fail(C1D_ERR_UNSUPPORTED, "this pass's plan packs its own weights");
    if (bytes)
        *bytes = tc_conv_prepack_bytes(pitched(pass == C1D_PASS_FORWARD ? fwd_geom(*desc, q) : bwd_geom(*desc, q)));
    return C1D_OK;
}

c1d_status c1d_pack_weights(int count, const c1d_desc* descs, const int32_t* passes, const float* const* w,
                            void* const* images, c1d_stream_t stream) {
    t_last_error.clear();
    if (count < 0 || (count > 0 && (!descs || !passes || !w || !images)))
        return fail(C1D_ERR_INVALID_ARGUMENT, "bad c1d_pack_weights arguments");
    if (count == 0) return C1D_OK;
    c1d_status st = check_device();
    if (st != C1D_OK) return st;
    std::vector<ConvGeom> gs(static_cast<size_t>(count));
    std::vector<int> raw(static_cast<size_t>(count));
    for (int i = 0; i < count; ++i) {
        const c1d_pass pass = static_cast<c1d_pass>(passes[i]);
        int64_t q = 0;
        st = validate(&descs[i], &q);
        if (st != C1D_OK) return st;
        const ExactAccumScope exact_scope(exact_for(descs[i]));
        const c1d_algo a = resolve(descs[i], pass, q);
        if (static_cast<int>(a) < 0 || !prepack_ok(descs[i], pass, q, a) || !w[i] || !images[i])
            return fail(C1D_ERR_UNSUPPORTED, "c1d_pack_weights: job " + std::to_string(i) + " cannot take an image");
        gs[static_cast<size_t>(i)] = pitched(pass == C1D_PASS_FORWARD ? fwd_geom(descs[i], q) : bwd_geom(descs[i], q));
        raw[static_cast<size_t>(i)] = pass == C1D_PASS_BACKWARD_DATA ? 1 : 0;
    }
    const cudaError_t e = launch_pack_images_multi(count, gs.data(), w, raw.data(), images,
                                                   reinterpret_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? C1D_OK : cuda_fail(e, "pack_weights");
}

c1d_status c1d_forward(const c1d_desc* desc, const void* x, const float* w_kcs, float* y, void* workspace,
                       size_t workspace_bytes, c1d_stream_t stream) {
    return conv_pass(desc, C1D_PASS_FORWARD, x, w_kcs, y, workspace, workspace_bytes,
                     reinterpret_cast<cudaStream_t>(stream));
}

c1d_status c1d_backward_data(const c1d_desc* desc, const void* dy, const float* w_kcs, float* dx, void* workspace,
                             size_t workspace_bytes, c1d_stream_t stream) {
    return conv_pass(desc, C1D_PASS_BACKWARD_DATA, dy, w_kcs, dx, workspace, workspace_bytes,
                     reinterpret_cast<cudaStream_t>(stream));
}

c1d_status c1d_backward_weight(const c1d_desc* desc, const void* x, const void* dy, float* dw_kcs, void* workspace,
                               size_t workspace_bytes, c1d_stream_t stream_) {
    t_last_error.clear();
    cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
    int64_t q = 0;
    c1d_status st = validate(desc, &q);
    if (st != C1D_OK) return st;
    const c1d_desc& d = *desc;
    const ExactAccumScope exact_scope(exact_for(d));
    if (!dw_kcs) return fail(C1D_ERR_INVALID_ARGUMENT, "NULL dw pointer");
    st = check_device();
    if (st != C1D_OK) return st;
    if (d.n == 0) {
        cudaError_t e = cudaMemsetAsync(dw_kcs, 0, sizeof(float) * static_cast<size_t>(d.k * d.c * d.s), stream);
        return e == cudaSuccess ? C1D_OK : cuda_fail(e, "memset");
    }
    if (!x || !dy) return fail(C1D_ERR_INVALID_ARGUMENT, "NULL tensor pointer");
    const c1d_algo algo = resolve(d, C1D_PASS_BACKWARD_WEIGHT, q);
    if (static_cast<int>(algo) < 0) return fail(C1D_ERR_UNSUPPORTED, "requested algo cannot run this shape");
    Bump bump{};
    st = acquire_workspace(workspace, workspace_bytes, workspace_for(d, C1D_PASS_BACKWARD_WEIGHT, q, algo), &bump,
                           stream);
    if (st != C1D_OK) return st;
    const bool bf16 = is_bf16(d);
    cudaError_t e;
    if (algo == C1D_ALGO_BF16X3) {
        e = split_wgrad_run(d, q, x, dy, dw_kcs, bump, stream);
        if (bump.overflow) return workspace_overflow();
        if (e != cudaSuccess) return cuda_fail(e, "tc_wgrad (bf16x3)");
        return C1D_OK;
    }
    if (algo == C1D_ALGO_DIRECT) {
        float* part = bump.take<float>(direct_wgrad_workspace_bytes(d.n, d.c, d.k, d.s, d.d, q));
        if (bump.overflow) return workspace_overflow();
        e = launch_direct_wgrad(x, dy, d.in_dtype, bf16 && d.in_dtype == C1D_DTYPE_F32, dw_kcs, part, d.n, d.c, d.k,
                                d.s, d.d, q, stream);
        if (e != cudaSuccess) return cuda_fail(e, "direct_wgrad");
        return C1D_OK;
    }
    const DilPlan dpl = dil_plan(d, q);
    if (xt_wgrad_ok(d, wgrad_pad(d, q).q_pad)) {
        const WgradPad wpd = wgrad_pad(d, q);
        // the octet-stream plan needs no aligned x pitch: dY is copied only when Q itself is
        // unaligned or stored as FP32
        const uint16_t* g16 = static_cast<const uint16_t*>(dy);
        if (q % 8 != 0 || d.in_dtype == C1D_DTYPE_F32) {
            uint16_t* tg = bump.take<uint16_t>(sizeof(uint16_t) * static_cast<size_t>(d.n * d.k * wpd.q_pad));
            if (bump.overflow) return workspace_overflow();
            e = q % 8 != 0 ? launch_pad_rows(dy, d.in_dtype, tg, d.n * d.k, q, wpd.q_pad, stream)
                           : launch_round_bf16(static_cast<const float*>(dy), tg, d.n * d.k * q, stream);
            if (e != cudaSuccess) return cuda_fail(e, "dy copy");
            g16 = tg;
        }
        // channel-octet streams of x (FP32 rounded on the way)
        const int64_t rows = xt_rows(d, wpd.q_pad);
        uint16_t* xt = bump.take<uint16_t>(sizeof(uint16_t) * 8 * static_cast<size_t>(d.n * ((d.c + 7) / 8) * rows));
        if (bump.overflow) return workspace_overflow();
        e = launch_to_octets(x, d.in_dtype, xt, d.n, d.c, d.w_in, rows, stream);
        if (e != cudaSuccess) return cuda_fail(e, "to_octets");
        void* kws = bump.take<char>(tc_wgrad_xt_workspace_bytes(d.n, d.c, d.k, d.s, d.d, wpd.q_pad));
        if (bump.overflow) return workspace_overflow();
        e = launch_tc_wgrad_xt(xt, rows, g16, dw_kcs, kws, d.n, d.c, d.k, d.s, d.d, wpd.q_pad, stream);
        if (e != cudaSuccess) return cuda_fail(e, "tc_wgrad (octet streams)");
        return C1D_OK;
    }
    if (dpl.kind == DilPlan::kPlanes) {
        // d = 8m: both operands as chunk planes; the plane items sum into the same dW
        uint16_t* px = bump.take<uint16_t>(sizeof(uint16_t) * static_cast<size_t>(d.n * d.c * d.w_in));
        uint16_t* pdy = bump.take<uint16_t>(sizeof(uint16_t) * static_cast<size_t>(d.n * d.k * q));
        if (bump.overflow) return workspace_overflow();
        e = launch_to_planes(x, d.in_dtype, px, d.n, d.c, d.w_in, dpl.m, stream);
        if (e == cudaSuccess) e = launch_to_planes(dy, d.in_dtype, pdy, d.n, d.k, q, dpl.m, stream);
        if (e != cudaSuccess) return cuda_fail(e, "to_planes");
        void* kws = bump.take<char>(tc_wgrad_workspace_bytes(d.n * dpl.m, d.c, d.k, d.s, 8, q / dpl.m));
        if (bump.overflow) return workspace_overflow();
        e = launch_tc_wgrad(px, pdy, dw_kcs, kws, d.n * dpl.m, d.c, d.k, d.s, 8, q / dpl.m, stream);
        if (e != cudaSuccess) return cuda_fail(e, "tc_wgrad (planes)");
        return C1D_OK;
    }
    e = cudaSuccess;
    const WgradPad wpd = wgrad_pad(d, q);
    if (dpl.kind == DilPlan::kPhases && xr_wgrad_ok(d, wpd.q_pad)) {
        // d < 8: x as expanded rows (rounded to BF16 on the way), dY padded / rounded if needed
        const uint16_t* g16 = static_cast<const uint16_t*>(dy);
        if (wpd.pad || d.in_dtype == C1D_DTYPE_F32) {
            uint16_t* tg = bump.take<uint16_t>(sizeof(uint16_t) * static_cast<size_t>(d.n * d.k * wpd.q_pad));
            if (bump.overflow) return workspace_overflow();
            e = wpd.pad ? launch_pad_rows(dy, d.in_dtype, tg, d.n * d.k, q, wpd.q_pad, stream)
                        : launch_round_bf16(static_cast<const float*>(dy), tg, d.n * d.k * q, stream);
            if (e != cudaSuccess) return cuda_fail(e, "dy copy");
            g16 = tg;
        }
        if (xin_wgrad_preferred(d) && tc_wgrad_xin_supported(d.n, d.c, d.k, d.s, d.d, wpd.q_pad)) {
            // the loaders build the rows from natural bf16 x (8-element pitch; FP32 rounded once)
            const int64_t xw = round8(d.w_in);
            const uint16_t* x16 = static_cast<const uint16_t*>(x);
            if (xw != d.w_in || d.in_dtype == C1D_DTYPE_F32) {
                uint16_t* tx = bump.take<uint16_t>(sizeof(uint16_t) * static_cast<size_t>(d.n * d.c * xw));
                if (bump.overflow) return workspace_overflow();
                e = launch_pad_rows(x, d.in_dtype, tx, d.n * d.c, d.w_in, xw, stream);
                if (e != cudaSuccess) return cuda_fail(e, "pad_rows");
                x16 = tx;
            }
            void* kws = bump.take<char>(tc_wgrad_xin_workspace_bytes(d.n, d.c, d.k, d.s, d.d, wpd.q_pad));
            if (bump.overflow) return workspace_overflow();
            e = launch_tc_wgrad_xin(x16, xw, g16, dw_kcs, kws, d.n, d.c, d.k, d.s, d.d, wpd.q_pad, stream);
            if (e != cudaSuccess) return cuda_fail(e, "tc_wgrad (expanded rows, inline)");
            return C1D_OK;
        }
        const int64_t rows = xr_wgrad_rows(d, wpd.q_pad);
        uint16_t* ex = bump.take<uint16_t>(sizeof(uint16_t) * 8 * static_cast<size_t>(d.n * d.c * rows));
        if (bump.overflow) return workspace_overflow();
        e = launch_expand_rows(x, d.in_dtype, ex, d.n * d.c, d.w_in, d.d, 0, rows, stream);
        if (e != cudaSuccess) return cuda_fail(e, "expand_rows");
        void* kws = bump.take<char>(tc_wgrad_workspace_bytes(d.n, d.c, d.k, d.s, d.d, wpd.q_pad));
        if (bump.overflow) return workspace_overflow();
        e = launch_tc_wgrad(ex, g16, dw_kcs, kws, d.n, d.c, d.k, d.s, d.d, wpd.q_pad, stream, rows * 8);
        if (e != cudaSuccess) return cuda_fail(e, "tc_wgrad (expanded rows)");
        return C1D_OK;
    }
    const uint16_t* xb = static_cast<const uint16_t*>(x);
    const uint16_t* gb = static_cast<const uint16_t*>(dy);
    if (wpd.pad) {  // zero-padded bf16 copies with 8-element pitches (rounds FP32 storage too)
        uint16_t* tx = bump.take<uint16_t>(sizeof(uint16_t) * static_cast<size_t>(d.n * d.c * wpd.x_pitch));
        uint16_t* tg = bump.take<uint16_t>(sizeof(uint16_t) * static_cast<size_t>(d.n * d.k * wpd.q_pad));
        if (bump.overflow) return workspace_overflow();
        e = launch_pad_rows(x, d.in_dtype, tx, d.n * d.c, d.w_in, wpd.x_pitch, stream);
        if (e == cudaSuccess) e = launch_pad_rows(dy, d.in_dtype, tg, d.n * d.k, q, wpd.q_pad, stream);
        if (e != cudaSuccess) return cuda_fail(e, "pad_rows");
        xb = tx;
        gb = tg;
    } else if (d.in_dtype == C1D_DTYPE_F32) {
        uint16_t* tx = bump.take<uint16_t>(sizeof(uint16_t) * static_cast<size_t>(d.n * d.c * d.w_in));
        uint16_t* tg = bump.take<uint16_t>(sizeof(uint16_t) * static_cast<size_t>(d.n * d.k * q));
        if (bump.overflow) return workspace_overflow();
        e = launch_round_bf16(static_cast<const float*>(x), tx, d.n * d.c * d.w_in, stream);
        if (e == cudaSuccess) e = launch_round_bf16(static_cast<const float*>(dy), tg, d.n * d.k * q, stream);
        if (e != cudaSuccess) return cuda_fail(e, "round_bf16");
        xb = tx;
        gb = tg;
    }
    const DilPlan dp = dil_plan(d, q);
    if (dp.kind == DilPlan::kPhases) {
        // phase b (real taps b + m*t): x shifted by b*d columns (bf16 copy), dilation-8 gradient
        // over its taps, scattered back into dW
        const int64_t xp = phase_x_pitch(d, wpd, dp);
        uint16_t* xs = bump.take<uint16_t>(sizeof(uint16_t) * static_cast<size_t>(d.n * d.c * xp));
        float* dwb = bump.take<float>(sizeof(float) * static_cast<size_t>(d.k * dp.p * d.c * dp.sp));
        size_t kbytes = 0;
        for (int64_t b = 0; b < dp.p; ++b)
            kbytes = std::max(kbytes, tc_wgrad_workspace_bytes(d.n, d.c, d.k, ceil_div(d.s - b, dp.m), 8, wpd.q_pad));
        void* kws = bump.take<char>(kbytes);
        for (int64_t b = 0; b < dp.p && e == cudaSuccess; ++b) {
            const int64_t sb = ceil_div(d.s - b, dp.m);
            if (bump.overflow) return workspace_overflow();
            e = launch_shift_copies(x, d.in_dtype, xs, d.n, d.c, d.w_in, 1, b * d.d, 0, xp, stream);
            if (e == cudaSuccess) e = launch_tc_wgrad(xs, gb, dwb, kws, d.n, d.c, d.k, sb, 8, wpd.q_pad, stream, xp);
            if (e == cudaSuccess) e = launch_scatter_phase_wgrad(dwb, dw_kcs, d.k, d.c, d.s, dp.m, b, stream);
        }
        if (e != cudaSuccess) return cuda_fail(e, "tc_wgrad (phases)");
        return C1D_OK;
    }
    void* kws = bump.take<char>(tc_wgrad_workspace_bytes(d.n, d.c, d.k, d.s, 8, wpd.q_pad));
    if (bump.overflow) return workspace_overflow();
    e = launch_tc_wgrad(xb, gb, dw_kcs, kws, d.n, d.c, d.k, d.s, 8, wpd.q_pad, stream, wpd.pad ? wpd.x_pitch : 0);
    if (e != cudaSuccess) return cuda_fail(e, "tc_wgrad");
    return C1D_OK;
}

c1d_status c1d_round_bf16(const float* in, uint16_t* out, int64_t count, c1d_stream_t stream) {
    t_last_error.clear();
    if (count < 0 || (count > 0 && (!in || !out))) return fail(C1D_ERR_INVALID_ARGUMENT, "bad round_bf16 arguments");
    cudaError_t e = launch_round_bf16(in, out, count, reinterpret_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? C1D_OK : cuda_fail(e, "round_bf16");
}

size_t c1d_layer_backward_workspace(int64_t n, int64_t k, int64_t q) {
    if (n <= 0 || k <= 0 || q <= 0) return 0;
    return align_up(static_cast<size_t>(n * k * layer_bias_blocks(q)) * sizeof(float));
}

c1d_status c1d_layer_forward_epilogue(float* pre, const float* bias, const float* skip, int64_t n, int64_t k, int64_t q,
                                      int relu, int store_pre, float* act, uint16_t* act_bf16, int64_t pad,
                                      c1d_stream_t stream) {
    t_last_error.clear();
    if (n < 0 || k <= 0 || q < 0 || pad < 0 || !pre || n * k > 65535)
        return fail(C1D_ERR_INVALID_ARGUMENT, "bad layer_forward_epilogue arguments");
    if (c1d_status st = check_device(); st != C1D_OK) return st;
    cudaError_t e = launch_layer_fwd_epilogue(pre, bias, skip, n, k, q, relu, store_pre, act, act_bf16, pad, nullptr,
                                              reinterpret_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? C1D_OK : cuda_fail(e, "layer_forward_epilogue");
}

c1d_status c1d_layer_backward_prologue(const float* gin, int64_t gin_w, int64_t gin_off, const float* gadd,
                                       const float* pre, const float* pre_bias, int64_t n, int64_t k, int64_t q,
                                       int relu, float* gsum,
                                       float* grad_pre, uint16_t* grad_pre_bf16, float* bias_grad, void* workspace,
                                       size_t workspace_bytes, c1d_stream_t stream) {
    t_last_error.clear();
    if (n < 0 || k <= 0 || q < 0 || !gin || gin_off < 0 || gin_w < gin_off + q || (relu && !pre) || n * k > 65535)
        return fail(C1D_ERR_INVALID_ARGUMENT, "bad layer_backward_prologue arguments");
    if (c1d_status st = check_device(); st != C1D_OK) return st;
    Bump ws{};
    const size_t need = bias_grad ? c1d_layer_backward_workspace(n, k, q) : 0;
    if (c1d_status st = acquire_workspace(workspace, workspace_bytes, need, &ws, reinterpret_cast<cudaStream_t>(stream));
        st != C1D_OK)
        return st;
    float* part =
        bias_grad ? ws.take<float>(static_cast<size_t>(n * k * layer_bias_blocks(q)) * sizeof(float)) : nullptr;
    cudaError_t e = launch_layer_bwd_prologue(gin, gin_w, gin_off, gadd, pre, pre_bias, nullptr, n, k, q, relu, gsum, grad_pre,
                                              grad_pre_bf16, bias_grad, part, reinterpret_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? C1D_OK : cuda_fail(e, "layer_backward_prologue");
}

c1d_status c1d_glued_workspace_size(const c1d_desc* desc, c1d_pass pass, int64_t glue_q, size_t* bytes, int* fused) {
    t_last_error.clear();
    int64_t q = 0;
    c1d_status st = validate(desc, &q);
    if (st != C1D_OK) return st;
    const ExactAccumScope exact_scope(exact_for(*desc));
    if (pass == C1D_PASS_BACKWARD_WEIGHT) return fail(C1D_ERR_INVALID_ARGUMENT, "glue applies to conv-shaped passes");
    const c1d_algo a = resolve(*desc, pass, q);
    if (static_cast<int>(a) < 0) return fail(C1D_ERR_UNSUPPORTED, "requested algo cannot run this shape");
    const GlueSizes gs = glue_sizes(*desc, pass, q, a, glue_q > 0 ? glue_q : 1);
    if (bytes) *bytes = gs.total();
    if (fused) *fused = gs.fused ? 1 : 0;
    return C1D_OK;
}

c1d_status c1d_forward_glued(const c1d_desc* desc, const void* x, const float* w_kcs, const c1d_fwd_glue* glue,
                             void* workspace, size_t workspace_bytes, c1d_stream_t stream_) {
    t_last_error.clear();
    cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
    int64_t q = 0;
    c1d_status st = validate(desc, &q);
    if (st != C1D_OK) return st;
    const c1d_desc& d = *desc;
    const ExactAccumScope exact_scope(exact_for(d));
    if (!glue || glue->act_pad < 0) return fail(C1D_ERR_INVALID_ARGUMENT, "bad forward glue");
    if (d.n == 0) return C1D_OK;
    if (d.n * d.k > 65535) return fail(C1D_ERR_UNSUPPORTED, "glue supports N*K <= 65535 rows");
    if (c1d_status s2 = check_device(); s2 != C1D_OK) return s2;
    const c1d_algo algo = resolve(d, C1D_PASS_FORWARD, q);
    if (static_cast<int>(algo) < 0) return fail(C1D_ERR_UNSUPPORTED, "requested algo cannot run this shape");
    const GlueSizes gs = glue_sizes(d, C1D_PASS_FORWARD, q, algo, q);
    Bump bump{};
    st = acquire_workspace(workspace, workspace_bytes, gs.total(), &bump, stream);
    if (st != C1D_OK) return st;
    char* conv_ws = bump.take<char>(gs.conv);
    if (gs.fused) {
        LayerGlue lg;
        lg.mode = 1;
        lg.relu = glue->relu;
        lg.bias = glue->bias;
        lg.skip = glue->skip;
        lg.pre = glue->pre;
        lg.act = glue->act;
        lg.act_bf16 = glue->act_bf16;
        lg.act_pitch = q + 2 * glue->act_pad;
        lg.act_off = glue->act_pad;
        lg.mask_out = glue->mask;
        return conv_pass(desc, C1D_PASS_FORWARD, x, w_kcs, nullptr, conv_ws, gs.conv, stream, &lg);
    }
    float* pre = glue->pre ? glue->pre : bump.take<float>(gs.scratch);
    st = conv_pass(desc, C1D_PASS_FORWARD, x, w_kcs, pre, conv_ws, gs.conv, stream);
    if (st != C1D_OK) return st;
    const cudaError_t e = launch_layer_fwd_epilogue(pre, glue->bias, glue->skip, d.n, d.k, q, glue->relu,
                                                    glue->pre != nullptr, glue->act, glue->act_bf16, glue->act_pad,
                                                    glue->mask, stream);
    return e == cudaSuccess ? C1D_OK : cuda_fail(e, "layer_forward_epilogue");
}

c1d_status c1d_backward_data_glued(const c1d_desc* desc, const void* dy, const float* w_kcs, const c1d_bwd_glue* glue,
                                   void* workspace, size_t workspace_bytes, c1d_stream_t stream_) {
    t_last_error.clear();
    cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
    int64_t q = 0;
    c1d_status st = validate(desc, &q);
    if (st != C1D_OK) return st;
    const c1d_desc& d = *desc;
    const ExactAccumScope exact_scope(exact_for(d));
    if (!glue || glue->off < 0 || glue->q <= 0 || glue->off + glue->q > d.w_in)
        return fail(C1D_ERR_INVALID_ARGUMENT, "bad backward glue window");
    if (d.n == 0) {
        if (glue->bias_grad) {
            const cudaError_t e = cudaMemsetAsync(glue->bias_grad, 0, sizeof(float) * static_cast<size_t>(d.c), stream);
            if (e != cudaSuccess) return cuda_fail(e, "memset");
        }
        return C1D_OK;
    }
    if (d.n * d.c > 65535) return fail(C1D_ERR_UNSUPPORTED, "glue supports N*C <= 65535 rows");
    if (c1d_status s2 = check_device(); s2 != C1D_OK) return s2;
    const c1d_algo algo = resolve(d, C1D_PASS_BACKWARD_DATA, q);
    if (static_cast<int>(algo) < 0) return fail(C1D_ERR_UNSUPPORTED, "requested algo cannot run this shape");
    const GlueSizes gs = glue_sizes(d, C1D_PASS_BACKWARD_DATA, q, algo, glue->q);
    Bump bump{};
    st = acquire_workspace(workspace, workspace_bytes, gs.total(), &bump, stream);
    if (st != C1D_OK) return st;
    char* conv_ws = bump.take<char>(gs.conv);
    float* part = bump.take<float>(gs.part);
    if (gs.fused) {
        LayerGlue lg;
        lg.mode = 2;
        lg.g_off = glue->off;
        lg.g_q = glue->q;
        lg.gadd = glue->gadd;
        lg.mask_in = glue->mask;
        lg.gsum = glue->gsum;
        lg.gp = glue->grad_pre;
        lg.gp_bf16 = glue->grad_pre_bf16;
        lg.part = glue->bias_grad ? part : nullptr;
        lg.bias_grad = glue->bias_grad;
        return conv_pass(desc, C1D_PASS_BACKWARD_DATA, dy, w_kcs, nullptr, conv_ws, gs.conv, stream, &lg);
    }
    if (d.s == 1 && d.precision == C1D_PRECISION_FP32 && d.in_dtype == C1D_DTYPE_F32 && algo == C1D_ALGO_DIRECT &&
        d.k <= 16 && glue->off == 0 && glue->q == q && d.w_in == q) {
        // 1-tap FP32 backward-data (the network's heads): the glue pass computes the few-filter
        // sum itself, in the pointwise kernel's order, instead of reading an FP32 dx scratch tensor
        const cudaError_t e = launch_layer_bwd_prologue(nullptr, q, 0, glue->gadd, nullptr, nullptr, glue->mask, d.n, d.c,
                                                        q, glue->mask != nullptr, glue->gsum, glue->grad_pre,
                                                        glue->grad_pre_bf16, glue->bias_grad, part, stream,
                                                        static_cast<const float*>(dy), w_kcs, static_cast<int>(d.k));
        return e == cudaSuccess ? C1D_OK : cuda_fail(e, "layer_backward_prologue (1-tap)");
    }
    float* dx = bump.take<float>(gs.scratch);
    st = conv_pass(desc, C1D_PASS_BACKWARD_DATA, dy, w_kcs, dx, conv_ws, gs.conv, stream);
    if (st != C1D_OK) return st;
    const cudaError_t e = launch_layer_bwd_prologue(dx, d.w_in, glue->off, glue->gadd, nullptr, nullptr, glue->mask, d.n,
                                                    d.c, glue->q, glue->mask != nullptr, glue->gsum, glue->grad_pre,
                                                    glue->grad_pre_bf16, glue->bias_grad, part, stream);
    return e == cudaSuccess ? C1D_OK : cuda_fail(e, "layer_backward_prologue");
}

c1d_status c1d_release_workspace(c1d_stream_t stream) {
    t_last_error.clear();
    const cudaError_t e = release_internal_workspace(reinterpret_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? C1D_OK : cuda_fail(e, "release_workspace");
}

uint64_t c1d_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

}  // extern "C"
