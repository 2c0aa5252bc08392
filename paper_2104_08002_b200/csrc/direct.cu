// direct.cu — CUDA-core (FFMA) direct convolution kernels: the any-shape path.
//
// These cover every shape the reference accepts (any C, K, S, d, width; FP32 or BF16 precision)
// and serve as the FP32 path. The tensor-core kernels (tc_conv.cu, tc_wgrad.cu) take over for
// the shapes they support. Accumulation is FP32 with FMA; results are deterministic (fixed
// iteration order, no atomics) and match the reference's naive oracle within its 1e-5 bound.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "sm100.cuh"

namespace c1d {

// shared-memory row pitch for the sliding-window kernels: an odd number of 16-B chunks, so 16-B
// reads of 8 consecutive rows hit 8 distinct chunk slots (one wavefront)
__host__ __device__ inline int slide_pitch(int words) { return (words + 3) / 8 * 8 + 4; }

// ------------------------------------------------------------------------------- weights
__global__ void prep_weights_kernel(const float* __restrict__ w, float* __restrict__ out, int64_t K, int64_t C,
                                    int64_t S, int mode, int round) {
    const int64_t total = K * C * S;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        float v;
        if (mode == kWeightsForward) {
            v = w[e];  // (k, c, s) -> (k, c, s)
        } else {
            // out index e = (c, k, s') holds w(k, c, S-1-s')
            const int64_t sp = e % S;
            const int64_t kk = (e / S) % K;
            const int64_t cc = e / (S * K);
            v = w[(kk * C + cc) * S + (S - 1 - sp)];
        }
        out[e] = round ? round_to_bf16(v) : v;
    }
}

cudaError_t launch_prep_weights(const float* w_kcs, float* out, int64_t K, int64_t C, int64_t S, int mode,
                                bool round, cudaStream_t stream) {
    const int64_t total = K * C * S;
    const int threads = 256;
    const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(total, threads), 4096));
    prep_weights_kernel<<<blocks, threads, 0, stream>>>(w_kcs, out, K, C, S, mode, round ? 1 : 0);
    note_launch();
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------- forward-shaped
// Block tile: 16 output channels x 256 output columns, 256 threads, each thread a 4x4
// register tile (4 channels x 4 columns strided by 64). Input channels are staged through
// shared memory in chunks of 8 together with the halo (taps-1)*dil.
namespace {
constexpr int kTO = 16;    // output channels per block
constexpr int kTX = 256;   // output columns per block
constexpr int kCC = 8;     // input channels per smem chunk
}  // namespace

template <typename TIn>
__global__ void __launch_bounds__(256) direct_conv_kernel(const TIn* __restrict__ in, const float* __restrict__ wg,
                                                          float* __restrict__ out, ConvGeom g, int round_in) {
    extern __shared__ float smem[];
    const int64_t halo = (g.taps - 1) * g.dil;
    const int64_t span = kTX + halo;
    float* xs = smem;                   // [kCC][span]
    float* ws = smem + kCC * span;      // [kTO][kCC][taps]
    const int tid = threadIdx.x;
    const int og = tid / 64;            // 4 output-channel groups of 4
    const int xg = tid % 64;            // column lane
    const int64_t x0 = static_cast<int64_t>(blockIdx.x) * kTX;
    const int64_t o0 = static_cast<int64_t>(blockIdx.y) * kTO;
    const int64_t n = blockIdx.z;
    const TIn* in_n = in + n * g.in_ch * g.in_w;

    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;

    for (int64_t c0 = 0; c0 < g.in_ch; c0 += kCC) {
        __syncthreads();
        for (int64_t e = tid; e < kCC * span; e += blockDim.x) {
            const int64_t cc = e / span, xx = e % span;
            const int64_t c = c0 + cc;
            const int64_t src = x0 + xx + g.in_off;
            float v = 0.0f;
            if (c < g.in_ch && src >= 0 && src < g.in_w) v = load_as_float(in_n, c * g.in_w + src, round_in != 0);
            xs[e] = v;
        }
        for (int64_t e = tid; e < kTO * kCC * g.taps; e += blockDim.x) {
            const int64_t s = e % g.taps;
            const int64_t cc = (e / g.taps) % kCC;
            const int64_t oo = e / (g.taps * kCC);
            const int64_t o = o0 + oo, c = c0 + cc;
            ws[e] = (o < g.out_ch && c < g.in_ch) ? wg[(o * g.in_ch + c) * g.taps + s] : 0.0f;
        }
        __syncthreads();
        const int cmax = static_cast<int>(std::min<int64_t>(kCC, g.in_ch - c0));
        for (int cc = 0; cc < cmax; ++cc) {
            const float* xr = xs + cc * span + xg;
            const float* wr = ws + (og * 4) * kCC * g.taps + cc * g.taps;
            for (int s = 0; s < g.taps; ++s) {
                float wv[4], xv[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) wv[i] = wr[i * kCC * g.taps + s];
#pragma unroll
                for (int j = 0; j < 4; ++j) xv[j] = xr[j * 64 + s * g.dil];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(wv[i], xv[j], acc[i][j]);
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t o = o0 + og * 4 + i;
        if (o >= g.out_ch) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t x = x0 + xg + 64 * j;
            if (x < g.out_w) out[(n * g.out_ch + o) * g.out_w + x] = acc[i][j];
        }
    }
}

// ------------------------------------------------------------------------------- sliding window
// Forward-shaped FFMA convolution, dilation-phase register windows. Block: persistent, walking
// 16-output x 512-column tiles; 256 threads, thread (q4, cg) owns outputs {q4, q4+4, q4+8, q4+12}
// and 8 columns of one dilation phase, x0 + ph + d*(i0 + i) (i < 8), so tap s of its columns is
// the 8-wide window at phase index i0 + s: the staged input rows are dilation-phase-major (column
// ph + d*i at [ph][i]) and the windows are 16-B vector reads, as are the 4 outputs' weights of a
// tap ([c][s][quad][4]). Input channels stream in chunks of 8 (one warp per row) through a double
// buffer (cp.async for FP32 input). Taps run in groups of SG (S itself for S <= 3, else 4 with the
// tap count padded by zero weights). The output tile is assembled in shared memory and written
// with coalesced stores.
namespace {
constexpr int kCT = 8;     // input channels per staged chunk
constexpr int kCO = 16;    // outputs per block
constexpr int kCQ = 512;   // columns per block
}  // namespace
__host__ __device__ inline int cslide_nbp(int d) { return ((kCQ + d - 1) / d + 7) / 8; }  // 8-blocks per phase
__host__ __device__ inline int cslide_lx(int d, int sp) { return (8 * cslide_nbp(d) + sp - 1 + 3 + 3) / 4 * 4; }
__host__ __device__ inline int cslide_sg(int s) { return s <= 3 ? s : 4; }
__host__ __device__ inline int cslide_sp(int s) { return (s + cslide_sg(s) - 1) / cslide_sg(s) * cslide_sg(s); }
static size_t cslide_smem(int d, int s) {
    const int sp = cslide_sp(s);
    const size_t buf = static_cast<size_t>(kCT * slide_pitch(d * cslide_lx(d, sp)) + kCT * sp * kCO);
    return sizeof(float) * (2 * buf + kCO * kCQ);  // double buffer + output tile
}
static bool cslide_ok(const ConvGeom& g) {
    return g.dil <= 64 && !g.xr_rows && !g.xr_inline && g.in_stride == 0 &&
           g.n * ceil_div(g.out_w, kCQ) * ceil_div(g.out_ch, kCO) < (int64_t{1} << 31) &&
           cslide_smem(static_cast<int>(g.dil), static_cast<int>(g.taps)) <= 200 * 1024;
}

// Copies columns [0, count) of one row into shared memory at dst with cp.async (zeros outside
// [lo, hi)): 16-B copies when src is 16-B aligned, else 8-B, else 4-B. count % 4 == 0.
// (`safe` is any valid address, named by the zero-byte copies.)
template <int V>
__device__ __forceinline__ void copy_row_v(uint32_t dst, const float* src, const float* safe, int lo, int hi,
                                           int count, int lane) {
    for (int col = V * lane; col < count; col += 32 * V) {
        const bool full = col >= lo && col + V <= hi;
        if (full || col + V <= lo || col >= hi) {
            if (V == 4) sm100::cp_async16_zfill(dst + 4u * col, full ? src + col : safe, full);
            else if (V == 2) sm100::cp_async8_zfill(dst + 4u * col, full ? src + col : safe, full);
            else sm100::cp_async4_zfill(dst + 4u * col, full ? src + col : safe, full);
        } else {
#pragma unroll
            for (int e = 0; e < V; ++e) {
                const bool ok = col + e >= lo && col + e < hi;
                sm100::cp_async4_zfill(dst + 4u * (col + e), ok ? src + col + e : safe, ok);
            }
        }
    }
}
__device__ __forceinline__ void copy_row(uint32_t dst, const float* src, const float* safe, int lo, int hi,
                                         int count, int lane) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(src);
    if ((a & 15) == 0) copy_row_v<4>(dst, src, safe, lo, hi, count, lane);
    else if ((a & 7) == 0) copy_row_v<2>(dst, src, safe, lo, hi, count, lane);
    else copy_row_v<1>(dst, src, safe, lo, hi, count, lane);
}

template <typename TIn, int SG, int NB>
__global__ void __launch_bounds__(256, 2) conv_slide_kernel(const TIn* __restrict__ in, const float* __restrict__ wg,
                                                            float* __restrict__ out, ConvGeom g, int round_in) {
    extern __shared__ float4 smem4[];
    float* smem = reinterpret_cast<float*>(smem4);
    const int d = static_cast<int>(g.dil), S = static_cast<int>(g.taps);
    const int sp = cslide_sp(S), nbp = cslide_nbp(d), lx = cslide_lx(d, sp);
    const int span = d * lx;  // staged input columns per row
    const int xpitch = slide_pitch(span);
    const int wwords = kCT * sp * kCO;
    const int buf_words = kCT * xpitch + wwords;
    float* tile = smem + 2 * buf_words;  // [16][512] output tile
    const bool async = sizeof(TIn) == 4 && round_in == 0;
    const int tid = threadIdx.x, lane = tid % 32, warp = tid / 32;
    const int q4 = tid % 4, cg = tid / 4;  // outputs {q4, q4+4, q4+8, q4+12}, column group 0..63
    const int64_t C = g.in_ch;
    const int nchunks = static_cast<int>(ceil_div(C, kCT));
    const int64_t tiles_x = ceil_div(g.out_w, kCQ), tiles_o = ceil_div(g.out_ch, kCO);
    const int tiles = static_cast<int>(g.n * tiles_x * tiles_o);
    const uint32_t sbase = sm100::smem_u32(smem);
    const int step_q = 32 / d, step_r = 32 % d;
    const int xstep = 4 * (step_r * lx + step_q), xwrap = 4 * (1 - d * lx);
    // this block's work: tiles blockIdx.x, +gridDim.x, ... (output tiles fastest, so the blocks
    // running together share their input columns in L2), each as nchunks channel chunks
    // (32-bit tile decode once per tile: tiles < 2^31 by the launch check)
    struct Tile { int64_t n, x0, o0; };
    const int ntx = static_cast<int>(tiles_x), nto = static_cast<int>(tiles_o);
    auto tile_of = [&](int t) {
        const int ot = t % nto, rest = t / nto;
        return Tile{rest / ntx, static_cast<int64_t>(rest % ntx) * kCQ, static_cast<int64_t>(ot) * kCO};
    };

    auto stage = [&](const Tile& tl, int chunk, int b) {
        const int64_t pos0 = tl.x0 + g.in_off;  // input position of staged column 0
        const int lo = static_cast<int>(std::max<int64_t>(0, std::min<int64_t>(span, -pos0)));
        const int64_t c = static_cast<int64_t>(chunk) * kCT + warp;  // one row per warp (kCT == 8 warps)
        const bool cok = c < C;
        const int hi = cok ? static_cast<int>(std::max<int64_t>(0, std::min<int64_t>(span, g.in_w - pos0))) : 0;
        const uint32_t xb = sbase + 4u * static_cast<uint32_t>(b * buf_words + warp * xpitch);
        const TIn* row = in + (tl.n * C + (cok ? c : 0)) * g.in_w;
        if (async && d == 1) {
            copy_row(xb, reinterpret_cast<const float*>(row) + pos0, reinterpret_cast<const float*>(row), lo, hi, span,
                     lane);
        } else {
            float* xr = smem + b * buf_words + warp * xpitch;
            int ph = lane % d, i = lane / d;
            uint32_t sd = xb + 4u * static_cast<uint32_t>(ph * lx + i);
            for (int col = lane; col < span; col += 32) {
                const bool ok = col >= lo && col < hi;
                if (async) {
                    sm100::cp_async4_zfill(sd, reinterpret_cast<const float*>(row) + (ok ? pos0 + col : 0), ok);
                } else {
                    xr[ph * lx + i] = ok ? load_as_float(row, pos0 + col, round_in != 0) : 0.0f;
                }
                ph += step_r;
                i += step_q;
                sd += xstep;
                if (ph >= d) ph -= d, ++i, sd += xwrap;
            }
        }
        // weights [cc][s][quad][j] = wg[(o0 + quad + 4j, c0 + cc, s)], zero past the edges
        const uint32_t wb = sbase + 4u * static_cast<uint32_t>(b * buf_words + kCT * xpitch);
        const int64_t c0 = static_cast<int64_t>(chunk) * kCT;
        for (int e = tid; e < wwords; e += 256) {
            const int j = e & 3, qq = (e >> 2) & 3, rest = e >> 4;
            const int s = rest % sp, cc = rest / sp;
            const int64_t o = tl.o0 + qq + 4 * j, ci = c0 + cc;
            const bool ok = o < g.out_ch && ci < C && s < S;
            sm100::cp_async4_zfill(wb + 4u * e, wg + (ok ? (o * C + ci) * S + s : 0), ok);
        }
        sm100::cp_async_commit();
    };

    float acc[NB][4][8];
#pragma unroll
    for (int a = 0; a < NB; ++a)
#pragma unroll
        for (int h = 0; h < 4; ++h)
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[a][h][i] = 0.0f;
    // items = (tile, chunk) pairs in order; `cur` is being computed, `nxt` is being staged
    int t_cur = blockIdx.x, chunk = 0;
    Tile cur = tile_of(t_cur);
    if (t_cur < tiles) stage(cur, 0, 0);
    for (int b = 0; t_cur < tiles; b ^= 1) {
        int t_nxt = t_cur, chunk_nxt = chunk + 1;
        if (chunk_nxt == nchunks) chunk_nxt = 0, t_nxt += gridDim.x;
        const Tile nxt = t_nxt != t_cur && t_nxt < tiles ? tile_of(t_nxt) : cur;
        if (t_nxt < tiles) {
            stage(nxt, chunk_nxt, b ^ 1);  // buffer b^1 was released by the barrier that ended the last item
            sm100::cp_async_wait_group<1>();
        } else {
            sm100::cp_async_wait_group<0>();
        }
        __syncthreads();
        const float* xs = smem + b * buf_words;
        const float* ws = xs + kCT * xpitch;
        const int cmax = static_cast<int>(std::min<int64_t>(kCT, C - static_cast<int64_t>(chunk) * kCT));
#pragma unroll
        for (int a = 0; a < NB; ++a) {
            const int blk = cg + 64 * a;
            if (blk >= d * nbp) break;
            const int ph = blk / nbp, i0 = 8 * (blk % nbp);
            for (int cc = 0; cc < cmax; ++cc) {
                const float4* xq = reinterpret_cast<const float4*>(xs + cc * xpitch + ph * lx + i0);
                const float4* wq = reinterpret_cast<const float4*>(ws + cc * sp * kCO) + q4;
                for (int s0 = 0; s0 < sp; s0 += SG) {
                    constexpr int NW = (8 + SG - 1 + 3) / 4;
                    float win[4 * NW];
#pragma unroll
                    for (int v = 0; v < NW; ++v) *reinterpret_cast<float4*>(&win[4 * v]) = xq[s0 / 4 + v];
#pragma unroll
                    for (int jj = 0; jj < SG; ++jj) {
                        const float4 w = wq[(s0 + jj) * 4];
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            acc[a][0][i] = fmaf(w.x, win[i + jj], acc[a][0][i]);
                            acc[a][1][i] = fmaf(w.y, win[i + jj], acc[a][1][i]);
                            acc[a][2][i] = fmaf(w.z, win[i + jj], acc[a][2][i]);
                            acc[a][3][i] = fmaf(w.w, win[i + jj], acc[a][3][i]);
                        }
                    }
                }
            }
        }
        if (chunk == nchunks - 1) {
            // tile done: assemble the 16 x 512 outputs in shared memory, then coalesced stores
#pragma unroll
            for (int a = 0; a < NB; ++a) {
                const int blk = cg + 64 * a;
                if (blk >= d * nbp) break;
                const int ph = blk / nbp, i0 = 8 * (blk % nbp);
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int col = ph + d * (i0 + i);
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                        if (col < kCQ) tile[(q4 + 4 * h) * kCQ + col] = acc[a][h][i];
                        acc[a][h][i] = 0.0f;
                    }
                }
            }
            __syncthreads();
            const int cols = static_cast<int>(std::min<int64_t>(kCQ, g.out_w - cur.x0));
            for (int r = warp; r < kCO; r += 8) {
                const int64_t o = cur.o0 + r;
                if (o >= g.out_ch) break;
                float* dst = out + (cur.n * g.out_ch + o) * g.out_w + cur.x0;
                for (int col = lane; col < cols; col += 32) dst[col] = tile[r * kCQ + col];
            }
        }
        __syncthreads();
        t_cur = t_nxt, chunk = chunk_nxt, cur = nxt;
    }
}

template <typename TIn, int SG>
static cudaError_t launch_cslide_sg(const TIn* in, const float* wg, float* out, const ConvGeom& g, int round_in,
                                    cudaStream_t stream) {
    const int d = static_cast<int>(g.dil);
    const size_t smem = cslide_smem(d, static_cast<int>(g.taps));
    // persistent blocks: up to two per SM (the register bound), each walking its tiles' channel
    // chunks through one double-buffered pipeline
    const int64_t tiles = g.n * ceil_div(g.out_w, kCQ) * ceil_div(g.out_ch, kCO);
    const int per_sm = static_cast<int>(std::max<size_t>(1, std::min<size_t>(2, (227 * 1024) / (smem + 1024))));
    const dim3 grid(static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(tiles, per_sm * num_sms()))));
    const bool two = d * cslide_nbp(d) > 64;
    cudaError_t e;
    if (two) {
        e = cudaFuncSetAttribute(conv_slide_kernel<TIn, SG, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        conv_slide_kernel<TIn, SG, 2><<<grid, 256, smem, stream>>>(in, wg, out, g, round_in);
    } else {
        e = cudaFuncSetAttribute(conv_slide_kernel<TIn, SG, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        conv_slide_kernel<TIn, SG, 1><<<grid, 256, smem, stream>>>(in, wg, out, g, round_in);
    }
    note_launch();
    return cudaGetLastError();
}

template <typename TIn>
static cudaError_t launch_cslide(const TIn* in, const float* wg, float* out, const ConvGeom& g, int round_in,
                                 cudaStream_t stream) {
    switch (cslide_sg(static_cast<int>(g.taps))) {
        case 1: return launch_cslide_sg<TIn, 1>(in, wg, out, g, round_in, stream);
        case 2: return launch_cslide_sg<TIn, 2>(in, wg, out, g, round_in, stream);
        case 3: return launch_cslide_sg<TIn, 3>(in, wg, out, g, round_in, stream);
        default: return launch_cslide_sg<TIn, 4>(in, wg, out, g, round_in, stream);
    }
}

// ------------------------------------------------------------------------------- 1-tap (pointwise)
// S = 1: out[n][o][x] = sum_i W[o][i] in[n][i][x + off]. Memory-bound; each thread owns 4
// consecutive columns for all (<= OMAX) outputs, the input is read exactly once. (The config-5
// network's two heads run as one 2-filter 1-tap conv.)
constexpr int kPwThreads = 256;
constexpr int kPwCols = 4 * kPwThreads;

template <typename TIn, int OMAX>
__global__ void __launch_bounds__(kPwThreads) pointwise_conv_kernel(const TIn* __restrict__ in,
                                                                    const float* __restrict__ wg,
                                                                    float* __restrict__ out, ConvGeom g,
                                                                    int round_in, int vec) {
    const int64_t n = blockIdx.y;
    const int64_t x0 = static_cast<int64_t>(blockIdx.x) * kPwCols + threadIdx.x * 4;
    if (x0 >= g.out_w) return;
    const int O = static_cast<int>(g.out_ch);
    float acc[OMAX][4];
#pragma unroll
    for (int o = 0; o < OMAX; ++o)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[o][j] = 0.0f;
    const int cnt = static_cast<int>(g.out_w - x0 < 4 ? g.out_w - x0 : 4);
    for (int64_t i = 0; i < g.in_ch; ++i) {
        const int64_t base = (n * g.in_ch + i) * g.in_w + x0 + g.in_off;
        float v[4];
        if (vec && cnt == 4) {
            load4_as_float(in, base, round_in != 0, v);
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) v[j] = j < cnt ? load_as_float(in, base + j, round_in != 0) : 0.0f;
        }
#pragma unroll
        for (int o = 0; o < OMAX; ++o) {
            const float w = o < O ? __ldg(wg + static_cast<int64_t>(o) * g.in_ch + i) : 0.0f;
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[o][j] = fmaf(w, v[j], acc[o][j]);
        }
    }
#pragma unroll
    for (int o = 0; o < OMAX; ++o) {
        if (o >= O) continue;
        float* dst = out + (n * g.out_ch + o) * g.out_w + x0;
        if (vec && cnt == 4) {
            *reinterpret_cast<float4*>(dst) = make_float4(acc[o][0], acc[o][1], acc[o][2], acc[o][3]);
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (j < cnt) dst[j] = acc[o][j];
        }
    }
}

template <typename TIn>
static cudaError_t launch_pointwise(const TIn* in, const float* wg, float* out, const ConvGeom& g, int round_in,
                                    cudaStream_t stream) {
    const dim3 grid(static_cast<unsigned>(ceil_div(g.out_w, kPwCols)), static_cast<unsigned>(g.n));
    // vector loads / stores: every row start 16-B (float) / 8-B (bf16) aligned
    const uintptr_t al = sizeof(TIn) == 4 ? 15u : 7u;
    const int vec = g.in_w % 4 == 0 && g.in_off % 4 == 0 && g.out_w % 4 == 0 && (reinterpret_cast<uintptr_t>(in) & al) == 0 &&
                    (reinterpret_cast<uintptr_t>(out) & 15u) == 0;
    if (g.out_ch <= 1)
        pointwise_conv_kernel<TIn, 1><<<grid, kPwThreads, 0, stream>>>(in, wg, out, g, round_in, vec);
    else if (g.out_ch <= 2)
        pointwise_conv_kernel<TIn, 2><<<grid, kPwThreads, 0, stream>>>(in, wg, out, g, round_in, vec);
    else if (g.out_ch <= 4)
        pointwise_conv_kernel<TIn, 4><<<grid, kPwThreads, 0, stream>>>(in, wg, out, g, round_in, vec);
    else if (g.out_ch <= 8)
        pointwise_conv_kernel<TIn, 8><<<grid, kPwThreads, 0, stream>>>(in, wg, out, g, round_in, vec);
    else
        pointwise_conv_kernel<TIn, 16><<<grid, kPwThreads, 0, stream>>>(in, wg, out, g, round_in, vec);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_direct_conv(const void* in, int in_dtype, bool round_in, const float* wg, float* out,
                               const ConvGeom& g, cudaStream_t stream) {
    if (g.taps == 1 && g.out_ch <= 16 && g.n <= 65535) {
        if (in_dtype == 0) return launch_pointwise(static_cast<const float*>(in), wg, out, g, round_in ? 1 : 0, stream);
        return launch_pointwise(static_cast<const uint16_t*>(in), wg, out, g, 0, stream);
    }
    if (cslide_ok(g)) {
        if (in_dtype == 0) return launch_cslide(static_cast<const float*>(in), wg, out, g, round_in ? 1 : 0, stream);
        return launch_cslide(static_cast<const uint16_t*>(in), wg, out, g, 0, stream);
    }
    const int64_t span = kTX + (g.taps - 1) * g.dil;
    const size_t smem = sizeof(float) * static_cast<size_t>(kCC * span + kTO * kCC * g.taps);
    if (smem > 227 * 1024) return cudaErrorInvalidValue;
    dim3 grid(static_cast<unsigned>(ceil_div(g.out_w, kTX)), static_cast<unsigned>(ceil_div(g.out_ch, kTO)),
              static_cast<unsigned>(g.n));
    if (g.n > 65535 || grid.y > 65535) return cudaErrorInvalidValue;
    cudaError_t e;
    if (in_dtype == 0) {
        e = cudaFuncSetAttribute(direct_conv_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        direct_conv_kernel<float><<<grid, 256, smem, stream>>>(static_cast<const float*>(in), wg, out, g,
                                                                round_in ? 1 : 0);
    } else {
        e = cudaFuncSetAttribute(direct_conv_kernel<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        direct_conv_kernel<uint16_t><<<grid, 256, smem, stream>>>(static_cast<const uint16_t*>(in), wg, out, g, 0);
    }
    note_launch();
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------- backward weight
// Register-tiled FFMA gradient. Block (kt, ct, split) owns a 32-filter x 32-channel tile and a
// contiguous range of (item, 128-column chunk) units of its split; taps are processed in groups
// of 8 (outer loop) so every thread keeps 4 filters x 8 taps of one channel in registers. Per
// column a thread reads 4 dY values (warp-broadcast) and 8 X values (one row per lane) from shared
// memory for 32 FMAs. Partials land in workspace[split][k][c][s] and a second kernel sums the
// splits in ascending order (deterministic; the reference reduces per-item partials in ascending
// item order, conv.cpp:308-314).
namespace {
constexpr int kWK = 32;     // filters per block tile
constexpr int kWC = 32;     // channels per block tile
constexpr int kWQ = 128;    // columns per unit
constexpr int kWG = 8;      // taps per group
}  // namespace

static int64_t wgrad_splits(int64_t n, int64_t c, int64_t k, int64_t q) {
    const int64_t tiles = ceil_div(k, kWK) * ceil_div(c, kWC);
    const int64_t units = n * ceil_div(q, kWQ);
    const int64_t want = std::max<int64_t>(1, (4 * num_sms() + tiles - 1) / tiles);
    return std::max<int64_t>(1, std::min<int64_t>(want, units));
}

static bool pointwise_wgrad_ok(int64_t n, int64_t c, int64_t k, int64_t s);

// the sliding-window kernel (below) whenever its shared memory fits: the X window of one 256-column
// chunk plus the (S-1)*d reach of all taps
namespace {
constexpr int kSWT = 16;     // filters / channels per block tile
constexpr int kSWQ = 256;    // columns per unit
constexpr int kSWG = 10;     // most taps per group (registers)
}  // namespace
static size_t slide_smem(int d, int sg);
static bool slide_wgrad_ok(int64_t n, int64_t s, int64_t d, int64_t q) {
    return d <= 256 && n * ceil_div(q, 256) < (int64_t{1} << 31) &&
           slide_smem(static_cast<int>(d), static_cast<int>(std::min<int64_t>(s, kSWG))) <= 200 * 1024;
}
static int64_t slide_wgrad_splits(int64_t n, int64_t c, int64_t k, int64_t s, int64_t d, int64_t q) {
    const int64_t tiles = ceil_div(k, 16) * ceil_div(c, 16);
    const int64_t units = n * ceil_div(q, 256);
    // one full wave: resident blocks per SM by the register bound of the widest tap group (<= 4 taps:
    // 3, else 2) and the shared-memory bound (227 KB, 1 KB reserved per block); at least 3 units per
    // block so the copy of the next unit overlaps the current one
    const int64_t widest = ceil_div(s, ceil_div(s, kSWG));
    const int64_t by_smem = (227 * 1024) / (static_cast<int64_t>(slide_smem(static_cast<int>(d), static_cast<int>(widest))) + 1024);
    const int64_t per_sm = std::max<int64_t>(1, std::min<int64_t>(widest <= 4 ? 3 : 2, by_smem));
    const int64_t want = std::max<int64_t>(1, per_sm * num_sms() / tiles);
    return std::max<int64_t>(1, std::min<int64_t>(want, units / 3));
}

size_t direct_wgrad_workspace_bytes(int64_t n, int64_t c, int64_t k, int64_t s, int64_t d, int64_t q) {
    if (pointwise_wgrad_ok(n, c, k, s)) return sizeof(float) * static_cast<size_t>(n * ceil_div(q, 1024) * k * c);
    if (k * c * s <= 16) return sizeof(float) * static_cast<size_t>(592 * k * c * s);
    return sizeof(float) * static_cast<size_t>(std::max(wgrad_splits(n, c, k, q), slide_wgrad_splits(n, c, k, s, d, q)) *
                                               k * c * s);
}

template <typename TIn>
__global__ void __launch_bounds__(256) direct_wgrad_kernel(const TIn* __restrict__ x, const TIn* __restrict__ dy,
                                                           float* __restrict__ part, int64_t N, int64_t C, int64_t K,
                                                           int64_t S, int64_t D, int64_t Q, int64_t splits,
                                                           int tg, int xpitch, int round_in) {
    extern __shared__ float smem[];
    float* gs = smem;                    // [kWK][kWQ]        dY chunk
    float* xs = smem + kWK * kWQ;        // [kWC][xpitch]     X window of one tap group
    const int tid = threadIdx.x;
    const int cl = tid % kWC, kg = tid / kWC;  // channel lane, filter quad (0..7)
    const int64_t k0 = static_cast<int64_t>(blockIdx.x) * kWK, c0 = static_cast<int64_t>(blockIdx.y) * kWC;
    const int64_t split = blockIdx.z;
    const int64_t chunks_per_item = ceil_div(Q, kWQ);
    const int64_t units = N * chunks_per_item;
    const int64_t u_begin = units * split / splits, u_end = units * (split + 1) / splits;
    const int64_t W = Q + (S - 1) * D;
    const int64_t span = kWQ + (tg - 1) * D;  // X columns one tap group reads per chunk
    for (int64_t s0 = 0; s0 < S; s0 += tg) {
        float acc[4][kWG];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < kWG; ++j) acc[i][j] = 0.0f;
        for (int64_t u = u_begin; u < u_end; ++u) {
            const int64_t n = u / chunks_per_item;
            const int64_t q0 = (u % chunks_per_item) * kWQ;
            __syncthreads();
            // dY chunk: row kk = e / kWQ (kWQ is a power of two: shifts, no 64-bit division)
            for (int e = tid; e < kWK * kWQ; e += 256) {
                const int kk = e / kWQ, xx = e % kWQ;
                const int64_t k = k0 + kk, pos = q0 + xx;
                gs[e] = (k < K && pos < Q) ? load_as_float(dy, (n * K + k) * Q + pos, round_in != 0) : 0.0f;
            }
            const int64_t xbase = q0 + s0 * D;
            for (int cc = tid / 32; cc < kWC; cc += 8) {  // one warp per channel row, coalesced
                const int64_t c = c0 + cc;
                const TIn* row = x + (n * C + c) * W;
                for (int xx = tid % 32; xx < span; xx += 32) {
                    const int64_t pos = xbase + xx;
                    xs[cc * xpitch + xx] = (c < C && pos < W) ? load_as_float(row, pos, round_in != 0) : 0.0f;
                }
            }
            __syncthreads();
            const float* xr = xs + cl * xpitch;
            const float* gr = gs + (kg * 4) * kWQ;
            for (int xx = 0; xx < kWQ; ++xx) {
                float gv[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) gv[i] = gr[i * kWQ + xx];
#pragma unroll
                for (int j = 0; j < kWG; ++j) {
                    if (j >= tg) break;
                    const float xv = xr[xx + j * D];
#pragma unroll
                    for (int i = 0; i < 4; ++i) acc[i][j] = fmaf(gv[i], xv, acc[i][j]);
                }
            }
        }
        const int64_t c = c0 + cl;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t k = k0 + kg * 4 + i;
            if (k >= K || c >= C) continue;
            float* dst = part + ((split * K + k) * C + c) * S;
#pragma unroll
            for (int j = 0; j < kWG; ++j)
                if (j < tg && s0 + j < S) dst[s0 + j] = acc[i][j];
        }
    }
}

// Sliding-window FFMA gradient (round 2; replaces direct_wgrad_kernel above, whose 32 x 32 tiles
// left 3/4 of the lanes idle at C = K = 16 and re-staged the whole chunk per 8-tap group: 792 us at
// C = K = 16, S = 9, d = 1). Block (k-tile of 16, c-tile of 16, split) with thread (kk, cc) owning
// ONE (filter, channel) pair and up to 16 taps in registers. Per 8 columns of one dilation phase a
// thread reads 8 dY values and 8 + sg - 1 X values (the window slides: X[c][x + s*d] for
// consecutive phase columns shares sg - 1 values) for 8 * sg FMAs. Units are (item, 256-column
// chunk), split contiguously over the grid; partials part[split][k][c][s], summed in ascending
// split order by reduce_splits_kernel (deterministic).
// per-phase lengths (multiples of 4 floats, room for the 8-column read-ahead) and row pitches (an odd
// number of 16-B chunks: 16-B reads of 8 consecutive rows hit 8 distinct chunk slots, one wavefront)
__host__ __device__ inline int slide_lg(int d) { return ((kSWQ + d - 1) / d + 8 + 3) / 4 * 4; }
__host__ __device__ inline int slide_lx(int d, int sg) { return ((kSWQ + d - 1) / d + 8 + sg - 1 + 3 + 3) / 4 * 4; }

// Copies `count` columns of one row (the first `lim` from src, zeros after) into shared memory at
// dst with cp.async: 16-B copies when src is 16-B aligned, else 8-B when 8-B aligned, else 4-B.
// count is a multiple of 4. One warp per row.
template <int V>
__device__ __forceinline__ void slide_copy_row_v(uint32_t dst, const float* src, int lim, int count, int lane) {
    for (int col = V * lane; col < count; col += 32 * V) {
        const bool full = col + V <= lim;
        if (full || col >= lim) {
            if (V == 4) sm100::cp_async16_zfill(dst + 4u * col, full ? src + col : src, full);
            else if (V == 2) sm100::cp_async8_zfill(dst + 4u * col, full ? src + col : src, full);
            else sm100::cp_async4_zfill(dst + 4u * col, full ? src + col : src, full);
        } else {
#pragma unroll
            for (int e = 0; e < V; ++e)
                sm100::cp_async4_zfill(dst + 4u * (col + e), src + (col + e < lim ? col + e : 0), col + e < lim);
        }
    }
}
__device__ __forceinline__ void slide_copy_row(uint32_t dst, const float* src, int lim, int count, int lane) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(src);
    if ((a & 15) == 0) slide_copy_row_v<4>(dst, src, lim, count, lane);
    else if ((a & 7) == 0) slide_copy_row_v<2>(dst, src, lim, count, lane);
    else slide_copy_row_v<1>(dst, src, lim, count, lane);
}

// One launch per tap group [s0, s0 + SG) (SG taps in registers, a compile-time count). The chunk is
// staged dilation-phase-major (column ph + d*i at [ph][i]) so a phase's columns are contiguous and
// the inner loop reads 16-B vectors. FP32 input streams in through double-buffered cp.async copies
// (the next unit lands while this one is computed); BF16 or rounded input is staged through
// registers. Partial sums are written split-minor: part[(k*C + c)*S + s][split].
template <typename TIn, int SG>
__global__ void __launch_bounds__(256, SG <= 4 ? 3 : 2) wgrad_slide_kernel(const TIn* __restrict__ x, const TIn* __restrict__ dy,
                                                          float* __restrict__ part, int64_t N, int64_t C, int64_t K,
                                                          int64_t S, int64_t D, int64_t Q, int64_t splits, int lx,
                                                          int round_in, int64_t s0) {
    extern __shared__ float4 smem4[];
    float* smem = reinterpret_cast<float*>(smem4);
    const int d = static_cast<int>(D);
    const int lg = slide_lg(d);           // per-phase dY length (multiple of 4)
    const int gpitch = slide_pitch(d * lg), xpitch = slide_pitch(d * lx);
    const int buf_words = kSWT * (gpitch + xpitch);  // one buffer: [16][gpitch] dY, then [16][xpitch] X
    const bool async = sizeof(TIn) == 4 && round_in == 0;
    const int tid = threadIdx.x, lane = tid % 32;
    const int64_t k0 = static_cast<int64_t>(blockIdx.x) * kSWT, c0 = static_cast<int64_t>(blockIdx.y) * kSWT;
    const int64_t split = blockIdx.z;
    const int64_t chunks_per_item = ceil_div(Q, kSWQ);
    const int64_t units = N * chunks_per_item;
    const int64_t u_begin = units * split / splits, u_end = units * (split + 1) / splits;
    const int64_t W = Q + (S - 1) * D;
    const int span = d * lx;  // staged X columns (the window plus the read-ahead, phase-padded)
    const int step_q = 32 / d, step_r = 32 % d;
    const int ph_l = lane % d, i_l = lane / d;  // this lane's first column (lane = ph + d*i)

    // stage unit u into buffer b: one warp per row (coalesced global reads); the shared-memory slot
    // of column col = ph + d*i is stepped through (phase, index) without divisions
    const uint32_t sbase = sm100::smem_u32(smem);
    const int gstep = 4 * (step_r * lg + step_q), xstep = 4 * (step_r * lx + step_q);  // bytes per 32 columns
    const int gwrap = 4 * (1 - d * lg), xwrap = 4 * (1 - d * lx);                      // phase wrap-around
    auto stage = [&](int64_t u, int b) {
        // (32-bit: units < 2^31 by slide_wgrad_ok)
        const int64_t n = static_cast<int>(u) / static_cast<int>(chunks_per_item);
        const int64_t q0 = static_cast<int64_t>(static_cast<int>(u) % static_cast<int>(chunks_per_item)) * kSWQ;
        const uint32_t gsb = sbase + 4u * static_cast<uint32_t>(b * buf_words);
        const uint32_t xsb = gsb + 4u * static_cast<uint32_t>(kSWT * gpitch);
        for (int r = tid / 32; r < kSWT; r += 8) {
            const int64_t k = k0 + r, c = c0 + r;
            const bool kok = k < K, cok = c < C;
            const TIn* grow = dy + (n * K + (kok ? k : 0)) * Q + q0;
            const TIn* xrow = x + (n * C + (cok ? c : 0)) * W + q0 + s0 * D;
            const int glim = kok ? static_cast<int>(std::min<int64_t>(kSWQ, Q - q0)) : 0;
            const int xlim = cok ? static_cast<int>(std::min<int64_t>(span, W - q0 - s0 * D)) : 0;
            if (async && d == 1) {  // phase-major = plain order: widest copies the row alignment allows
                slide_copy_row(gsb + 4u * static_cast<uint32_t>(r * gpitch), reinterpret_cast<const float*>(grow),
                               glim, lg, lane);
                slide_copy_row(xsb + 4u * static_cast<uint32_t>(r * xpitch), reinterpret_cast<const float*>(xrow),
                               xlim, span, lane);
                continue;
            }
            uint32_t sd = gsb + 4u * static_cast<uint32_t>(r * gpitch + ph_l * lg + i_l);
            float* grs = smem + b * buf_words + r * gpitch;
            int ph = ph_l, i = i_l;
            for (int col = lane; col < d * lg; col += 32) {
                if (async) {
                    sm100::cp_async4_zfill(sd, grow + (col < glim ? col : 0), col < glim);
                } else {
                    grs[ph * lg + i] = col < glim ? load_as_float(grow, col, round_in != 0) : 0.0f;
                }
                ph += step_r;
                i += step_q;
                sd += gstep;
                if (ph >= d) ph -= d, ++i, sd += gwrap;
            }
            sd = xsb + 4u * static_cast<uint32_t>(r * xpitch + ph_l * lx + i_l);
            float* xrs = smem + b * buf_words + kSWT * gpitch + r * xpitch;
            ph = ph_l, i = i_l;
            for (int col = lane; col < span; col += 32) {
                if (async) {
                    sm100::cp_async4_zfill(sd, xrow + (col < xlim ? col : 0), col < xlim);
                } else {
                    xrs[ph * lx + i] = col < xlim ? load_as_float(xrow, col, round_in != 0) : 0.0f;
                }
                ph += step_r;
                i += step_q;
                sd += xstep;
                if (ph >= d) ph -= d, ++i, sd += xwrap;
            }
        }
        if (async) sm100::cp_async_commit();
    };

    // register tile: filters {kp, kp+8} x channels {cp, cp+8} x SG taps; the four warp pairs (qtr)
    // take every fourth 8-column block of the unit and are summed in a fixed order at the end
    const int qtr = tid / 64, kp = (tid % 64) / 8, cp = tid % 8;
    float acc[2][2][SG];
#pragma unroll
    for (int f = 0; f < 2; ++f)
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int j = 0; j < SG; ++j) acc[f][h][j] = 0.0f;
    if (u_begin < u_end) stage(u_begin, 0);
    int b = 0;
    for (int64_t u = u_begin; u < u_end; ++u, b ^= 1) {
        if (u + 1 < u_end) {
            stage(u + 1, b ^ 1);  // buffer b^1 was released by the barrier that ended unit u-1
            if (async) sm100::cp_async_wait_group<1>();
        } else if (async) {
            sm100::cp_async_wait_group<0>();
        }
        __syncthreads();
        const float* gb = smem + b * buf_words;
        const float* xb = gb + kSWT * gpitch;
        // phase by phase, 8 columns at a time: column ph + d*i; tap s of it is X column ph + d*(i + s)
        int blk0 = 0;  // 8-column blocks before this phase
        for (int ph = 0; ph < d; ++ph) {
            const int cols = ph < kSWQ ? (kSWQ - 1 - ph) / d + 1 : 0;
            const int nb = (cols + 7) / 8;
            const float4* g0 = reinterpret_cast<const float4*>(gb + kp * gpitch + ph * lg);
            const float4* g1 = reinterpret_cast<const float4*>(gb + (kp + 8) * gpitch + ph * lg);
            const float4* x0 = reinterpret_cast<const float4*>(xb + cp * xpitch + ph * lx);
            const float4* x1 = reinterpret_cast<const float4*>(xb + (cp + 8) * xpitch + ph * lx);
            for (int t = (qtr - blk0) & 3; t < nb; t += 4) {
                constexpr int NW = (8 + SG - 1 + 3) / 4;
                float ga[8], gc[8], wa[4 * NW], wc[4 * NW];
                *reinterpret_cast<float4*>(&ga[0]) = g0[2 * t];
                *reinterpret_cast<float4*>(&ga[4]) = g0[2 * t + 1];
                *reinterpret_cast<float4*>(&gc[0]) = g1[2 * t];
                *reinterpret_cast<float4*>(&gc[4]) = g1[2 * t + 1];
#pragma unroll
                for (int v = 0; v < NW; ++v) {
                    *reinterpret_cast<float4*>(&wa[4 * v]) = x0[2 * t + v];
                    *reinterpret_cast<float4*>(&wc[4 * v]) = x1[2 * t + v];
                }
#pragma unroll
                for (int j = 0; j < 8; ++j)
#pragma unroll
                    for (int s = 0; s < SG; ++s) {
                        acc[0][0][s] = fmaf(ga[j], wa[j + s], acc[0][0][s]);
                        acc[0][1][s] = fmaf(ga[j], wc[j + s], acc[0][1][s]);
                        acc[1][0][s] = fmaf(gc[j], wa[j + s], acc[1][0][s]);
                        acc[1][1][s] = fmaf(gc[j], wc[j + s], acc[1][1][s]);
                    }
            }
            blk0 += nb;
        }
        __syncthreads();
    }
    // fixed-order sum of the four quarters through shared memory (all copies have landed)
    float* red = smem;  // [16 filters][16 channels][SG]
    for (int q = 0; q < 4; ++q) {
        if (qtr == q) {
#pragma unroll
            for (int f = 0; f < 2; ++f)
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int j = 0; j < SG; ++j) {
                        float* r = red + ((kp + 8 * f) * kSWT + cp + 8 * h) * SG + j;
                        *r = q == 0 ? acc[f][h][j] : *r + acc[f][h][j];
                    }
        }
        __syncthreads();
    }
    for (int e = tid; e < kSWT * kSWT * SG; e += 256) {
        const int64_t k = k0 + e / (kSWT * SG), c = c0 + (e / SG) % kSWT;
        const int j = e % SG;
        if (k < K && c < C) part[((k * C + c) * S + s0 + j) * splits + split] = red[e];
    }
}

// Split-minor partials (part[e][split]): one warp per output, lane j sums splits j, j+32, ... in
// ascending order, then a fixed butterfly adds the 32 lane sums (deterministic).
__global__ void __launch_bounds__(256) reduce_splits_minor_kernel(const float* __restrict__ part,
                                                                  float* __restrict__ out, int64_t count, int splits) {
    const int lane = threadIdx.x % 32;
    for (int64_t e = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / 32; e < count;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x / 32) {
        const float* p = part + e * splits;
        float v = 0.0f;
#pragma unroll 4
        for (int sp = lane; sp < splits; sp += 32) v += p[sp];
#pragma unroll
        for (int o = 16; o > 0; o /= 2) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) out[e] = v;
    }
}

__global__ void reduce_splits_kernel(const float* __restrict__ part, float* __restrict__ out, int64_t count,
                                     int64_t splits) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x) {
        float v = 0.0f;
        for (int64_t sp = 0; sp < splits; ++sp) v += part[sp * count + e];
        out[e] = v;
    }
}

// Many splits: 32 outputs per block, each of the 8 warps sums the splits congruent to it mod 8 (in
// ascending order), then warp 0 adds the 8 partial sums in warp order — a fixed order, so the
// result is deterministic.
__global__ void __launch_bounds__(256) reduce_splits_wide_kernel(const float* __restrict__ part,
                                                                 float* __restrict__ out, int64_t count, int splits) {
    __shared__ float sums[8][33];
    const int lane = threadIdx.x % 32, wp = threadIdx.x / 32;
    for (int64_t e0 = static_cast<int64_t>(blockIdx.x) * 32; e0 < count; e0 += static_cast<int64_t>(gridDim.x) * 32) {
        const int64_t e = e0 + lane;
        float v = 0.0f;
        if (e < count) {
            const float* p = part + e;
#pragma unroll 4
            for (int sp = wp; sp < splits; sp += 8) v += p[static_cast<int64_t>(sp) * count];
        }
        sums[wp][lane] = v;
        __syncthreads();
        if (wp == 0 && e < count) {
            float t = sums[0][lane];
#pragma unroll
            for (int w = 1; w < 8; ++w) t += sums[w][lane];
            out[e] = t;
        }
        __syncthreads();
    }
}

static void launch_reduce_splits(const float* part, float* out, int64_t count, int64_t splits, cudaStream_t stream) {
    if (splits >= 32) {
        reduce_splits_wide_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(count, 32), 4096)), 256, 0,
                                    stream>>>(part, out, count, static_cast<int>(splits));
    } else {
        reduce_splits_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(count, 256), 2048)), 256, 0, stream>>>(
            part, out, count, splits);
    }
    note_launch();
}

// Tiny gradients (K*C*S <= 16, e.g. the 1-filter, 1-tap heads of the config-5 network): each
// output is a dot product over all N*Q columns. Threads stride over columns (coalesced), keep all
// outputs in registers, and every block writes one partial per output; a fixed-order pass sums
// the blocks (deterministic).
constexpr int kSmallOut = 16;
constexpr int kSmallBlocks = 592;  // 4 waves of 148 SMs

template <typename TIn>
__global__ void __launch_bounds__(256) small_wgrad_kernel(const TIn* __restrict__ x, const TIn* __restrict__ dy,
                                                          float* __restrict__ part, int64_t N, int64_t C, int64_t K,
                                                          int64_t S, int64_t D, int64_t Q, int round_in) {
    const int O = static_cast<int>(K * C * S);
    const int64_t W = Q + (S - 1) * D;
    float acc[kSmallOut];
#pragma unroll
    for (int o = 0; o < kSmallOut; ++o) acc[o] = 0.0f;
    const int64_t total = N * Q;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t n = e / Q, qq = e % Q;
#pragma unroll
        for (int o = 0; o < kSmallOut; ++o) {
            if (o < O) {
                const int64_t ss = o % S, cc = (o / S) % C, kk = o / (S * C);
                const float g = load_as_float(dy, (n * K + kk) * Q + qq, round_in != 0);
                const float xv = load_as_float(x, (n * C + cc) * W + qq + ss * D, round_in != 0);
                acc[o] = fmaf(xv, g, acc[o]);
            }
        }
    }
    __shared__ float red[kSmallOut][8];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
#pragma unroll
    for (int o = 0; o < kSmallOut; ++o) {
        float v = acc[o];
        for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
        if (lane == 0) red[o][warp] = v;
    }
    __syncthreads();
    if (threadIdx.x < O) {
        float v = 0.0f;
        for (int w = 0; w < 8; ++w) v += red[threadIdx.x][w];
        part[static_cast<int64_t>(blockIdx.x) * O + threadIdx.x] = v;
    }
}

// 1-tap gradients with few filters (K <= 4, C <= 64; e.g. the network's merged heads):
// dw[k][c] = sum_{n,x} dy[n][k][x] x[n][c][x]. Block (bx, n) owns 1024 columns of item n; each
// thread keeps all K*C sums for its 4 columns, then a fixed-shape tree makes one partial per block
// and output, and a block per output sums the partials in a fixed pattern (deterministic).
// Each thread accumulates kPwGroups column groups of 4 (the block covers kPwGroups x 1024 columns)
// before the K x C warp reductions, which cost more instructions than the loads of one group.
constexpr int kPwGroups = 4;
template <typename TIn, int KMAX, int CMAX>
__global__ void __launch_bounds__(kPwThreads) pointwise_wgrad_kernel(const TIn* __restrict__ x,
                                                                     const TIn* __restrict__ dy,
                                                                     float* __restrict__ part, int64_t C, int64_t K,
                                                                     int64_t Q, int round_in, int vec) {
    __shared__ float red[kPwThreads / 32][KMAX * CMAX];
    const int64_t n = blockIdx.y;
    float acc[KMAX][CMAX];
#pragma unroll
    for (int kk = 0; kk < KMAX; ++kk)
#pragma unroll
        for (int cc = 0; cc < CMAX; ++cc) acc[kk][cc] = 0.0f;
    for (int grp = 0; grp < kPwGroups; ++grp) {
        const int64_t x0 = (static_cast<int64_t>(blockIdx.x) * kPwGroups + grp) * kPwCols + threadIdx.x * 4;
        const int cnt = static_cast<int>(x0 < Q ? (Q - x0 < 4 ? Q - x0 : 4) : 0);
        if (cnt == 0) break;
        const bool v4 = vec && cnt == 4;
        float gv[KMAX][4];
#pragma unroll
        for (int kk = 0; kk < KMAX; ++kk) {
            if (v4 && kk < K) {
                load4_as_float(dy, (n * K + kk) * Q + x0, round_in != 0, gv[kk]);
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    gv[kk][j] = (kk < K && j < cnt) ? load_as_float(dy, (n * K + kk) * Q + x0 + j, round_in != 0) : 0.0f;
            }
        }
#pragma unroll
        for (int cc = 0; cc < CMAX; ++cc) {
            if (cc >= C) break;
            float xv[4];
            if (v4) {
                load4_as_float(x, (n * C + cc) * Q + x0, round_in != 0, xv);
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    xv[j] = j < cnt ? load_as_float(x, (n * C + cc) * Q + x0 + j, round_in != 0) : 0.0f;
            }
#pragma unroll
            for (int kk = 0; kk < KMAX; ++kk)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[kk][cc] = fmaf(gv[kk][j], xv[j], acc[kk][cc]);
        }
    }
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
#pragma unroll
    for (int kk = 0; kk < KMAX; ++kk)
#pragma unroll
        for (int cc = 0; cc < CMAX; ++cc) {
            float v = acc[kk][cc];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
            if (lane == 0) red[warp][kk * CMAX + cc] = v;
        }
    __syncthreads();
    const int64_t P = static_cast<int64_t>(gridDim.x) * gridDim.y;
    const int64_t pidx = n * gridDim.x + blockIdx.x;
    for (int o = threadIdx.x; o < KMAX * CMAX; o += kPwThreads) {
        const int kk = o / CMAX, cc = o % CMAX;
        if (kk >= K || cc >= C) continue;
        float v = 0.0f;
        for (int w = 0; w < kPwThreads / 32; ++w) v += red[w][o];
        part[(kk * C + cc) * P + pidx] = v;  // [output][partial]
    }
}

// out[o] = sum_p part[o * P + p], one CTA per output: thread t sums p = t, t+256, ... in order,
// then a fixed tree.
__global__ void __launch_bounds__(256) reduce_partials_kernel(const float* __restrict__ part,
                                                              float* __restrict__ out, int64_t P) {
    __shared__ float red[8];
    const int64_t o = blockIdx.x;
    float t = 0.0f;
    for (int64_t p = threadIdx.x; p < P; p += 256) t += part[o * P + p];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
        float s = 0.0f;
        for (int w = 0; w < 8; ++w) s += red[w];
        out[o] = s;
    }
}

static bool pointwise_wgrad_ok(int64_t n, int64_t c, int64_t k, int64_t s) {
    return s == 1 && k <= 4 && c <= 64 && n <= 65535;
}

template <typename TIn>
static cudaError_t launch_pointwise_wgrad(const TIn* x, const TIn* dy, float* dw, float* part, int64_t n, int64_t c,
                                          int64_t k, int64_t q, int round_in, cudaStream_t stream) {
    const dim3 grid(static_cast<unsigned>(ceil_div(q, kPwCols * kPwGroups)), static_cast<unsigned>(n));
    const uintptr_t al = sizeof(TIn) == 4 ? 15u : 7u;
    const int vec = q % 4 == 0 && (reinterpret_cast<uintptr_t>(x) & al) == 0 &&
                    (reinterpret_cast<uintptr_t>(dy) & al) == 0;  // vector loads of x and dy rows
    if (k <= 2 && c <= 16)
        pointwise_wgrad_kernel<TIn, 2, 16><<<grid, kPwThreads, 0, stream>>>(x, dy, part, c, k, q, round_in, vec);
    else if (c <= 16)
        pointwise_wgrad_kernel<TIn, 4, 16><<<grid, kPwThreads, 0, stream>>>(x, dy, part, c, k, q, round_in, vec);
    else
        pointwise_wgrad_kernel<TIn, 4, 64><<<grid, kPwThreads, 0, stream>>>(x, dy, part, c, k, q, round_in, vec);
    note_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    reduce_partials_kernel<<<static_cast<unsigned>(k * c), 256, 0, stream>>>(part, dw,
                                                                             static_cast<int64_t>(grid.x) * grid.y);
    note_launch();
    return cudaGetLastError();
}

static size_t slide_smem(int d, int sg) {  // two buffers
    return 2 * sizeof(float) *
           static_cast<size_t>(kSWT * slide_pitch(d * slide_lg(d)) + kSWT * slide_pitch(d * slide_lx(d, sg)));
}

template <typename TIn, int SG>
static cudaError_t launch_slide_sg(dim3 grid, size_t smem, cudaStream_t stream, const TIn* x, const TIn* dy, float* part,
                                   int64_t n, int64_t c, int64_t k, int64_t s, int64_t d, int64_t q, int64_t splits,
                                   int lx, int round_in, int64_t s0) {
    cudaError_t e = cudaFuncSetAttribute(wgrad_slide_kernel<TIn, SG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    wgrad_slide_kernel<TIn, SG><<<grid, 256, smem, stream>>>(x, dy, part, n, c, k, s, d, q, splits, lx, round_in, s0);
    note_launch();
    return cudaGetLastError();
}

template <typename TIn>
static cudaError_t launch_slide(int sg, dim3 grid, size_t smem, cudaStream_t stream, const TIn* x, const TIn* dy,
                                float* part, int64_t n, int64_t c, int64_t k, int64_t s, int64_t d, int64_t q,
                                int64_t splits, int lx, int round_in, int64_t s0) {
#define C1D_SLIDE(SGV) \
    case SGV:          \
        return launch_slide_sg<TIn, SGV>(grid, smem, stream, x, dy, part, n, c, k, s, d, q, splits, lx, round_in, s0)
    switch (sg) {
        C1D_SLIDE(1); C1D_SLIDE(2); C1D_SLIDE(3); C1D_SLIDE(4); C1D_SLIDE(5); C1D_SLIDE(6); C1D_SLIDE(7);
        C1D_SLIDE(8); C1D_SLIDE(9);
        default: C1D_SLIDE(10);
    }
#undef C1D_SLIDE
}

cudaError_t launch_direct_wgrad(const void* x, const void* dy, int in_dtype, bool round_in, float* dw_kcs,
                                float* workspace, int64_t n, int64_t c, int64_t k, int64_t s, int64_t d,
                                int64_t q, cudaStream_t stream) {
    if (pointwise_wgrad_ok(n, c, k, s)) {
        if (in_dtype == 0)
            return launch_pointwise_wgrad(static_cast<const float*>(x), static_cast<const float*>(dy), dw_kcs,
                                          workspace, n, c, k, q, round_in ? 1 : 0, stream);
        return launch_pointwise_wgrad(static_cast<const uint16_t*>(x), static_cast<const uint16_t*>(dy), dw_kcs,
                                      workspace, n, c, k, q, 0, stream);
    }
    if (k * c * s <= kSmallOut) {
        if (in_dtype == 0)
            small_wgrad_kernel<float><<<kSmallBlocks, 256, 0, stream>>>(static_cast<const float*>(x),
                                                                      static_cast<const float*>(dy), workspace, n, c,
                                                                      k, s, d, q, round_in ? 1 : 0);
        else
            small_wgrad_kernel<uint16_t><<<kSmallBlocks, 256, 0, stream>>>(static_cast<const uint16_t*>(x),
                                                                         static_cast<const uint16_t*>(dy), workspace,
                                                                         n, c, k, s, d, q, 0);
        note_launch();
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        // part is [block][o] with o in KCS order; sum blocks in ascending order
        const int64_t count = k * c * s;
        // reuse reduce_splits_kernel: it expects part[split * count + e]
        reduce_splits_kernel<<<1, 32, 0, stream>>>(workspace, dw_kcs, count, kSmallBlocks);
        note_launch();
        return cudaGetLastError();
    }
    if (slide_wgrad_ok(n, s, d, q)) {
        const int64_t splits = slide_wgrad_splits(n, c, k, s, d, q);
        dim3 grid(static_cast<unsigned>(ceil_div(k, kSWT)), static_cast<unsigned>(ceil_div(c, kSWT)),
                  static_cast<unsigned>(splits));
        cudaError_t e = cudaSuccess;
        // balanced tap groups of at most kSWG taps (S = 25 -> 9 + 8 + 8)
        const int64_t groups = ceil_div(s, kSWG);
        for (int64_t gi = 0, s0 = 0; gi < groups && e == cudaSuccess; ++gi) {
            const int sg = static_cast<int>(s / groups + (gi < s % groups ? 1 : 0));
            const int lx = slide_lx(static_cast<int>(d), sg);
            const size_t smem = slide_smem(static_cast<int>(d), sg);
            e = in_dtype == 0 ? launch_slide<float>(sg, grid, smem, stream, static_cast<const float*>(x),
                                                    static_cast<const float*>(dy), workspace, n, c, k, s, d, q, splits,
                                                    lx, round_in ? 1 : 0, s0)
                              : launch_slide<uint16_t>(sg, grid, smem, stream, static_cast<const uint16_t*>(x),
                                                       static_cast<const uint16_t*>(dy), workspace, n, c, k, s, d, q,
                                                       splits, lx, 0, s0);
            s0 += sg;
        }
        if (e != cudaSuccess) return e;
        const int64_t count = k * c * s;
        reduce_splits_minor_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(count, 8), 4096)), 256, 0,
                                     stream>>>(workspace, dw_kcs, count, static_cast<int>(splits));
        note_launch();
        return cudaGetLastError();
    }
    const int64_t splits = wgrad_splits(n, c, k, q);
    // taps per group: 8, fewer when a huge dilation would not fit the X window in shared memory
    int tg = static_cast<int>(std::min<int64_t>(kWG, s));
    auto smem_for = [&](int g) {
        const int64_t span = kWQ + (g - 1) * d;
        return sizeof(float) * static_cast<size_t>(kWK * kWQ + kWC * (span | 1));
    };
    while (tg > 1 && smem_for(tg) > 200 * 1024) --tg;
    const int xpitch = static_cast<int>((kWQ + (tg - 1) * d) | 1);  // odd: 32 channel rows, distinct banks
    const size_t smem = smem_for(tg);
    if (smem > 227 * 1024) return cudaErrorInvalidValue;
    dim3 grid(static_cast<unsigned>(ceil_div(k, kWK)), static_cast<unsigned>(ceil_div(c, kWC)),
              static_cast<unsigned>(splits));
    cudaError_t e;
    if (in_dtype == 0) {
        e = cudaFuncSetAttribute(direct_wgrad_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        direct_wgrad_kernel<float><<<grid, 256, smem, stream>>>(static_cast<const float*>(x),
                                                                 static_cast<const float*>(dy), workspace, n, c, k, s,
                                                                 d, q, splits, tg, xpitch, round_in ? 1 : 0);
    } else {
        e = cudaFuncSetAttribute(direct_wgrad_kernel<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        direct_wgrad_kernel<uint16_t><<<grid, 256, smem, stream>>>(static_cast<const uint16_t*>(x),
                                                                    static_cast<const uint16_t*>(dy), workspace, n, c,
                                                                    k, s, d, q, splits, tg, xpitch, 0);
    }
    note_launch();
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const int64_t count = k * c * s;
    launch_reduce_splits(workspace, dw_kcs, count, splits, stream);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------- bf16 rounding
__global__ void round_bf16_kernel(const float* __restrict__ in, uint16_t* __restrict__ out, int64_t count) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 4;
    // vectorised body when 16-byte aligned
    const bool vec = ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
    if (vec) {
        for (; i + 3 < count; i += stride * 4) {
            const float4 v = *reinterpret_cast<const float4*>(in + i);
            uint2 o;
            o.x = static_cast<uint32_t>(fp32_to_bf16_bits(v.x)) | (static_cast<uint32_t>(fp32_to_bf16_bits(v.y)) << 16);
            o.y = static_cast<uint32_t>(fp32_to_bf16_bits(v.z)) | (static_cast<uint32_t>(fp32_to_bf16_bits(v.w)) << 16);
            *reinterpret_cast<uint2*>(out + i) = o;
        }
        for (int64_t j = i; j < count && j < i + 4; ++j) out[j] = fp32_to_bf16_bits(in[j]);
    } else {
        for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < count; j += stride)
            out[j] = fp32_to_bf16_bits(in[j]);
    }
}

cudaError_t launch_round_bf16(const float* in, uint16_t* out, int64_t count, cudaStream_t stream) {
    if (count <= 0) return cudaSuccess;
    const int threads = 256;
    const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(ceil_div(count, 4), threads), 8 * num_sms()));
    round_bf16_kernel<<<blocks, threads, 0, stream>>>(in, out, count);
    note_launch();
    return cudaGetLastError();
}

}  // namespace c1d
