// split.cu — FP32 precision on the BF16 tensor-core kernels by operand splitting.
//
// Every FP32 value v is written as v = hi + lo + e with hi = bf16(v), lo = bf16(v - hi) (both
// round-to-nearest-even), |e| <= 2^-18 |v|. A product w*x is then
//   w_hi*x_hi + w_hi*x_lo + w_lo*x_hi  (+ w_lo*x_lo)
// with every partial product exact in the tensor core's FP32 accumulator. The split is expressed
// as extra channels so the tcgen05 kernels do all the work:
//   forward / backward-data:  x' = [x_hi | x_lo | x_hi | x_lo] (4C channels),
//                             w' = [w_hi | w_hi | w_lo | w_lo]; channel block 0 (hi*hi) accumulates
//                             in its own TMEM region, the three correction blocks in a second one
//   backward-weight:          x' = [x_hi | x_lo] (2C), dy' = [dy_hi | dy_lo] (2K); the 2K x 2C
//                             weight gradient's four blocks are summed (hi*hi + hi*lo + lo*hi + lo*lo).
// Error per product is <= 2*2^-18 relative (the two split residuals), plus the tensor core's
// FP32 accumulation error on the main chain; c1d_api.cu gates the path so the total stays inside
// the reference's 1e-5 FP32 bound.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace c1d {

// in: [N][C][W] fp32 -> out: [N][R*C][W] bf16 bits, channel block b of `pattern` (bit b: 0 = hi,
// 1 = lo) for b < R. One row (item, channel) per blockIdx.y step; each thread splits 8 consecutive
// columns and writes them as one 16-B store per block when wp is a multiple of 8 (output rows then
// 16-B aligned); rows whose input start is 16-B aligned read two float4s.
__global__ void split_channels_kernel(const float* __restrict__ in, uint16_t* __restrict__ out, int64_t n,
                                      int64_t c, int64_t w, int reps, unsigned pattern, int64_t wp,
                                      int64_t in_item) {
    for (int64_t row = blockIdx.y; row < n * c; row += gridDim.y) {
        const int64_t item = row / c, ch = row - item * c;
        const float* src = in + item * in_item + ch * w;
        const bool vec = ((reinterpret_cast<uintptr_t>(src) & 15u) == 0);
        const bool vout = (wp % 8) == 0 && (reinterpret_cast<uintptr_t>(out) & 15u) == 0;
        for (int64_t x0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 8; x0 < wp;
             x0 += static_cast<int64_t>(gridDim.x) * blockDim.x * 8) {
            float v[8];
            if (vec && x0 + 8 <= w) {
                const float4 a = __ldg(reinterpret_cast<const float4*>(src + x0));
                const float4 b = __ldg(reinterpret_cast<const float4*>(src + x0 + 4));
                v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
                v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
            } else {
#pragma unroll
                for (int j = 0; j < 8; ++j) v[j] = x0 + j < w ? __ldg(src + x0 + j) : 0.0f;  // pitch padding: zeros
            }
            uint32_t hi[4], lo[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                uint16_t h[2], l[2];
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    h[e] = fp32_to_bf16_bits(v[2 * j + e]);
                    l[e] = fp32_to_bf16_bits(v[2 * j + e] - bf16_bits_to_fp32(h[e]));
                }
                hi[j] = static_cast<uint32_t>(h[0]) | (static_cast<uint32_t>(h[1]) << 16);
                lo[j] = static_cast<uint32_t>(l[0]) | (static_cast<uint32_t>(l[1]) << 16);
            }
            for (int r = 0; r < reps; ++r) {
                const bool is_lo = (pattern >> r) & 1u;
                uint16_t* dst = out + ((item * reps + r) * c + ch) * wp + x0;
                if (vout) {
                    *reinterpret_cast<uint4*>(dst) =
                        is_lo ? make_uint4(lo[0], lo[1], lo[2], lo[3]) : make_uint4(hi[0], hi[1], hi[2], hi[3]);
                } else {  // unpadded odd-width rows: element stores
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        if (x0 + j < wp) dst[j] = static_cast<uint16_t>((is_lo ? lo[j / 2] : hi[j / 2]) >> (16 * (j % 2)));
                }
            }
        }
    }
}

// Weights KCS fp32 [K][C][S] -> expanded KCS fp32 [K*kr][C*cr][S] whose entries are the bf16 hi or
// lo parts (exactly representable), selected per (k-block, c-block) by `sel` (bit kb*cr + cb).
__global__ void split_weights_kernel(const float* __restrict__ w, float* __restrict__ out, int64_t K, int64_t C,
                                     int64_t S, int kr, int cr, unsigned sel) {
    const int64_t total = K * kr * C * cr * S;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = e % S;
        const int64_t cc = (e / S) % (C * cr);
        const int64_t kk = e / (S * C * cr);
        const int64_t cb = cc / C, c = cc % C, kb = kk / K, k = kk % K;
        const float v = w[(k * C + c) * S + s];
        const uint16_t hi = fp32_to_bf16_bits(v);
        const float hif = bf16_bits_to_fp32(hi);
        const float lof = bf16_bits_to_fp32(fp32_to_bf16_bits(v - hif));
        out[e] = ((sel >> (kb * cr + cb)) & 1u) ? lof : hif;
    }
}

// dw[k][c][s] = sum over the 2x2 (k-block, c-block) tiles of dw4[(kb*K + k)][(cb*C + c)][s]
__global__ void sum_split_blocks_kernel(const float* __restrict__ dw4, float* __restrict__ dw, int64_t K, int64_t C,
                                        int64_t S) {
    const int64_t total = K * C * S;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = e % S, c = (e / S) % C, k = e / (S * C);
        // fixed order: small terms first
        const float ll = dw4[((K + k) * 2 * C + (C + c)) * S + s];
        const float lh = dw4[((K + k) * 2 * C + c) * S + s];
        const float hl = dw4[(k * 2 * C + (C + c)) * S + s];
        const float hh = dw4[(k * 2 * C + c) * S + s];
        dw[e] = hh + (hl + (lh + ll));
    }
}

// dw = hh + (hl + lh): the block-launch form of the split backward-weight (same order as
// sum_split_blocks without the lo x lo term)
__global__ void sum3_kernel(const float* __restrict__ hh, const float* __restrict__ hl, const float* __restrict__ lh,
                            float* __restrict__ dw, int64_t count) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x)
        dw[e] = hh[e] + (hl[e] + lh[e]);
}

static unsigned blocks_for(int64_t total) {
    return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, 256), 16 * num_sms())));
}

cudaError_t launch_split_channels(const float* in, uint16_t* out, int64_t n, int64_t c, int64_t w, int reps,
                                  unsigned pattern, cudaStream_t stream, int64_t w_pitch, int64_t in_item_stride) {
    const int64_t wp = w_pitch > 0 ? w_pitch : w;
    const int64_t si = in_item_stride > 0 ? in_item_stride : c * w;
    const int64_t rows = n * c;
    const unsigned gx = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(wp, 8 * 256), 64)));
    const unsigned gy = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(rows, 65535)));
    split_channels_kernel<<<dim3(gx, gy), 256, 0, stream>>>(in, out, n, c, w, reps, pattern, wp, si);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_split_weights(const float* w, float* out, int64_t K, int64_t C, int64_t S, int kr, int cr,
                                 unsigned sel, cudaStream_t stream) {
    split_weights_kernel<<<blocks_for(K * kr * C * cr * S), 256, 0, stream>>>(w, out, K, C, S, kr, cr, sel);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_sum_split_blocks(const float* dw4, float* dw, int64_t K, int64_t C, int64_t S,
                                    cudaStream_t stream) {
    sum_split_blocks_kernel<<<blocks_for(K * C * S), 256, 0, stream>>>(dw4, dw, K, C, S);
    note_launch();
    return cudaGetLastError();
}

__global__ void add_into_kernel(float* __restrict__ out, const float* __restrict__ add, int64_t count) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x)
        out[e] += add[e];
}

cudaError_t launch_add_into(float* out, const float* add, int64_t count, cudaStream_t stream) {
    add_into_kernel<<<blocks_for(count), 256, 0, stream>>>(out, add, count);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_sum3(const float* hh, const float* hl, const float* lh, float* dw, int64_t count,
                        cudaStream_t stream) {
    sum3_kernel<<<blocks_for(count), 256, 0, stream>>>(hh, hl, lh, dw, count);
    note_launch();
    return cudaGetLastError();
}

}  // namespace c1d
