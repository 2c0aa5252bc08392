// relayout.cu — dilations other than 8 on the dilation-8 tensor-core kernels.
//
// The row-tap kernels need one tap = 8 columns = 16 bytes. Two exact rewrites bring other
// dilations there (the reference computes the same sums, conv.cpp:86-138, in tap order):
//
//  d < 8, 8 % d == 0 (m = 8/d): tap s = b + m*t reads x[q + b*d + 8t], so the conv is ONE
//     dilation-8 conv over P = min(m, S) "phase channels" (b, i) = source channel i shifted by b*d
//     columns, with S' = ceil(S/m) taps and weights w'[o][b*I + i][t] = w[o][i][b + m*t]. TMA and
//     cp.async need 16-B aligned starts, so the shifted channels are materialised as bf16 copies
//     (shift_copies). Backward-weight runs one launch per phase on that phase's shifted x copy and
//     scatters tap t of phase b back to tap b + m*t.
//  d < 8 (the default since round 1's expanded-row mode; phases remain the fallback): expanded
//     rows. E[nc][r] = the 8 elements x[d*r .. d*r+7] (a (8/d)x larger bf16 tensor). In E a tap is
//     one 16-B row and 8 output columns are 8/d rows, so tc_conv reads the MMA's A operand straight
//     from E with an M-group stride of 128/d bytes: 16 consecutive taps per MMA at any d | 8.
//  d = 8m (m >= 2): chunk planes. Column 8u+e lives in plane u mod m; a dilation-8m tap step is one
//     chunk inside a plane, so the conv is a dilation-8 conv on N*m planes of width W/m (inputs
//     de-interleaved here, outputs re-interleaved).
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace c1d {

namespace {

unsigned blocks_for(int64_t total) {
    return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, 256), 16 * num_sms())));
}

__global__ void phase_split_weights_kernel(const float* __restrict__ w, float* __restrict__ out, int64_t O,
                                           int64_t I, int64_t S, int64_t m, int64_t P) {
    const int64_t Sp = ceil_div(S, m);
    const int64_t total = O * P * I * Sp;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = e % Sp;
        const int64_t vc = (e / Sp) % (P * I);
        const int64_t o = e / (Sp * P * I);
        const int64_t b = vc / I, i = vc % I;
        const int64_t s = b + m * t;
        out[e] = s < S ? w[(o * I + i) * S + s] : 0.0f;
    }
}

__global__ void scatter_phase_wgrad_kernel(const float* __restrict__ dwb, float* __restrict__ dw, int64_t K,
                                           int64_t C, int64_t S, int64_t m, int64_t b) {
    const int64_t Sb = ceil_div(S - b, m);  // taps of phase b
    const int64_t total = K * C * Sb;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = e % Sb;
        const int64_t kc = e / Sb;
        dw[kc * S + b + m * t] = dwb[e];
    }
}

// out[(n*m + r)][c][8u + e] = in[n][c][8(u*m + r) + e]; 16-byte chunks, one per thread
template <typename TIn>
__global__ void to_planes_kernel(const TIn* __restrict__ in, uint16_t* __restrict__ out, int64_t n, int64_t c,
                                 int64_t w, int64_t m) {
    const int64_t wp = w / m;          // plane width (columns)
    const int64_t chunks = wp / 8;     // chunks per plane row
    const int64_t total = n * m * c * chunks;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t u = e % chunks;
        const int64_t cc = (e / chunks) % c;
        const int64_t r = (e / (chunks * c)) % m;
        const int64_t nn = e / (chunks * c * m);
        const int64_t src = (nn * c + cc) * w + 8 * (u * m + r);
        uint16_t v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if constexpr (sizeof(TIn) == 4)
                v[j] = fp32_to_bf16_bits(reinterpret_cast<const float*>(in)[src + j]);
            else
                v[j] = reinterpret_cast<const uint16_t*>(in)[src + j];
        }
        uint4 pk;
        pk.x = v[0] | (static_cast<uint32_t>(v[1]) << 16);
        pk.y = v[2] | (static_cast<uint32_t>(v[3]) << 16);
        pk.z = v[4] | (static_cast<uint32_t>(v[5]) << 16);
        pk.w = v[6] | (static_cast<uint32_t>(v[7]) << 16);
        *reinterpret_cast<uint4*>(out + ((nn * m + r) * c + cc) * wp + 8 * u) = pk;
    }
}

// out[n][c][8(u*m + r) + e] = in[(n*m + r)][c][8u + e] (FP32)
__global__ void from_planes_kernel(const float* __restrict__ in, float* __restrict__ out, int64_t n, int64_t c,
                                   int64_t w, int64_t m) {
    const int64_t wp = w / m;
    const int64_t chunks = wp / 8;
    const int64_t total = n * m * c * chunks;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t u = e % chunks;
        const int64_t cc = (e / chunks) % c;
        const int64_t r = (e / (chunks * c)) % m;
        const int64_t nn = e / (chunks * c * m);
        const float4* src = reinterpret_cast<const float4*>(in + ((nn * m + r) * c + cc) * wp + 8 * u);
        float4* dst = reinterpret_cast<float4*>(out + (nn * c + cc) * w + 8 * (u * m + r));
        dst[0] = src[0];
        dst[1] = src[1];
    }
}

template <typename TIn, typename TOut>
__global__ void shift_copies_kernel(const TIn* __restrict__ in, TOut* __restrict__ out, int64_t n, int64_t I,
                                    int64_t w, int64_t P, int64_t base, int64_t delta, int64_t w_out) {
    const int64_t total = n * P * I * w_out;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = e % w_out;
        const int64_t row = e / w_out;  // (n, b, i)
        const int64_t i = row % I, b = (row / I) % P, nn = row / (I * P);
        const int64_t src = j + base + b * delta;
        if constexpr (sizeof(TOut) == 4) {  // FP32 copy (the split-FP32 path splits afterwards)
            out[e] = (src >= 0 && src < w) ? in[(nn * I + i) * w + src] : 0.0f;
        } else {
            uint16_t v = 0;
            if (src >= 0 && src < w) {
                const int64_t at = (nn * I + i) * w + src;
                if constexpr (sizeof(TIn) == 4)
                    v = fp32_to_bf16_bits(reinterpret_cast<const float*>(in)[at]);
                else
                    v = reinterpret_cast<const uint16_t*>(in)[at];
            }
            out[e] = v;
        }
    }
}

// grid (column blocks of 1024, rows in y with a stride loop): 4 columns per thread, 32-bit
// column math (a per-element 64-bit division made this HBM-trivial copy ALU-bound)
template <typename TIn>
__global__ void __launch_bounds__(256) pad_rows_kernel(const TIn* __restrict__ in, uint16_t* __restrict__ out,
                                                       int64_t rows, int64_t w, int64_t w_pad) {
    const int j0 = (blockIdx.x * 256 + threadIdx.x) * 4;
    if (j0 >= w_pad) return;
    for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
        const TIn* src = in + r * w;
        uint16_t* dst = out + r * w_pad;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
            const int j = j0 + jj;
            if (j >= w_pad) break;
            uint16_t v = 0;
            if (j < w) {
                if constexpr (sizeof(TIn) == 4)
                    v = fp32_to_bf16_bits(__ldg(reinterpret_cast<const float*>(src) + j));
                else
                    v = __ldg(reinterpret_cast<const uint16_t*>(src) + j);
            }
            dst[j] = v;
        }
    }
}

// one 16-B row per thread: out[nc][r][0..7] = in[nc][d*r + off + 0..7]
template <typename TIn>
__global__ void expand_rows_kernel(const TIn* __restrict__ in, uint4* __restrict__ out, int64_t nc, int64_t w,
                                   int64_t d, int64_t off, int64_t rows) {
    const int64_t total = nc * rows;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e % rows, row = e / rows;
        const int64_t c0 = d * r + off;
        const TIn* src = in + row * w;
        uint16_t v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int64_t col = c0 + j;
            uint16_t b = 0;
            if (col >= 0 && col < w) {
                if constexpr (sizeof(TIn) == 4)
                    b = fp32_to_bf16_bits(reinterpret_cast<const float*>(src)[col]);
                else
                    b = reinterpret_cast<const uint16_t*>(src)[col];
            }
            v[j] = b;
        }
        uint4 pk;
        pk.x = v[0] | (static_cast<uint32_t>(v[1]) << 16);
        pk.y = v[2] | (static_cast<uint32_t>(v[3]) << 16);
        pk.z = v[4] | (static_cast<uint32_t>(v[5]) << 16);
        pk.w = v[6] | (static_cast<uint32_t>(v[7]) << 16);
        out[e] = pk;
    }
}

// Channel-octet streams for tc_wgrad2's xt mode: out[n][o][u][0..7] = bf16(in[n][8o + e][u]) for
// u < rows (zero for channels >= C or columns >= w). Thread u of a block reads column u of the
// octet's 8 channel rows (each load instruction is coalesced along the row) and writes one 16-B
// row (consecutive threads: consecutive rows).
template <typename TIn>
__global__ void __launch_bounds__(256) to_octets_kernel(const TIn* __restrict__ in, uint4* __restrict__ out,
                                                        int64_t c, int64_t w, int64_t rows, int64_t octets) {
    const int64_t no = blockIdx.y;  // n * octets + o
    const int64_t n = no / octets, o = no % octets;
    const int64_t u = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x;
    if (u >= rows) return;
    uint16_t v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int64_t ch = 8 * o + e;
        uint16_t b = 0;
        if (ch < c && u < w) {
            const TIn* src = in + (n * c + ch) * w + u;
            if constexpr (sizeof(TIn) == 4)
                b = fp32_to_bf16_bits(__ldg(reinterpret_cast<const float*>(src)));
            else
                b = __ldg(reinterpret_cast<const uint16_t*>(src));
        }
        v[e] = b;
    }
    uint4 pk;
    pk.x = v[0] | (static_cast<uint32_t>(v[1]) << 16);
    pk.y = v[2] | (static_cast<uint32_t>(v[3]) << 16);
    pk.z = v[4] | (static_cast<uint32_t>(v[5]) << 16);
    pk.w = v[6] | (static_cast<uint32_t>(v[7]) << 16);
    out[no * rows + u] = pk;
}

}  // namespace

cudaError_t launch_to_octets(const void* in, int in_dtype, uint16_t* out, int64_t n, int64_t c, int64_t w,
                             int64_t rows, cudaStream_t stream) {
    const int64_t octets = (c + 7) / 8;
    if (n * octets > 65535) return cudaErrorInvalidValue;
    const dim3 grid(static_cast<unsigned>(ceil_div(rows, 256)), static_cast<unsigned>(n * octets));
    if (in_dtype == 0)
        to_octets_kernel<float><<<grid, 256, 0, stream>>>(static_cast<const float*>(in), reinterpret_cast<uint4*>(out), c,
                                                          w, rows, octets);
    else
        to_octets_kernel<uint16_t><<<grid, 256, 0, stream>>>(static_cast<const uint16_t*>(in),
                                                             reinterpret_cast<uint4*>(out), c, w, rows, octets);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_expand_rows(const void* in, int in_dtype, uint16_t* out, int64_t nc, int64_t w, int64_t d,
                               int64_t off, int64_t rows, cudaStream_t stream) {
    const unsigned blocks = blocks_for(nc * rows);
    if (in_dtype == 0)
        expand_rows_kernel<float><<<blocks, 256, 0, stream>>>(static_cast<const float*>(in), reinterpret_cast<uint4*>(out),
                                                              nc, w, d, off, rows);
    else
        expand_rows_kernel<uint16_t><<<blocks, 256, 0, stream>>>(static_cast<const uint16_t*>(in),
                                                                 reinterpret_cast<uint4*>(out), nc, w, d, off, rows);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_shift_copies(const void* in, int in_dtype, uint16_t* out, int64_t n, int64_t I, int64_t w,
                                int64_t P, int64_t base, int64_t delta, int64_t w_out, cudaStream_t stream) {
    const int64_t total = n * P * I * w_out;
    if (in_dtype == 0)
        shift_copies_kernel<float, uint16_t><<<blocks_for(total), 256, 0, stream>>>(static_cast<const float*>(in), out,
                                                                                    n, I, w, P, base, delta, w_out);
    else
        shift_copies_kernel<uint16_t, uint16_t><<<blocks_for(total), 256, 0, stream>>>(
            static_cast<const uint16_t*>(in), out, n, I, w, P, base, delta, w_out);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_shift_copies_f32(const float* in, float* out, int64_t n, int64_t I, int64_t w, int64_t P,
                                    int64_t base, int64_t delta, int64_t w_out, cudaStream_t stream) {
    shift_copies_kernel<float, float><<<blocks_for(n * P * I * w_out), 256, 0, stream>>>(in, out, n, I, w, P, base,
                                                                                         delta, w_out);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_pad_rows(const void* in, int in_dtype, uint16_t* out, int64_t rows, int64_t w, int64_t w_pad,
                            cudaStream_t stream) {
    if (w_pad >= (int64_t{1} << 30)) return cudaErrorInvalidValue;
    const dim3 grid(static_cast<unsigned>(ceil_div(w_pad, 1024)), static_cast<unsigned>(std::min<int64_t>(rows, 65535)));
    if (rows == 0) return cudaSuccess;
    if (in_dtype == 0)
        pad_rows_kernel<float><<<grid, 256, 0, stream>>>(static_cast<const float*>(in), out, rows, w, w_pad);
    else
        pad_rows_kernel<uint16_t><<<grid, 256, 0, stream>>>(static_cast<const uint16_t*>(in), out, rows, w, w_pad);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_phase_split_weights(const float* w, float* out, int64_t O, int64_t I, int64_t S, int64_t m,
                                       int64_t P, cudaStream_t stream) {
    phase_split_weights_kernel<<<blocks_for(O * P * I * ceil_div(S, m)), 256, 0, stream>>>(w, out, O, I, S, m, P);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_scatter_phase_wgrad(const float* dwb, float* dw, int64_t K, int64_t C, int64_t S, int64_t m,
                                       int64_t b, cudaStream_t stream) {
    scatter_phase_wgrad_kernel<<<blocks_for(K * C * ceil_div(S - b, m)), 256, 0, stream>>>(dwb, dw, K, C, S, m, b);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_to_planes(const void* in, int in_dtype, uint16_t* out, int64_t n, int64_t c, int64_t w,
                             int64_t m, cudaStream_t stream) {
    if (w % (8 * m)) return cudaErrorInvalidValue;
    const unsigned blocks = blocks_for(n * c * (w / 8));
    if (in_dtype == 0)
        to_planes_kernel<float><<<blocks, 256, 0, stream>>>(static_cast<const float*>(in), out, n, c, w, m);
    else
        to_planes_kernel<uint16_t><<<blocks, 256, 0, stream>>>(static_cast<const uint16_t*>(in), out, n, c, w, m);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_from_planes(const float* in, float* out, int64_t n, int64_t c, int64_t w, int64_t m,
                               cudaStream_t stream) {
    if (w % (8 * m)) return cudaErrorInvalidValue;
    from_planes_kernel<<<blocks_for(n * c * (w / 8)), 256, 0, stream>>>(in, out, n, c, w, m);
    note_launch();
    return cudaGetLastError();
}

}  // namespace c1d
