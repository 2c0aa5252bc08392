// layer.cu — the per-layer glue of the reference's ConvLayer (proj/src/train.cpp:173-221), fused
// into one memory pass each way.
//
// Forward (train.cpp:176-192): after the conv, pre += bias; a = ReLU(pre); a += skip. The
// reference keeps every activation FP32 and the next BF16 layer rounds its (zero-padded) input
// inside the conv (conv.cpp:182-183). Here one pass adds the bias (stored back only on request:
// the backward recomputes the ReLU mask from the conv output and the bias), applies ReLU and the
// skip, and writes the activation as FP32
// (for skips / FP32 consumers) and/or straight into the next layer's zero-padded BF16 input
// (same RNE as bf16.hpp:29-40), so no pad copy and no separate rounding pass remain.
//
// Backward (train.cpp:205-221): g = incoming gradient (optionally the interior of a padded
// backward-data output, plus a skip gradient), gp = g * (pre > 0), bias grad = sum over items and
// columns of gp, and gp feeds the next backward-weight / backward-data as FP32 or BF16. The bias
// gradient is reduced deterministically: fixed-shape block trees, then a fixed-order sum.
#include "common.cuh"
#include "kernels.h"

namespace c1d {

namespace {

constexpr int kEltThreads = 256;
constexpr int kEltPerThread = 4;
constexpr int kEltPerBlock = kEltThreads * kEltPerThread;  // columns per block (one row)

__device__ __forceinline__ void store_bf16x4(uint16_t* dst, const float v[4], bool vec) {
    const uint16_t b0 = fp32_to_bf16_bits(v[0]), b1 = fp32_to_bf16_bits(v[1]);
    const uint16_t b2 = fp32_to_bf16_bits(v[2]), b3 = fp32_to_bf16_bits(v[3]);
    if (vec) {
        uint2 u;
        u.x = static_cast<uint32_t>(b0) | (static_cast<uint32_t>(b1) << 16);
        u.y = static_cast<uint32_t>(b2) | (static_cast<uint32_t>(b3) << 16);
        *reinterpret_cast<uint2*>(dst) = u;
    } else {
        dst[0] = b0;
        dst[1] = b1;
        dst[2] = b2;
        dst[3] = b3;
    }
}

// grid (ceil(q / 1024), n*k). `vec`: every row start of every operand is 16-B aligned and q % 4 == 0.
// mask: (pre + bias > 0) as channel-block words (kernels.h LayerGlue), zeroed by the launcher.
__global__ void __launch_bounds__(kEltThreads) fwd_epilogue_kernel(float* __restrict__ pre, const float* __restrict__ bias,
                                                                  const float* __restrict__ skip, int64_t k, int64_t q,
                                                                  int relu, int store_pre, float* __restrict__ act,
                                                                  uint16_t* __restrict__ act_bf16, int64_t pad,
                                                                  uint32_t* __restrict__ mask, bool vec) {
    const int64_t row = blockIdx.y;
    const int k32 = static_cast<int>(k), row32 = static_cast<int>(blockIdx.y);  // 32-bit (n*k <= 65535)
    const int item = row32 / k32, ch = row32 - item * k32;
    const int64_t x0 = static_cast<int64_t>(blockIdx.x) * kEltPerBlock + threadIdx.x * kEltPerThread;
    const bool live = x0 < q;
    const float b = bias ? bias[ch] : 0.0f;
    float* pr = pre + row * q + x0;
    const int cnt = live ? static_cast<int>(q - x0 < kEltPerThread ? q - x0 : kEltPerThread) : 0;
    const bool v4 = vec && cnt == kEltPerThread;
    float v[4] = {0.f, 0.f, 0.f, 0.f}, sk[4] = {0.f, 0.f, 0.f, 0.f};
    if (v4) {
        const float4 t = *reinterpret_cast<const float4*>(pr);
        v[0] = t.x, v[1] = t.y, v[2] = t.z, v[3] = t.w;
        if (skip) {
            const float4 s = *reinterpret_cast<const float4*>(skip + row * q + x0);
            sk[0] = s.x, sk[1] = s.y, sk[2] = s.z, sk[3] = s.w;
        }
    } else {
        for (int j = 0; j < 4; ++j) {
            v[j] = j < cnt ? pr[j] : 0.0f;
            if (skip && j < cnt) sk[j] = skip[row * q + x0 + j];
        }
    }
    float a[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        v[j] += b;
        a[j] = (relu && !(v[j] > 0.0f)) ? 0.0f : v[j];
        a[j] += sk[j];
    }
    if (!live) return;
    if (mask) {  // channel-block words (kernels.h): OR this row's bit into the 4 columns' words
        uint32_t* wd = mask + static_cast<int64_t>(item * ((k32 + 15) / 16) + ch / 16) * q + x0;
        const uint32_t bit = 1u << (ch % 16);
        for (int j = 0; j < cnt; ++j)
            if (v[j] > 0.0f) atomicOr(wd + j, bit);
    }
    if (v4) {
        if (bias && store_pre) *reinterpret_cast<float4*>(pr) = make_float4(v[0], v[1], v[2], v[3]);
        if (act) *reinterpret_cast<float4*>(act + row * q + x0) = make_float4(a[0], a[1], a[2], a[3]);
    } else {
        for (int j = 0; j < cnt; ++j) {
            if (bias && store_pre) pr[j] = v[j];
            if (act) act[row * q + x0 + j] = a[j];
        }
    }
    if (act_bf16) {
        uint16_t* dst = act_bf16 + row * (q + 2 * pad) + pad + x0;
        if (v4 && ((pad & 3) == 0)) {
            store_bf16x4(dst, a, true);
        } else {
            for (int j = 0; j < cnt; ++j) dst[j] = fp32_to_bf16_bits(a[j]);
        }
    }
}

// grid (nbx = ceil(q / 1024), n*k). Block partial of the bias gradient -> part[row * nbx + bx].
__global__ void __launch_bounds__(kEltThreads) bwd_prologue_kernel(
    const float* __restrict__ gin, int64_t gin_w, int64_t gin_off, const float* __restrict__ gadd,
    const float* __restrict__ pre, const float* __restrict__ pre_bias, const uint32_t* __restrict__ mask, int64_t k,
    int64_t q, int relu, float* __restrict__ gsum, float* __restrict__ grad_pre,
    uint16_t* __restrict__ grad_pre_bf16, float* __restrict__ part, bool vec, const float* __restrict__ pw_dy,
    const float* __restrict__ pw_w, int pw_k) {
    __shared__ float red[kEltThreads / 32];
    const int64_t row = blockIdx.y;
    // (item, channel) of the row in 32-bit math (the launcher bounds n*k by 65535): 64-bit divisions
    // per thread made this pass issue-bound (the heads' 1-tap backward: 298 us)
    const int k32 = static_cast<int>(k), row32 = static_cast<int>(blockIdx.y);
    const int item = row32 / k32, ch = row32 - item * k32;
    const int64_t x0 = static_cast<int64_t>(blockIdx.x) * kEltPerBlock + threadIdx.x * kEltPerThread;
    float gp[4] = {0.f, 0.f, 0.f, 0.f};
    if (x0 < q) {
        const int cnt = static_cast<int>(q - x0 < kEltPerThread ? q - x0 : kEltPerThread);
        const bool v4 = vec && cnt == kEltPerThread;
        const float* gi = gin + row * gin_w + gin_off + x0;
        float g[4], ad[4] = {0.f, 0.f, 0.f, 0.f}, pr[4] = {1.f, 1.f, 1.f, 1.f};
        if (pw_dy) {
            // gin = the 1-tap backward-data of pw_k filters computed here (the FP32 pointwise
            // conv's order: fmaf over the filters from 0), instead of read from a scratch tensor
#pragma unroll
            for (int j = 0; j < 4; ++j) g[j] = 0.0f;
            for (int f = 0; f < pw_k; ++f) {
                const float wv = __ldg(pw_w + f * k + ch);
                const float* src = pw_dy + static_cast<int64_t>(item * pw_k + f) * q + x0;
                float dv[4];
                if (v4) {  // q % 4 == 0 and 16-B aligned rows (launcher's vec flag)
                    const float4 t = __ldg(reinterpret_cast<const float4*>(src));
                    dv[0] = t.x, dv[1] = t.y, dv[2] = t.z, dv[3] = t.w;
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j) dv[j] = j < cnt ? __ldg(src + j) : 0.0f;
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) g[j] = fmaf(wv, dv[j], g[j]);
            }
            if (v4) {
                if (gadd) {
                    const float4 t = *reinterpret_cast<const float4*>(gadd + row * q + x0);
                    ad[0] = t.x, ad[1] = t.y, ad[2] = t.z, ad[3] = t.w;
                }
                if (relu && !mask) {
                    const float4 t = *reinterpret_cast<const float4*>(pre + row * q + x0);
                    pr[0] = t.x, pr[1] = t.y, pr[2] = t.z, pr[3] = t.w;
                }
            } else {
                if (gadd)
                    for (int j = 0; j < cnt; ++j) ad[j] = gadd[row * q + x0 + j];
                if (relu && !mask)
                    for (int j = 0; j < cnt; ++j) pr[j] = pre[row * q + x0 + j];
            }
        } else if (v4) {
            const float4 t = *reinterpret_cast<const float4*>(gi);
            g[0] = t.x, g[1] = t.y, g[2] = t.z, g[3] = t.w;
            if (gadd) {
                const float4 s = *reinterpret_cast<const float4*>(gadd + row * q + x0);
                ad[0] = s.x, ad[1] = s.y, ad[2] = s.z, ad[3] = s.w;
            }
            if (relu && !mask) {
                const float4 s = *reinterpret_cast<const float4*>(pre + row * q + x0);
                pr[0] = s.x, pr[1] = s.y, pr[2] = s.z, pr[3] = s.w;
            }
        } else {
            for (int j = 0; j < 4; ++j) {
                g[j] = j < cnt ? gi[j] : 0.0f;
                if (gadd && j < cnt) ad[j] = gadd[row * q + x0 + j];
                if (relu && !mask && j < cnt) pr[j] = pre[row * q + x0 + j];
            }
        }
        const float pb = (relu && pre_bias) ? pre_bias[ch] : 0.0f;  // mask of pre + bias
        // or the forward's mask words: bit c % 16 of word (n, c / 16, x)
        const uint32_t* mwd = mask ? mask + static_cast<int64_t>(item * ((k32 + 15) / 16) + ch / 16) * q + x0 : nullptr;
        const uint32_t mbit = 1u << (ch % 16);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            g[j] += ad[j];
            const bool keep = mask ? (j < cnt && (mwd[j] & mbit) != 0) : (pr[j] + pb > 0.0f);
            gp[j] = (relu && !keep) ? 0.0f : g[j];
            if (j >= cnt) gp[j] = 0.0f;
        }
        if (v4) {
            if (gsum) *reinterpret_cast<float4*>(gsum + row * q + x0) = make_float4(g[0], g[1], g[2], g[3]);
            if (grad_pre) *reinterpret_cast<float4*>(grad_pre + row * q + x0) = make_float4(gp[0], gp[1], gp[2], gp[3]);
            if (grad_pre_bf16) store_bf16x4(grad_pre_bf16 + row * q + x0, gp, true);
        } else {
            for (int j = 0; j < cnt; ++j) {
                if (gsum) gsum[row * q + x0 + j] = g[j];
                if (grad_pre) grad_pre[row * q + x0 + j] = gp[j];
                if (grad_pre_bf16) grad_pre_bf16[row * q + x0 + j] = fp32_to_bf16_bits(gp[j]);
            }
        }
    }
    if (!part) return;
    // fixed-shape tree: thread sum (j = 0..3), warp butterfly, then warps 0..7 in order
    float s = ((gp[0] + gp[1]) + (gp[2] + gp[3]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        float t = 0.0f;
        for (int w = 0; w < kEltThreads / 32; ++w) t += red[w];
        part[row * gridDim.x + blockIdx.x] = t;
    }
}

// The 1-tap glued backward-data of a few-filter layer (the network's heads) for all k <= KMAX
// channels of an item at once: block (bx, n) owns 1024 columns of item n, each thread 4 columns. The
// PWK filter rows of dy and the channel-block mask word are loaded once per column instead of once
// per channel row (bwd_prologue_kernel's one-row-per-block layout re-read them k times and spent its
// time on per-row index math: 256 us at batch 64 against ~55 us of HBM writes). Same arithmetic in
// the same order as bwd_prologue_kernel (fmaf over the filters from 0, + gadd, mask; the bias
// partial of a (row, block) is the same fixed tree), so the outputs are bit-identical.
// With pw_dy == nullptr the incoming gradient is read from gin (row pitch gin_w, offset gin_off)
// instead: the same per-item layout for any k <= KMAX (e.g. the heads' own bias gradient).
template <int KMAX, int PWK>
__global__ void __launch_bounds__(kEltThreads) pw_bwd_prologue_kernel(
    const float* __restrict__ gin, int64_t gin_w, int64_t gin_off,
    const float* __restrict__ pw_dy, const float* __restrict__ pw_w, int pw_k, const float* __restrict__ gadd,
    const uint32_t* __restrict__ mask, int k, int64_t q, float* __restrict__ gsum, float* __restrict__ grad_pre,
    uint16_t* __restrict__ grad_pre_bf16, float* __restrict__ part) {
    __shared__ float red[kEltThreads / 32][KMAX];
    const int n = blockIdx.y;
    const int64_t x0 = static_cast<int64_t>(blockIdx.x) * kEltPerBlock + threadIdx.x * kEltPerThread;
    const bool live = x0 < q;  // q % 4 == 0: a live thread owns 4 valid columns
    float dv[PWK][4];
#pragma unroll
    for (int f = 0; f < PWK; ++f) {
        float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
        if (pw_dy && live && f < pw_k) t = __ldg(reinterpret_cast<const float4*>(pw_dy + (static_cast<int64_t>(n) * pw_k + f) * q + x0));
        dv[f][0] = t.x, dv[f][1] = t.y, dv[f][2] = t.z, dv[f][3] = t.w;
    }
    uint4 mw = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
    if (mask && live) mw = __ldg(reinterpret_cast<const uint4*>(mask + static_cast<int64_t>(n) * q + x0));  // k <= 16: one word
    const uint32_t mws[4] = {mw.x, mw.y, mw.z, mw.w};
    float bs[KMAX];
#pragma unroll
    for (int c = 0; c < KMAX; ++c) {
        bs[c] = 0.0f;
        if (c >= k) continue;
        const int64_t row = static_cast<int64_t>(n) * k + c;
        float g[4] = {0.f, 0.f, 0.f, 0.f}, ad[4] = {0.f, 0.f, 0.f, 0.f}, gp[4];
        if (pw_dy) {
#pragma unroll
            for (int f = 0; f < PWK; ++f) {
                if (f >= pw_k) break;
                const float wv = __ldg(pw_w + f * k + c);
#pragma unroll
                for (int j = 0; j < 4; ++j) g[j] = fmaf(wv, dv[f][j], g[j]);
            }
        }
        if (!live) continue;
        if (!pw_dy) {
            const float4 t = __ldg(reinterpret_cast<const float4*>(gin + row * gin_w + gin_off + x0));
            g[0] = t.x, g[1] = t.y, g[2] = t.z, g[3] = t.w;
        }
        if (gadd) {
            const float4 t = *reinterpret_cast<const float4*>(gadd + row * q + x0);
            ad[0] = t.x, ad[1] = t.y, ad[2] = t.z, ad[3] = t.w;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            g[j] += ad[j];
            gp[j] = (mask && (mws[j] & (1u << c)) == 0) ? 0.0f : g[j];
        }
        if (gsum) *reinterpret_cast<float4*>(gsum + row * q + x0) = make_float4(g[0], g[1], g[2], g[3]);
        if (grad_pre) *reinterpret_cast<float4*>(grad_pre + row * q + x0) = make_float4(gp[0], gp[1], gp[2], gp[3]);
        if (grad_pre_bf16) store_bf16x4(grad_pre_bf16 + row * q + x0, gp, true);
        bs[c] = ((gp[0] + gp[1]) + (gp[2] + gp[3]));
    }
    if (!part) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int c = 0; c < KMAX; ++c) {
        if (c >= k) break;
        float t = bs[c];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0) red[warp][c] = t;
    }
    __syncthreads();
    if (threadIdx.x < k) {
        float t = 0.0f;
        for (int w = 0; w < kEltThreads / 32; ++w) t += red[w][threadIdx.x];
        part[(static_cast<int64_t>(n) * k + threadIdx.x) * gridDim.x + blockIdx.x] = t;
    }
}

// bias_grad[c] = sum of part[(item*k + c) * nbx + bx] over items and blocks; one CTA per channel,
// thread t sums the entries t, t+256, ... (items outer, blocks inner) in order, then a fixed tree.
__global__ void __launch_bounds__(kEltThreads) bias_grad_reduce_kernel(const float* __restrict__ part,
                                                                       float* __restrict__ bias_grad, int64_t n,
                                                                       int64_t k, int64_t nbx) {
    __shared__ float red[kEltThreads / 32];
    const int64_t c = blockIdx.x;
    const int64_t total = n * nbx;
    float t = 0.0f;
    // entries e = threadIdx.x, +256, ... in order; (i, b) = (e / nbx, e % nbx) advanced without divisions
    int64_t i = threadIdx.x / nbx, b = threadIdx.x - (threadIdx.x / nbx) * nbx;
    for (int64_t e = threadIdx.x; e < total; e += kEltThreads) {
        t += part[(i * k + c) * nbx + b];
        b += kEltThreads;
        while (b >= nbx) {
            b -= nbx;
            ++i;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
        float s = 0.0f;
        for (int w = 0; w < kEltThreads / 32; ++w) s += red[w];
        bias_grad[c] = s;
    }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

int64_t layer_bias_blocks(int64_t q) { return ceil_div(q, kEltPerBlock); }

cudaError_t launch_layer_fwd_epilogue(float* pre, const float* bias, const float* skip, int64_t n, int64_t k, int64_t q,
                                      int relu, int store_pre, float* act, uint16_t* act_bf16, int64_t pad,
                                      uint32_t* mask, cudaStream_t stream) {
    if (n * k == 0 || q == 0) return cudaSuccess;
    if (n * k > 65535) return cudaErrorInvalidValue;
    const bool vec = (q % 4 == 0) && aligned16(pre) && (!skip || aligned16(skip)) && (!act || aligned16(act));
    if (mask) {
        const cudaError_t e = cudaMemsetAsync(mask, 0, sizeof(uint32_t) * static_cast<size_t>(n * ceil_div(k, 16) * q), stream);
        if (e != cudaSuccess) return e;
    }
    const dim3 grid(static_cast<unsigned>(ceil_div(q, kEltPerBlock)), static_cast<unsigned>(n * k));
    fwd_epilogue_kernel<<<grid, kEltThreads, 0, stream>>>(pre, bias, skip, k, q, relu, store_pre, act, act_bf16, pad, mask,
                                                          vec && (!act_bf16 || ((reinterpret_cast<uintptr_t>(act_bf16) & 7u) == 0 &&
                                                                                ((q + 2 * pad) % 4) == 0)));
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_layer_bwd_prologue(const float* gin, int64_t gin_w, int64_t gin_off, const float* gadd,
                                      const float* pre, const float* pre_bias, const uint32_t* mask, int64_t n,
                                      int64_t k, int64_t q, int relu, float* gsum,
                                      float* grad_pre, uint16_t* grad_pre_bf16, float* bias_grad, float* part,
                                      cudaStream_t stream, const float* pw_dy, const float* pw_w, int pw_k) {
    if (n * k == 0 || q == 0) return cudaSuccess;
    if (n * k > 65535) return cudaErrorInvalidValue;
    const bool vec = (q % 4 == 0) && (gin_w % 4 == 0) && (gin_off % 4 == 0) && (pw_dy ? aligned16(pw_dy) : aligned16(gin)) &&
                     (!gadd || aligned16(gadd)) && (!pre || aligned16(pre)) && (!gsum || aligned16(gsum)) &&
                     (!grad_pre || aligned16(grad_pre)) &&
                     (!grad_pre_bf16 || (reinterpret_cast<uintptr_t>(grad_pre_bf16) & 7u) == 0);
    const int64_t nbx = layer_bias_blocks(q);
    // few channels per item (the heads): one block row per item, all channels per thread
    if (vec && k <= 16 && (!pw_dy || pw_k <= 2) && (relu == 0 || mask != nullptr) && (pw_dy || gin) &&
        (!mask || (reinterpret_cast<uintptr_t>(mask) & 15u) == 0) && n <= 65535) {
        const dim3 g2(static_cast<unsigned>(nbx), static_cast<unsigned>(n));
        const uint32_t* m = relu ? mask : nullptr;
        float* pt = bias_grad ? part : nullptr;
        if (pw_dy && pw_k == 2)
            pw_bwd_prologue_kernel<16, 2><<<g2, kEltThreads, 0, stream>>>(gin, gin_w, gin_off, pw_dy, pw_w, pw_k, gadd, m,
                                                                          static_cast<int>(k), q, gsum, grad_pre,
                                                                          grad_pre_bf16, pt);
        else
            pw_bwd_prologue_kernel<16, 1><<<g2, kEltThreads, 0, stream>>>(gin, gin_w, gin_off, pw_dy, pw_w, pw_k, gadd, m,
                                                                          static_cast<int>(k), q, gsum, grad_pre,
                                                                          grad_pre_bf16, pt);
        note_launch();
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess || !bias_grad) return e;
        return launch_bias_grad_reduce(part, bias_grad, n, k, nbx, stream);
    }
    const dim3 grid(static_cast<unsigned>(nbx), static_cast<unsigned>(n * k));
    bwd_prologue_kernel<<<grid, kEltThreads, 0, stream>>>(gin, gin_w, gin_off, gadd, pre, pre_bias, mask, k, q, relu, gsum,
                                                          grad_pre, grad_pre_bf16, bias_grad ? part : nullptr, vec,
                                                          pw_dy, pw_w, pw_k);
    note_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || !bias_grad) return e;
    return launch_bias_grad_reduce(part, bias_grad, n, k, nbx, stream);
}

cudaError_t launch_bias_grad_reduce(const float* part, float* bias_grad, int64_t n, int64_t k, int64_t nbx,
                                    cudaStream_t stream) {
    bias_grad_reduce_kernel<<<static_cast<unsigned>(k), kEltThreads, 0, stream>>>(part, bias_grad, n, k, nbx);
    note_launch();
    return cudaGetLastError();
}

}  // namespace c1d
