// train.cu — the training-step pieces around the conv layers:
//
//   c1d_fill_poisson / c1d_fill_bernoulli   seeded input samplers of BASELINE config 5
//   c1d_mse_bce_loss                        mse_loss + bce_with_logits, values and gradients in one
//                                           pass (proj/src/train.cpp:106-135)
//   c1d_sgd_update                          p <- p - lr*g over a flat bucket (train.cpp:137-141)
//
// All HBM-bound elementwise work: grid-stride loops over 16-B vectors, grids sized to the SM count.
#include <algorithm>
#include <cmath>

#include "../../include/c1d.h"
#include "common.cuh"
#include "kernels.h"

namespace c1d {
namespace {

// ---- counter-based sampler ------------------------------------------------------------------
// Element i draws from its own splitmix64 stream: state = splitmix64(seed ^ splitmix64(i)), each
// uniform = (next() >> 11) * 2^-53. Independent of the launch shape, so a batch is bitwise the
// same however it is split; oracle/conv1d_oracle.c (orc_sample_*) restates it for the tests.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
struct SplitMix {
    uint64_t s;
    __device__ __forceinline__ double next_double() {
        s += 0x9E3779B97F4A7C15ull;
        return static_cast<double>(mix64(s) >> 11) * 0x1.0p-53;
    }
};
__device__ __forceinline__ SplitMix stream_of(uint64_t seed, uint64_t i) {
    return SplitMix{mix64(seed ^ mix64(i + 0x9E3779B97F4A7C15ull))};
}

// Knuth's product-of-uniforms Poisson draw: the smallest k with u_0 * ... * u_k <= exp(-lambda)
// (limit = exp(-lambda) is computed once on the host so device and oracle compare the same double).
__global__ void poisson_kernel(float* out, int64_t count, double limit, uint64_t seed) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x) {
        SplitMix r = stream_of(seed, static_cast<uint64_t>(i));
        double prod = r.next_double();
        uint32_t k = 0;
        while (prod > limit) {
            ++k;
            prod = __dmul_rn(prod, r.next_double());
        }
        out[i] = static_cast<float>(k);
    }
}

__global__ void bernoulli_kernel(float* out, int64_t count, double p, uint64_t seed) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x) {
        SplitMix r = stream_of(seed, static_cast<uint64_t>(i));
        out[i] = r.next_double() < p ? 1.0f : 0.0f;
    }
}

// ---- losses ---------------------------------------------------------------------------------
// Stable forms of train.cpp:39-46 (stable_softplus, stable_sigmoid), evaluated in double.

constexpr int kLossThreads = 256;

// One pass over (item, column): the MSE and BCE terms are summed in double per thread (columns in
// ascending order within the thread's fixed slice), then per block in a fixed tree; block partials
// go to `part` and the last block to finish sums them in block order (a ticket counter decides
// who, not the order), so the loss is deterministic. Gradients use the reference's formulas in
// double and round once: 2*diff/count, (sigmoid(l) - m)/count, then * bce_weight in float.
__global__ void __launch_bounds__(kLossThreads) mse_bce_kernel(
    const float* __restrict__ pred, const float* __restrict__ logits, int64_t in_stride,
    const float* __restrict__ target, const float* __restrict__ labels, int64_t n, int64_t width, float bce_weight,
    float* __restrict__ grad_pred, float* __restrict__ grad_logits, int64_t grad_stride, double* __restrict__ part) {
    const int64_t count = n * width;
    const double inv = 1.0 / static_cast<double>(count);
    const int64_t per = (count + gridDim.x - 1) / gridDim.x;
    const int64_t b0 = blockIdx.x * per, b1 = min(count, b0 + per);
    double mse = 0.0, bce = 0.0;
    // (item, column) of this thread's first element; then advanced without divisions
    int64_t e = b0 + threadIdx.x;
    int64_t i = e / width, x = e - i * width;
    for (; e < b1; e += kLossThreads) {
        const double p = pred[i * in_stride + x], t = target[e];
        const double diff = p - t;
        mse += diff * diff;
        const double l = logits[i * in_stride + x], m = labels[e];
        // one exp serves both stable forms: t = exp(-|l|); softplus = max(l, 0) + log1p(t),
        // sigmoid = l >= 0 ? 1/(1+t) : t/(1+t) -- the same operations the reference's branches do
        const double tl = exp(-fabs(l));
        bce += ((l > 0.0 ? l : 0.0) + log1p(tl)) - m * l;
        if (grad_pred) grad_pred[i * grad_stride + x] = static_cast<float>(2.0 * diff * inv);
        if (grad_logits) {
            const double sg = l >= 0.0 ? 1.0 / (1.0 + tl) : tl / (1.0 + tl);
            grad_logits[i * grad_stride + x] = __fmul_rn(bce_weight, static_cast<float>((sg - m) * inv));
        }
        x += kLossThreads;
        while (x >= width) {
            x -= width;
            ++i;
        }
    }
    __shared__ double sm[2][kLossThreads];
    sm[0][threadIdx.x] = mse;
    sm[1][threadIdx.x] = bce;
    __syncthreads();
    for (int h = kLossThreads / 2; h > 0; h >>= 1) {
        if (threadIdx.x < h) {
            sm[0][threadIdx.x] += sm[0][threadIdx.x + h];
            sm[1][threadIdx.x] += sm[1][threadIdx.x + h];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = sm[0][0];
        part[2 * blockIdx.x + 1] = sm[1][0];
    }
}

// The block partials summed in a fixed shape (thread t takes partials t, t + 256, ... in order, then
// a tree), so the loss is deterministic. A second launch instead of a last-block ticket: the ticket
// needed a per-call memset node, which cost ~14 us in the graph-replayed network step.
__global__ void __launch_bounds__(kLossThreads) mse_bce_final_kernel(const double* __restrict__ part, int nblocks,
                                                                     int64_t count, float bce_weight,
                                                                     double* __restrict__ loss3) {
    __shared__ double sm[2][kLossThreads];
    const double inv = 1.0 / static_cast<double>(count);
    double a = 0.0, b = 0.0;
    for (int j = threadIdx.x; j < nblocks; j += kLossThreads) {
        a += part[2 * j];
        b += part[2 * j + 1];
    }
    sm[0][threadIdx.x] = a;
    sm[1][threadIdx.x] = b;
    __syncthreads();
    for (int h = kLossThreads / 2; h > 0; h >>= 1) {
        if (threadIdx.x < h) {
            sm[0][threadIdx.x] += sm[0][threadIdx.x + h];
            sm[1][threadIdx.x] += sm[1][threadIdx.x + h];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double ta = sm[0][0], tb = sm[1][0];
        loss3[0] = ta * inv;
        loss3[1] = tb * inv;
        loss3[2] = ta * inv + static_cast<double>(bce_weight) * (tb * inv);
    }
}

// p <- p - lr*g with the reference's float rounding (one multiply, one subtract, no FMA).
__global__ void sgd_kernel(float* __restrict__ p, const float* __restrict__ g, int64_t count, float lr) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    const int64_t i0 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    const int64_t nv = (reinterpret_cast<uintptr_t>(p) % 16 == 0 && reinterpret_cast<uintptr_t>(g) % 16 == 0) ? count / 4 : 0;
    for (int64_t v = i0; v < nv; v += stride) {
        float4 a = reinterpret_cast<float4*>(p)[v];
        const float4 b = reinterpret_cast<const float4*>(g)[v];
        a.x = __fsub_rn(a.x, __fmul_rn(lr, b.x));
        a.y = __fsub_rn(a.y, __fmul_rn(lr, b.y));
        a.z = __fsub_rn(a.z, __fmul_rn(lr, b.z));
        a.w = __fsub_rn(a.w, __fmul_rn(lr, b.w));
        reinterpret_cast<float4*>(p)[v] = a;
    }
    for (int64_t i = 4 * nv + i0; i < count; i += stride) p[i] = __fsub_rn(p[i], __fmul_rn(lr, g[i]));
}

int grid_for(int64_t count, int threads) {
    const int64_t want = (count + threads - 1) / threads;
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, 8 * num_sms())));
}

c1d_status bad(const char* what) {
    set_last_error(what);
    return C1D_ERR_INVALID_ARGUMENT;
}

}  // namespace

size_t loss_workspace_bytes() { return 2 * sizeof(double) * 2 * 1024 + 256; }

}  // namespace c1d

using namespace c1d;

extern "C" {

c1d_status c1d_fill_poisson(float* out, int64_t count, double lambda, uint64_t seed, c1d_stream_t stream) {
    if (count < 0 || (count > 0 && !out) || !(lambda > 0.0)) return bad("bad fill_poisson arguments");
    if (count == 0) return C1D_OK;
    poisson_kernel<<<grid_for(count, 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(out, count, std::exp(-lambda),
                                                                                             seed);
    note_launch(1);
    return cudaGetLastError() == cudaSuccess ? C1D_OK : C1D_ERR_CUDA;
}

c1d_status c1d_fill_bernoulli(float* out, int64_t count, double p, uint64_t seed, c1d_stream_t stream) {
    if (count < 0 || (count > 0 && !out) || !(p >= 0.0 && p <= 1.0)) return bad("bad fill_bernoulli arguments");
    if (count == 0) return C1D_OK;
    bernoulli_kernel<<<grid_for(count, 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(out, count, p, seed);
    note_launch(1);
    return cudaGetLastError() == cudaSuccess ? C1D_OK : C1D_ERR_CUDA;
}

size_t c1d_loss_workspace_size(void) { return loss_workspace_bytes(); }

c1d_status c1d_mse_bce_loss(const float* pred, const float* logits, int64_t in_stride, const float* target,
                            const float* labels, int64_t n, int64_t width, float bce_weight, float* grad_pred,
                            float* grad_logits, int64_t grad_stride, double* loss3, void* workspace,
                            size_t workspace_bytes, c1d_stream_t stream) {
    if (n <= 0 || width <= 0 || !pred || !logits || !target || !labels || !loss3 || in_stride < width ||
        ((grad_pred || grad_logits) && grad_stride < width))
        return bad("bad mse_bce_loss arguments");
    if (!workspace || workspace_bytes < loss_workspace_bytes()) {
        set_last_error("mse_bce_loss needs c1d_loss_workspace_size() bytes of workspace");
        return C1D_ERR_WORKSPACE;
    }
    const int64_t count = n * width;
    const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(1024, (count + 4095) / 4096)));
    double* part = static_cast<double*>(workspace);
    mse_bce_kernel<<<blocks, kLossThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        pred, logits, in_stride, target, labels, n, width, bce_weight, grad_pred, grad_logits, grad_stride, part);
    mse_bce_final_kernel<<<1, kLossThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(part, blocks, count,
                                                                                      bce_weight, loss3);
    note_launch(2);
    return cudaGetLastError() == cudaSuccess ? C1D_OK : C1D_ERR_CUDA;
}

c1d_status c1d_sgd_update(float* params, const float* grads, int64_t count, float lr, c1d_stream_t stream) {
    if (count < 0 || (count > 0 && (!params || !grads))) return bad("bad sgd_update arguments");
    if (!(lr > 0.0f)) return bad("sgd_step needs a positive learning rate");  // train.cpp:139
    if (count == 0) return C1D_OK;
    sgd_kernel<<<grid_for(count / 4 + 1, 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(params, grads, count, lr);
    note_launch(1);
    return cudaGetLastError() == cudaSuccess ? C1D_OK : C1D_ERR_CUDA;
}

}  // extern "C"
