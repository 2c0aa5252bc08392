/*
 * c1d.h — C ABI of the B200-native 1D dilated convolution layer (arXiv 2104.08002 hot path).
 *
 * Drop-in boundary for the reference's operator API (namespace conv1d in
 * /root/reference/proj/include/conv1d/conv.hpp). The reference has no FFI of its own: its three
 * pass entry points are C++ free functions over host std::vector tensors. This header replaces
 * them with plain-pointer, device-memory entry points; paper_2104_08002_b200/host/conv1d_gpu.cpp
 * re-implements the exact reference C++ signatures on top of it.
 *
 *   c1d_forward          replaces conv1d::conv1d_forward          conv.hpp:42-43, conv.cpp:165-191
 *   c1d_backward_data    replaces conv1d::conv1d_backward_data    conv.hpp:49-50, conv.cpp:193-227
 *   c1d_backward_weight  replaces conv1d::conv1d_backward_weight  conv.hpp:56-57, conv.cpp:229-326
 *   c1d_output_width     replaces conv1d::output_width            conv.hpp:33,   conv.cpp:142-151
 *   c1d_conv_flops       replaces conv1d::conv_flops              conv.hpp:37,   conv.cpp:161-163
 *   c1d_round_bf16       replaces conv1d::fp32_to_bf16 over spans bf16.hpp:29-40, conv.cpp:69-73
 *
 * Conventions
 *   - Tensors are NCW with the width axis contiguous (tensor.hpp:13-36): x is (N, C, W_in),
 *     y / dy is (N, K, Q) with Q = W_in - d*(S-1), dx is (N, C, W_in).
 *   - Weights are passed in the natural (K, C, S) order (WeightKCS, tensor.hpp:42-56) as FP32;
 *     the per-pass packing (pack_weights_forward/backward, tensor.cpp:5-41) happens on the device.
 *     dW is returned in KCS order, FP32.
 *   - All tensor pointers are DEVICE pointers. Outputs are always FP32 (as in the reference).
 *   - x / dy storage is FP32 or BF16 (desc.in_dtype). With precision BF16 and FP32 storage the
 *     inputs and weights are rounded to BF16 (round-to-nearest-even) inside the call, exactly as
 *     the reference does (conv.cpp:182-183, 218-219, 248-249); products accumulate in FP32.
 *   - Errors are status codes, one per reference exception class used on this path
 *     (errors.hpp:8-64); nothing is thrown across the ABI. Validation happens before any launch.
 *     c1d_last_error_message() returns the human-readable detail for the calling thread.
 *   - Calls are asynchronous on `stream` and reentrant on disjoint outputs. Results are
 *     bitwise deterministic run to run (no atomics; fixed-order reductions).
 *   - Deviation from the reference: BF16 accepts odd C, K and widths (channels are zero-padded
 *     to tensor-core tile shapes). Set C1D_FLAG_STRICT_BF16_DIMS to get the reference's OddDims
 *     rejection (conv.cpp:40-57) instead.
 */
#ifndef C1D_H_
#define C1D_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define C1D_API_VERSION 1

#if defined(__GNUC__)
#define C1D_EXPORT __attribute__((visibility("default")))
#else
#define C1D_EXPORT
#endif

typedef struct CUstream_st* c1d_stream_t; /* == cudaStream_t; NULL = legacy default stream */

typedef enum c1d_status {
    C1D_OK = 0,
    C1D_ERR_SHAPE_MISMATCH = 1, /* conv1d::ShapeMismatch */
    C1D_ERR_ODD_DIMS = 2,       /* conv1d::OddDims (only with C1D_FLAG_STRICT_BF16_DIMS) */
    C1D_ERR_TOO_NARROW = 3,     /* conv1d::TooNarrow */
    C1D_ERR_INVALID_ARGUMENT = 4,
    C1D_ERR_WORKSPACE = 5,   /* caller workspace too small */
    C1D_ERR_UNSUPPORTED = 6, /* requested algo cannot run this shape */
    C1D_ERR_CUDA = 7,        /* CUDA runtime / launch failure */
    C1D_ERR_NO_DEVICE = 8    /* no sm_100 device visible */
} c1d_status;

typedef enum c1d_precision { C1D_PRECISION_FP32 = 0, C1D_PRECISION_BF16 = 1 } c1d_precision;
typedef enum c1d_dtype { C1D_DTYPE_F32 = 0, C1D_DTYPE_BF16 = 1 } c1d_dtype;

/* Kernel family. AUTO picks the tcgen05 tensor-core kernels whenever the shape allows them and
 * the direct (FFMA) kernels otherwise. */
typedef enum c1d_algo {
    C1D_ALGO_AUTO = 0,
    C1D_ALGO_DIRECT = 1,  /* CUDA-core FFMA direct convolution, any shape */
    C1D_ALGO_TCGEN05 = 2, /* tcgen05.mma BF16 tensor-core kernels (TMEM accumulators) */
    C1D_ALGO_BF16X3 = 3   /* FP32 precision on the tcgen05 kernels: operands split into bf16 hi+lo
                             parts, v = hi + lo; the hi*hi, hi*lo, lo*hi and lo*lo partial
                             products accumulate in FP32 in TMEM (4 BF16 products per term) */
} c1d_algo;

typedef enum c1d_pass { C1D_PASS_FORWARD = 0, C1D_PASS_BACKWARD_DATA = 1, C1D_PASS_BACKWARD_WEIGHT = 2 } c1d_pass;

#define C1D_FLAG_STRICT_BF16_DIMS 0x1u
/* Accumulation accuracy. The tensor cores accumulate FP32 into TMEM with a consistent shrink toward
 * zero of ~1.2e-9 (norm-relative) per accumulated product, so one accumulator over a long reduction
 * drifts: BASELINE config 3 backward-weight sums 1.92M products per dW entry, and a single chain per
 * CTA (52k products) lands at ~6e-5 from the FP32-on-rounded result, inside the reference's BF16
 * bound (1e-2, acceptance.cpp:526) but not its FP32 one (1e-5). With this flag every chain is capped
 * at ~4096 products (backward-weight restarts its accumulators and sums the segments in a fixed
 * order; conv-shaped passes with C_in*S > 4096 split their channels over two TMEM regions): ~4e-6
 * at config 3, at some cost in time (config-3 backward-weight ~+45%). FP32 precision always runs
 * this way. */
#define C1D_FLAG_EXACT_ACCUM 0x2u
/* The weight pointer of c1d_forward / c1d_backward_data (and the glued variants) is a weight image
 * made by c1d_pack_weights for this desc and pass, not KCS weights. The call skips its own packing
 * launch and loads the image while the previous kernel on the stream is still running, so the image
 * must be complete before that kernel is launched (pack earlier than the kernel right before the
 * call; c1d_pack_weights itself never lets its successor start early). Only plans with at most 32
 * filters per group on the dilation-8 tensor-core path take images (c1d_packed_weights_size). */
#define C1D_FLAG_PREPACKED_WEIGHTS 0x4u

/* Mirrors conv1d::ConvParams (conv.hpp:18-25) plus the tensor sizes the reference reads from
 * its Tensor3D arguments. */
typedef struct c1d_desc {
    int64_t n;         /* batch */
    int64_t c;         /* input channels */
    int64_t k;         /* filters */
    int64_t s;         /* taps */
    int64_t d;         /* dilation */
    int64_t w_in;      /* pre-padded input width W_in; Q = W_in - d*(S-1) */
    int32_t precision; /* c1d_precision */
    int32_t in_dtype;  /* c1d_dtype of x and dy */
    int32_t algo;      /* c1d_algo */
    uint32_t flags;    /* C1D_FLAG_* */
    int64_t block_w;   /* accepted for API parity; results do not depend on it */
} c1d_desc;

C1D_EXPORT int c1d_api_version(void);
C1D_EXPORT const char* c1d_strerror(c1d_status status);
/* Detail text of the last failing call on this host thread ("" if none). */
C1D_EXPORT const char* c1d_last_error_message(void);

/* Q = W_in - d*(S-1); C1D_ERR_TOO_NARROW when W_in <= d*(S-1). */
C1D_EXPORT c1d_status c1d_output_width(const c1d_desc* desc, int64_t* q_out);
/* 2*N*K*C*S*Q, counted identically for all three passes. -1 on invalid desc. */
C1D_EXPORT int64_t c1d_conv_flops(const c1d_desc* desc);

/* Device workspace bytes the pass needs (0 if none). Passing workspace == NULL to a pass makes
 * the library use an internal, lazily grown buffer per (device, stream) instead: calls on different
 * streams never share it. An outgrown buffer is retired, never freed behind the caller's back
 * (CUDA graphs captured on that stream keep its address), and growing never synchronises, so it
 * is legal under stream capture. c1d_release_workspace frees them. */
C1D_EXPORT c1d_status c1d_workspace_size(const c1d_desc* desc, c1d_pass pass, size_t* bytes);

/* Frees the internal workspace buffers (current and retired) of `stream` on the current device,
 * after synchronising the stream. Call it when a stream is destroyed, and only once no captured
 * CUDA graph that used the stream's internal workspace will be replayed again. */
C1D_EXPORT c1d_status c1d_release_workspace(c1d_stream_t stream);

/* Which kernel family the pass will run for this desc (resolves C1D_ALGO_AUTO). */
C1D_EXPORT c1d_status c1d_selected_algo(const c1d_desc* desc, c1d_pass pass, c1d_algo* algo);

/* y (N,K,Q) = conv(x (N,C,W_in), w (K,C,S)) */
C1D_EXPORT c1d_status c1d_forward(const c1d_desc* desc, const void* x, const float* w_kcs, float* y, void* workspace,
                       size_t workspace_bytes, c1d_stream_t stream);

/* dx (N,C,W_in) = gradient w.r.t. the padded input, from dy (N,K,Q) */
C1D_EXPORT c1d_status c1d_backward_data(const c1d_desc* desc, const void* dy, const float* w_kcs, float* dx,
                             void* workspace, size_t workspace_bytes, c1d_stream_t stream);

/* dw (K,C,S) = sum_n sum_q x(n,c,q+d*s) dy(n,k,q) */
C1D_EXPORT c1d_status c1d_backward_weight(const c1d_desc* desc, const void* x, const void* dy, float* dw_kcs,
                               void* workspace, size_t workspace_bytes, c1d_stream_t stream);

/* out[i] = bf16 bits of in[i], round-to-nearest-even, NaN -> quiet NaN (bf16.hpp:29-40). */
/* Size of the weight image of (desc, pass) for C1D_FLAG_PREPACKED_WEIGHTS; C1D_ERR_UNSUPPORTED
 * when that pass's plan packs its own weights. */
C1D_EXPORT c1d_status c1d_packed_weights_size(const c1d_desc* desc, c1d_pass pass, size_t* bytes);
/* Pack `count` images in one launch (several when count > 32): image i from the KCS weights w[i] of
 * descs[i] for passes[i] (C1D_PASS_FORWARD or C1D_PASS_BACKWARD_DATA; backward-data images are the
 * transposed, tap-reversed filters, as c1d_backward_data packs them). */
C1D_EXPORT c1d_status c1d_pack_weights(int count, const c1d_desc* descs, const int32_t* passes,
                                       const float* const* w, void* const* images, c1d_stream_t stream);
C1D_EXPORT c1d_status c1d_round_bf16(const float* in, uint16_t* out, int64_t count, c1d_stream_t stream);

/* ---- Fused layer glue of the reference's ConvLayer (train.cpp:173-221) ----
 * Rows are the N*K (item, channel) pairs of a (N, K, Q) activation; fp32 unless stated.
 *
 * Forward epilogue, after the conv wrote pre (N, K, Q):
 *   v = pre + bias[k] (bias optional); stored back into pre only if store_pre   train.cpp:177-178
 *   a = relu ? max(v, 0) : v; a += skip (optional)                              train.cpp:179-192
 *   act      (optional, (N, K, Q))          = a
 *   act_bf16 (optional, (N, K, Q + 2*pad))  interior [pad, pad+Q) = RNE bf16(a); the 2*pad border
 *            columns are never written (keep them zero: the next layer's same padding)
 */
C1D_EXPORT c1d_status c1d_layer_forward_epilogue(float* pre, const float* bias, const float* skip, int64_t n,
                                                 int64_t k, int64_t q, int relu, int store_pre, float* act,
                                                 uint16_t* act_bf16, int64_t pad, c1d_stream_t stream);
/* Backward prologue:
 *   g  = gin[row * gin_w + gin_off + x] + gadd[row * Q + x] (gadd optional): the incoming gradient,
 *        e.g. the interior of a padded backward-data output plus a skip gradient
 *   gsum (optional) = g;  gp = relu ? (pre + pre_bias[k] > 0 ? g : 0) : g  (pre_bias optional:
 *   the bias the forward epilogue added without storing it)      train.cpp:205-210
 *   grad_pre (optional fp32) = gp;  grad_pre_bf16 (optional) = RNE bf16(gp)
 *   bias_grad (optional, K floats) = sum over items and columns of gp, fixed-order (deterministic)
 * workspace: c1d_layer_backward_workspace(n, k, q) bytes, or NULL for the internal buffer. */
C1D_EXPORT size_t c1d_layer_backward_workspace(int64_t n, int64_t k, int64_t q);
C1D_EXPORT c1d_status c1d_layer_backward_prologue(const float* gin, int64_t gin_w, int64_t gin_off, const float* gadd,
                                                  const float* pre, const float* pre_bias, int64_t n, int64_t k,
                                                  int64_t q, int relu,
                                                  float* gsum, float* grad_pre, uint16_t* grad_pre_bf16,
                                                  float* bias_grad, void* workspace, size_t workspace_bytes,
                                                  c1d_stream_t stream);

/* ---- Layer-glued conv passes: the conv and the ConvLayer glue in one call ----
 * On the tcgen05 path (dilation 8 and the d < 8 phase rewrite) the glue runs inside the conv's
 * TMEM -> global epilogue, so the FP32 conv output never reaches HBM; elsewhere the call runs the
 * conv into workspace scratch followed by one glue pass (same results up to the bias-gradient
 * summation order; both orders are fixed, so every call is deterministic). ReLU masks are
 * channel-block words: an (N, ceil(K/16), width) uint32 tensor whose word (n, b, x) holds the bits of
 * channels 16b .. 16b+15 at column x (bit j = channel 16b + j; bits 16-31 zero). BF16 outputs use
 * the reference's round-to-nearest-even for every non-NaN value; a NaN becomes the canonical bf16
 * NaN (its payload is not kept).
 *
 * Forward (train.cpp:176-192) on y = conv(x, w):
 *   v = y + bias[k];  mask bit = (v > 0);  a = relu ? (v > 0 ? v : 0) : v;  a += skip
 *   pre = v, act = a, act_bf16[(n*K + k)*(Q + 2*act_pad) + act_pad + q] = RNE bf16(a)
 *   (every output optional; the 2*act_pad border columns of act_bf16 are never written)   */
typedef struct c1d_fwd_glue {
    const float* bias;  /* (K) or NULL */
    const float* skip;  /* (N, K, Q) added after the ReLU, or NULL */
    float* pre;         /* (N, K, Q) conv + bias, or NULL */
    float* act;         /* (N, K, Q) activation, or NULL */
    uint16_t* act_bf16; /* (N, K, Q + 2*act_pad) zero-bordered bf16 activation, or NULL */
    uint32_t* mask;     /* (N, ceil(K/16), Q) ReLU mask words, or NULL */
    int64_t act_pad;
    int32_t relu;
    int32_t reserved; /* 0 */
} c1d_fwd_glue;
/* Backward (train.cpp:205-221) on dx = backward_data(dy, w), (N, C, W_in): the glued layer (the one
 * whose activation fed this conv) owns columns [off, off + q) of dx:
 *   g = dx[:, :, off + x] + gadd;  gp = mask ? (bit x ? g : 0) : g   (mask NULL = no ReLU)
 *   gsum = g, grad_pre = gp, grad_pre_bf16 = RNE bf16(gp)  ((N, C, q) each, optional)
 *   bias_grad (C floats, optional) = sum of gp over items and columns, fixed order   */
typedef struct c1d_bwd_glue {
    int64_t off, q;
    const float* gadd;     /* (N, C, q) or NULL */
    const uint32_t* mask;  /* (N, ceil(C/16), q) words from the glued layer's forward, or NULL */
    float* gsum;
    float* grad_pre;
    uint16_t* grad_pre_bf16;
    float* bias_grad;
} c1d_bwd_glue;
/* Workspace for a glued pass (glue_q = the backward window q; ignored for the forward) and whether
 * the glue runs fused in the conv epilogue (*fused = 1) or as a separate pass (0). */
C1D_EXPORT c1d_status c1d_glued_workspace_size(const c1d_desc* desc, c1d_pass pass, int64_t glue_q, size_t* bytes,
                                               int* fused);
C1D_EXPORT c1d_status c1d_forward_glued(const c1d_desc* desc, const void* x, const float* w_kcs,
                                        const c1d_fwd_glue* glue, void* workspace, size_t workspace_bytes,
                                        c1d_stream_t stream);
C1D_EXPORT c1d_status c1d_backward_data_glued(const c1d_desc* desc, const void* dy, const float* w_kcs,
                                              const c1d_bwd_glue* glue, void* workspace, size_t workspace_bytes,
                                              c1d_stream_t stream);
/* ---- The training step around the conv layers (BASELINE config 5) ----
 * Seeded input samplers (new: the reference's Rng has none). Element i draws from its own
 * splitmix64 stream (state = mix64(seed ^ mix64(i + golden)), uniform = (next >> 11) * 2^-53), so
 * the values do not depend on the launch shape or on how a batch is split:
 *   Poisson(lambda): Knuth's product of uniforms, the smallest k with u_0*...*u_k <= exp(-lambda)
 *   Bernoulli(p):    1 if u < p else 0                                                     */
C1D_EXPORT c1d_status c1d_fill_poisson(float* out, int64_t count, double lambda, uint64_t seed, c1d_stream_t stream);
C1D_EXPORT c1d_status c1d_fill_bernoulli(float* out, int64_t count, double p, uint64_t seed, c1d_stream_t stream);
/* mse_loss + bce_with_logits (train.cpp:106-135) in one pass over n items x width columns:
 *   pred(i, x) = pred[i*in_stride + x], logits likewise; target / labels contiguous (n, width)
 *   loss3[0] = mean((pred - target)^2), loss3[1] = mean(softplus(l) - m*l) (stable form),
 *   loss3[2] = loss3[0] + bce_weight * loss3[1]      (double, on the device; deterministic)
 *   grad_pred(i, x)   = float(2*(pred - target)/count)                 (optional)
 *   grad_logits(i, x) = bce_weight * float((sigmoid(l) - m)/count)    (optional; stride grad_stride)
 * workspace: c1d_loss_workspace_size() bytes, not shared by concurrent calls. */
C1D_EXPORT size_t c1d_loss_workspace_size(void);
C1D_EXPORT c1d_status c1d_mse_bce_loss(const float* pred, const float* logits, int64_t in_stride, const float* target,
                                       const float* labels, int64_t n, int64_t width, float bce_weight,
                                       float* grad_pred, float* grad_logits, int64_t grad_stride, double* loss3,
                                       void* workspace, size_t workspace_bytes, c1d_stream_t stream);
/* params[i] -= lr * grads[i] in float (sgd_step, train.cpp:137-141); lr must be positive. */
C1D_EXPORT c1d_status c1d_sgd_update(float* params, const float* grads, int64_t count, float lr, c1d_stream_t stream);

/* Number of kernels this library has launched since load (instrumentation for benchmarks). */
C1D_EXPORT uint64_t c1d_launch_count(void);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* C1D_H_ */
