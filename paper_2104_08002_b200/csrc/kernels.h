// kernels.h — internal launch interface between the C ABI (c1d_api.cu) and the kernels.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace c1d {

// Count of kernels this library launched (c1d_launch_count()).
void note_launch(int n = 1);

// Generic "forward-shaped" convolution:
//   out[n][o][x] = sum_i sum_s wg[o][i][s] * in[n][i][x + s*dil + in_off]   (0 outside [0,in_w))
// forward:       in = x  (C ch, W_in), out = y  (K ch, Q),    wg = W (KCS),   in_off = 0
// backward-data: in = dy (K ch, Q),    out = dx (C ch, W_in), wg = W' (CKS, taps reversed),
//                in_off = -d*(S-1)  (the reference's zero_pad_width, conv.cpp:206-208, done
//                as predicated loads instead of a padded copy)
struct ConvGeom {
    int64_t n, in_ch, in_w, out_ch, out_w, taps, dil, in_off;
};

enum WeightMode { kWeightsForward = 0, kWeightsBackwardData = 1 };

// out (o, i, s) fp32 from w_kcs; mode 1 transposes to (C, K, S) with the tap axis reversed
// (pack_weights_backward, tensor.cpp:23-41). round -> BF16 round-to-nearest-even.
cudaError_t launch_prep_weights(const float* w_kcs, float* out, int64_t K, int64_t C, int64_t S, int mode,
                                bool round, cudaStream_t stream);

// in_dtype: 0 = f32, 1 = bf16 bits. round_in: round FP32 inputs to BF16 on load.
cudaError_t launch_direct_conv(const void* in, int in_dtype, bool round_in, const float* wg, float* out,
                               const ConvGeom& g, cudaStream_t stream);

size_t direct_wgrad_workspace_bytes(int64_t n, int64_t c, int64_t k, int64_t s, int64_t q);
cudaError_t launch_direct_wgrad(const void* x, const void* dy, int in_dtype, bool round_in, float* dw_kcs,
                                float* workspace, int64_t n, int64_t c, int64_t k, int64_t s, int64_t d,
                                int64_t q, cudaStream_t stream);

cudaError_t launch_round_bf16(const float* in, uint16_t* out, int64_t count, cudaStream_t stream);

// layer.cu: fused ConvLayer glue (train.cpp:173-221)
int64_t layer_bias_blocks(int64_t q);  // bias-gradient partials per (item, channel) row
cudaError_t launch_layer_fwd_epilogue(float* pre, const float* bias, const float* skip, int64_t n, int64_t k, int64_t q,
                                      int relu, int store_pre, float* act, uint16_t* act_bf16, int64_t pad,
                                      cudaStream_t stream);
cudaError_t launch_layer_bwd_prologue(const float* gin, int64_t gin_w, int64_t gin_off, const float* gadd,
                                      const float* pre, const float* pre_bias, int64_t n, int64_t k, int64_t q,
                                      int relu, float* gsum,
                                      float* grad_pre, uint16_t* grad_pre_bf16, float* bias_grad, float* part,
                                      cudaStream_t stream);

// ---- tcgen05 (sm_100a) kernels -----------------------------------------------------------
// Row-tap BF16 tensor-core convolution for dilation 8 (fwd and bwd-data). Returns
// cudaErrorNotSupported when the shape is outside its envelope.
struct TcConvPlan;
// main_ch > 0 (split-FP32 mode): input channels >= main_ch accumulate into a second TMEM region
// that the epilogue adds to the first, so the long accumulation chain only carries the main term.
bool tc_conv_supported(const ConvGeom& g, int64_t main_ch = 0);
size_t tc_conv_workspace_bytes(const ConvGeom& g, int64_t main_ch = 0);
cudaError_t launch_tc_conv(const uint16_t* in_bf16, const float* wg, float* out, const ConvGeom& g,
                           void* workspace, cudaStream_t stream, int64_t main_ch = 0);

bool tc_wgrad_supported(int64_t n, int64_t c, int64_t k, int64_t s, int64_t d, int64_t q);
size_t tc_wgrad_workspace_bytes(int64_t n, int64_t c, int64_t k, int64_t s, int64_t d, int64_t q);
cudaError_t launch_tc_wgrad(const uint16_t* x_bf16, const uint16_t* dy_bf16, float* dw_kcs, void* workspace,
                            int64_t n, int64_t c, int64_t k, int64_t s, int64_t d, int64_t q, cudaStream_t stream);

// FP32-on-tensor-core operand splitting (split.cu)
cudaError_t launch_split_channels(const float* in, uint16_t* out, int64_t n, int64_t c, int64_t w, int reps,
                                  unsigned pattern, cudaStream_t stream);
cudaError_t launch_split_weights(const float* w, float* out, int64_t K, int64_t C, int64_t S, int kr, int cr,
                                 unsigned sel, cudaStream_t stream);
cudaError_t launch_sum_split_blocks(const float* dw4, float* dw, int64_t K, int64_t C, int64_t S,
                                    cudaStream_t stream);

int num_sms();

}  // namespace c1d
