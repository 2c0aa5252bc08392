// kernels.h — internal launch interface between the C ABI (c1d_api.cu) and the kernels.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace c1d {

// Count of kernels this library launched (c1d_launch_count()).
void note_launch(int n = 1);
void set_last_error(const char* msg);  // detail text for c1d_last_error_message()

// Accumulation-chain mode of the calling host thread's current pass (set by the C ABI from the
// desc: FP32 precision, or BF16 with C1D_FLAG_EXACT_ACCUM). When set, the tensor-core kernels cap
// every FP32 accumulation chain at ~4096 products (segmented backward-weight chains, two-region
// conv reductions); see c1d.h C1D_FLAG_EXACT_ACCUM.
bool exact_accum();
struct ExactAccumScope {
    bool saved;
    explicit ExactAccumScope(bool on);
    ~ExactAccumScope();
};

// Generic "forward-shaped" convolution:
//   out[n][o][x] = sum_i sum_s wg[o][i][s] * in[n][i][x + s*dil + in_off]   (0 outside [0,in_w))
// forward:       in = x  (C ch, W_in), out = y  (K ch, Q),    wg = W (KCS),   in_off = 0
// backward-data: in = dy (K ch, Q),    out = dx (C ch, W_in), wg = W' (CKS, taps reversed),
//                in_off = -d*(S-1)  (the reference's zero_pad_width, conv.cpp:206-208, done
//                as predicated loads instead of a padded copy)
// in_stride: row pitch of the input in elements when it is not in_w (a zero-padded copy whose
// pitch is a multiple of 8 elements, the TMA stride granule).
struct ConvGeom {
    int64_t n, in_ch, in_w, out_ch, out_w, taps, dil, in_off;
    int64_t in_stride = 0;
    // expanded rows (d = 1, 2, 4): the input is the row tensor E of launch_expand_rows, rows of 8
    // bf16 elements E[n*C + c][r][e] = x[n][c][d*r + e + in_off]; out[q] uses rows q/d + s.
    int64_t xr_rows = 0;  // rows per (item, channel) of E; 0 = natural rows
    // xr_inline (d = 1, 2, 4): the input stays natural bf16 rows (pitch in_stride or in_w, a
    // multiple of 8) and the kernel builds E's rows in shared memory (no E tensor in HBM)
    bool xr_inline = false;
};

enum WeightMode { kWeightsForward = 0, kWeightsBackwardData = 1 };

// out (o, i, s) fp32 from w_kcs; mode 1 transposes to (C, K, S) with the tap axis reversed
// (pack_weights_backward, tensor.cpp:23-41). round -> BF16 round-to-nearest-even.
cudaError_t launch_prep_weights(const float* w_kcs, float* out, int64_t K, int64_t C, int64_t S, int mode,
                                bool round, cudaStream_t stream);

// in_dtype: 0 = f32, 1 = bf16 bits. round_in: round FP32 inputs to BF16 on load.
cudaError_t launch_direct_conv(const void* in, int in_dtype, bool round_in, const float* wg, float* out,
                               const ConvGeom& g, cudaStream_t stream);

size_t direct_wgrad_workspace_bytes(int64_t n, int64_t c, int64_t k, int64_t s, int64_t d, int64_t q);
cudaError_t launch_direct_wgrad(const void* x, const void* dy, int in_dtype, bool round_in, float* dw_kcs,
                                float* workspace, int64_t n, int64_t c, int64_t k, int64_t s, int64_t d,
                                int64_t q, cudaStream_t stream);

cudaError_t launch_round_bf16(const float* in, uint16_t* out, int64_t count, cudaStream_t stream);

// layer.cu: fused ConvLayer glue (train.cpp:173-221)
int64_t layer_bias_blocks(int64_t q);  // bias-gradient partials per (item, channel) row
// mask: optional ReLU mask (pre + bias > 0) in the LayerGlue channel-block layout (written by the
// forward epilogue; read by the backward prologue instead of pre + pre_bias).
cudaError_t launch_layer_fwd_epilogue(float* pre, const float* bias, const float* skip, int64_t n, int64_t k, int64_t q,
                                      int relu, int store_pre, float* act, uint16_t* act_bf16, int64_t pad,
                                      uint32_t* mask, cudaStream_t stream);
cudaError_t launch_layer_bwd_prologue(const float* gin, int64_t gin_w, int64_t gin_off, const float* gadd,
                                      const float* pre, const float* pre_bias, const uint32_t* mask, int64_t n,
                                      int64_t k, int64_t q, int relu, float* gsum,
                                      float* grad_pre, uint16_t* grad_pre_bf16, float* bias_grad, float* part,
                                      cudaStream_t stream, const float* pw_dy = nullptr,
                                      const float* pw_w = nullptr, int pw_k = 0);
// bias_grad[c] = fixed-order sum of part[(i*k + c)*nbx + b] over items i < n and blocks b < nbx
cudaError_t launch_bias_grad_reduce(const float* part, float* bias_grad, int64_t n, int64_t k, int64_t nbx,
                                    cudaStream_t stream);

// Layer glue applied inside a conv's output stage (tc_conv epilogue). With
// v0 the conv output at (item n, channel k, column x):
//  mode 1 (forward, train.cpp:176-192): v = v0 + bias[k]; mask bit of (n, k, x) = v > 0;
//         r = relu ? (v > 0 ? v : 0) : v; a = r + skip; pre = v, act = a,
//         act_bf16[row * act_pitch + act_off + x] = RNE bf16(a)   (each output optional)
//  mode 2 (backward, train.cpp:205-221), xi = x - g_off in [0, g_q) (other columns dropped):
//         g = v0 + gadd; gp = (mask_in ? bit xi : 1) ? g : 0; gsum = g, gp32 = gp, gp_bf16 = bf16(gp);
//         bias_grad[k] = sum of gp over items and columns (fixed-order: per-CTA partials in
//         part[k * num_sms() + cta], then one reduce launch)
// ReLU masks are channel-block words: word (n, b, x) of an (N, ceil(K/16), width) uint32 tensor holds
// channels 16b .. 16b+15 of column x in bits 0..15 (width = the conv output width in mode 1, g_q in
// mode 2), so a backward epilogue lane reads one word per 16-row block of its own column.
struct LayerGlue {
    int mode = 0;
    int relu = 0;
    const float* bias = nullptr;
    const float* skip = nullptr;
    float* pre = nullptr;
    float* act = nullptr;
    uint16_t* act_bf16 = nullptr;
    int64_t act_pitch = 0, act_off = 0;
    uint32_t* mask_out = nullptr;
    int64_t g_off = 0, g_q = 0;
    const float* gadd = nullptr;
    const uint32_t* mask_in = nullptr;
    float* gsum = nullptr;
    float* gp = nullptr;
    uint16_t* gp_bf16 = nullptr;
    float* part = nullptr;
    float* bias_grad = nullptr;
    int64_t part_stride = 0;  // set by the launcher
};

// ---- tcgen05 (sm_100a) kernels -----------------------------------------------------------
// Row-tap BF16 tensor-core convolution for dilation 8 (fwd and bwd-data). Returns
// cudaErrorNotSupported when the shape is outside its envelope.
struct TcConvPlan;
// main_ch > 0 (split-FP32 mode): input channels >= main_ch accumulate into a second TMEM region
// that the epilogue adds to the first, so the long accumulation chain only carries the main term.
bool tc_conv_supported(const ConvGeom& g, int64_t main_ch = 0);
// input tiles per super-tile of the carry mode (d = 8, natural rows) for this geometry, 0 if none
int tc_conv_carry_tiles(const ConvGeom& g, int64_t main_ch = 0);
size_t tc_conv_workspace_bytes(const ConvGeom& g, int64_t main_ch = 0);
// wg: (o, i, s) weights of the forward-shaped problem, or with w_bwd_raw the caller's KCS weights of
// a backward-data pass (transposed and tap-reversed while packing).
// glue (optional, mode 1/2): the layer glue replaces the plain FP32 store of `out` (which may then be
// NULL); its bias-gradient partials need out_ch * num_sms() floats at glue->part.
cudaError_t launch_tc_conv(const uint16_t* in_bf16, const float* wg, float* out, const ConvGeom& g,
                           void* workspace, cudaStream_t stream, int64_t main_ch = 0, bool w_bwd_raw = false,
                           const LayerGlue* glue = nullptr, const uint16_t* prepacked = nullptr);
// Bytes of a prepacked weight image for this geometry (0: the plan needs its own packing).
size_t tc_conv_prepack_bytes(const ConvGeom& g);
// Pack `count` weight images (fwd KCS, or raw layer weights with bwd_raw) in one or a few launches.
cudaError_t launch_pack_images_multi(int count, const ConvGeom* gs, const float* const* w, const int* bwd_raw,
                                     void* const* images, cudaStream_t stream);

bool tc_wgrad_supported(int64_t n, int64_t c, int64_t k, int64_t s, int64_t d, int64_t q);
size_t tc_wgrad_workspace_bytes(int64_t n, int64_t c, int64_t k, int64_t s, int64_t d, int64_t q);
// x_w: row pitch of x (elements) if not q + d*(s-1)
cudaError_t launch_tc_wgrad(const uint16_t* x_bf16, const uint16_t* dy_bf16, float* dw_kcs, void* workspace,
                            int64_t n, int64_t c, int64_t k, int64_t s, int64_t d, int64_t q, cudaStream_t stream,
                            int64_t x_w = 0);
bool tc_wgrad_v3_supported(int64_t n, int64_t c, int64_t k, int64_t s, int64_t d, int64_t q);
// d = 1, 2, 4 with the expanded rows built by the loaders from natural bf16 x rows (pitch x_w, a
// multiple of 8 elements covering q + d*(s-1))
bool tc_wgrad_xin_supported(int64_t n, int64_t c, int64_t k, int64_t s, int64_t d, int64_t q);
size_t tc_wgrad_xin_workspace_bytes(int64_t n, int64_t c, int64_t k, int64_t s, int64_t d, int64_t q);
cudaError_t launch_tc_wgrad_xin(const uint16_t* x_bf16, int64_t x_w, const uint16_t* dy_bf16, float* dw_kcs,
                                void* workspace, int64_t n, int64_t c, int64_t k, int64_t s, int64_t d, int64_t q,
                                cudaStream_t stream);
// any d < 8 (1, 2, 4) on channel-octet streams XT[n][ceil(C/8)][rows][8] (launch_to_octets): every
// tap shift is a descriptor offset (tc_wgrad.cu, W2Plan::xt); rows >= q + d*(s-1)
bool tc_wgrad_xt_supported(int64_t n, int64_t c, int64_t k, int64_t s, int64_t d, int64_t q);
size_t tc_wgrad_xt_workspace_bytes(int64_t n, int64_t c, int64_t k, int64_t s, int64_t d, int64_t q);
// zero rows XT needs past q + d*(s-1): a stage's TMA window may run that far past the last column
int64_t tc_wgrad_xt_pad_rows(int64_t n, int64_t c, int64_t k, int64_t s, int64_t d, int64_t q);
cudaError_t launch_tc_wgrad_xt(const uint16_t* xt, int64_t rows, const uint16_t* dy_bf16, float* dw_kcs,
                               void* workspace, int64_t n, int64_t c, int64_t k, int64_t s, int64_t d, int64_t q,
                               cudaStream_t stream);
// XT[n][o][u][e] = bf16(in[n][8o + e][u]), u < rows (zero past C / w)
cudaError_t launch_to_octets(const void* in, int in_dtype, uint16_t* out, int64_t n, int64_t c, int64_t w,
                             int64_t rows, cudaStream_t stream);

// relayout.cu: dilations other than 8 on the dilation-8 tensor-core kernels
// (O, I, S) -> (O, P*I, S'), S' = ceil(S/m): out[o][b*I + i][t] = w[o][i][b + m*t] (0 past S), P = min(m, S)
cudaError_t launch_phase_split_weights(const float* w, float* out, int64_t O, int64_t I, int64_t S, int64_t m,
                                       int64_t P, cudaStream_t stream);
// dW[k][c][b + m*t] = dwb[k][c][t] for t < ceil((S-b)/m)
cudaError_t launch_scatter_phase_wgrad(const float* dwb, float* dw, int64_t K, int64_t C, int64_t S, int64_t m,
                                       int64_t b, cudaStream_t stream);
// planes (d = 8m): in (N, C, W) -> out (N*m, C, W/m): out[n*m + r][c][8u + e] = in[n][c][8(u*m + r) + e]
// (bf16 out; `round` rounds FP32 input with the reference RNE); and the inverse for FP32 results.
cudaError_t launch_to_planes(const void* in, int in_dtype, uint16_t* out, int64_t n, int64_t c, int64_t w,
                             int64_t m, cudaStream_t stream);
cudaError_t launch_from_planes(const float* in, float* out, int64_t n, int64_t c, int64_t w, int64_t m,
                               cudaStream_t stream);
// Shifted phase copies (TMA and cp.async need 16-B aligned starts, so column shifts that are not
// multiples of 8 are materialised): out[n][b*I + i][j] = bf16(in[n][i][j + base + b*delta]) for
// b < P, 0 where the source column is outside [0, w); out rows have pitch w_out.
cudaError_t launch_shift_copies(const void* in, int in_dtype, uint16_t* out, int64_t n, int64_t I, int64_t w,
                                int64_t P, int64_t base, int64_t delta, int64_t w_out, cudaStream_t stream);
cudaError_t launch_shift_copies_f32(const float* in, float* out, int64_t n, int64_t I, int64_t w, int64_t P,
                                    int64_t base, int64_t delta, int64_t w_out, cudaStream_t stream);
// out[r][j] = bf16(in[r][j]) for j < w, 0 for w <= j < w_pad (rows of a zero-padded bf16 copy)
cudaError_t launch_pad_rows(const void* in, int in_dtype, uint16_t* out, int64_t rows, int64_t w, int64_t w_pad,
                            cudaStream_t stream);

// Row tensor for the expanded-row tensor-core mode (dilations 1, 2, 4): out[nc][r][e] =
// bf16(in[nc][d*r + e + off]) (0 outside [0, w)), r < rows; 16-B rows.
cudaError_t launch_expand_rows(const void* in, int in_dtype, uint16_t* out, int64_t nc, int64_t w, int64_t d,
                               int64_t off, int64_t rows, cudaStream_t stream);
// rows of E a tc_conv launch over geometry g (dil 1, 2, 4) reads per (item, channel)
int64_t tc_conv_xr_rows(const ConvGeom& g);

// FP32-on-tensor-core operand splitting (split.cu)
// w_pitch: output row pitch (zero-filled past w), default w; in_item_stride: input elements per
// item (a channel subset of a wider tensor), default c * w
cudaError_t launch_split_channels(const float* in, uint16_t* out, int64_t n, int64_t c, int64_t w, int reps,
                                  unsigned pattern, cudaStream_t stream, int64_t w_pitch = 0,
                                  int64_t in_item_stride = 0, uint16_t* out2 = nullptr, unsigned pattern2 = 0);
cudaError_t launch_add_into(float* out, const float* add, int64_t count, cudaStream_t stream);
cudaError_t launch_split_weights(const float* w, float* out, int64_t K, int64_t C, int64_t S, int kr, int cr,
                                 unsigned sel, cudaStream_t stream);
cudaError_t launch_sum3(const float* hh, const float* hl, const float* lh, float* dw, int64_t count,
                        cudaStream_t stream);
cudaError_t launch_sum_split_blocks(const float* dw4, float* dw, int64_t K, int64_t C, int64_t S,
                                    cudaStream_t stream);
// split patterns: 2-bit fields per channel block (0 hi, 1 mid / two-level lo, 2 three-level lo)
constexpr unsigned kSplitHL = 0x4u;      // [hi | lo] (two-level)
// conv-shaped FP32 passes: six channel blocks of the three-level split, x' = [h m h l h m] against
// w' = [h h m h l m]: the products hh (main chain), hm, mh, hl, lh, mm (weights >= 2^-16)
constexpr int kSplitBlocks = 6;
constexpr unsigned kSplitX = 0x484u;  // fields 0 1 0 2 0 1
constexpr unsigned kSplitW = 0x610u;  // fields 0 0 1 0 2 1
constexpr unsigned kSplitHM = 0x4u;      // [hi | mid] (three-level)
constexpr unsigned kSplitHL3 = 0x8u;     // [hi | lo3]
constexpr unsigned kSplitL3H = 0x2u;     // [lo3 | hi]
cudaError_t launch_sum_split3(const float* a, const float* b, float* dw, int64_t K, int64_t C, int64_t S,
                              cudaStream_t stream);
cudaError_t launch_sum6(const float* t, float* dw, int64_t count, cudaStream_t stream);

int num_sms();

}  // namespace c1d
