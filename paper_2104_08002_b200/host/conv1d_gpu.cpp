// conv1d_gpu.cpp — drop-in replacement of the reference's conv pass translation unit
// (/root/reference/proj/src/conv.cpp) on top of the B200 C ABI (include/c1d.h).
//
// It defines exactly the symbols conv.hpp declares:
//   conv1d::output_width / conv_shapes / conv_flops            conv.hpp:31-37  (conv.cpp:142-163)
//   conv1d::conv1d_forward                                     conv.hpp:42-43  (conv.cpp:165-191)
//   conv1d::conv1d_backward_data                               conv.hpp:49-50  (conv.cpp:193-227)
//   conv1d::conv1d_backward_weight                             conv.hpp:56-57  (conv.cpp:229-326)
// with the reference's host-side semantics: host std::vector tensors in, results returned by value,
// the same exception classes (errors.hpp) thrown for the same conditions, `threads` ignored
// (the GPU path is parallel over the whole tensor and bitwise thread-count invariant).
// Link it instead of conv.cpp next to the reference's other sources and the reference's host code
// (tests, bench, train) runs on the B200 kernels unchanged.
//
// Weights arrive packed (PackedWeights, tensor.hpp:67-75); unpack_weights (tensor.cpp:43-58)
// recovers the natural KCS order the C ABI takes. Each call copies inputs host->device, runs the
// pass on the current device and copies the result back (return-by-value semantics).
//
// BF16 odd dimensions: the reference rejects odd C/K/widths in BF16 (conv.cpp:40-57). The GPU
// kernels accept them; this shim keeps the reference behaviour (C1D_FLAG_STRICT_BF16_DIMS) unless
// C1D_RELAXED_BF16=1 is set in the environment.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/c1d.h"
#include "conv1d/conv.hpp"
#include "conv1d/errors.hpp"
#include "conv1d/tensor.hpp"

namespace conv1d {
namespace {

c1d_desc make_desc(const ConvParams& p, idx_t n, idx_t w_in) {
    c1d_desc d{};
    d.n = n;
    d.c = p.channels;
    d.k = p.filters;
    d.s = p.taps;
    d.d = p.dilation;
    d.w_in = w_in;
    d.precision = p.precision == Precision::Bf16 ? C1D_PRECISION_BF16 : C1D_PRECISION_FP32;
    d.in_dtype = C1D_DTYPE_F32;  // the reference hands FP32 data and rounds internally
    d.algo = C1D_ALGO_AUTO;
    const char* relaxed = std::getenv("C1D_RELAXED_BF16");
    d.flags = (relaxed && relaxed[0] == '1') ? 0u : C1D_FLAG_STRICT_BF16_DIMS;
    d.block_w = p.block_w;
    return d;
}

[[noreturn]] void raise(c1d_status st) {
    std::string msg = c1d_last_error_message();
    if (msg.empty()) msg = c1d_strerror(st);
    switch (st) {
        case C1D_ERR_SHAPE_MISMATCH: throw ShapeMismatch(msg);
        case C1D_ERR_ODD_DIMS: throw OddDims(msg);
        case C1D_ERR_TOO_NARROW: throw TooNarrow(msg);
        default: throw Error("c1d: " + msg);
    }
}

void check(c1d_status st) {
    if (st != C1D_OK) raise(st);
}

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Error(std::string("CUDA ") + what + ": " + cudaGetErrorString(e));
}

// RAII device buffer
struct DevBuf {
    void* p = nullptr;
    explicit DevBuf(size_t bytes) {
        if (bytes) cuda_check(cudaMalloc(&p, bytes), "cudaMalloc");
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

void h2d(void* dst, const void* src, size_t bytes) {
    if (bytes) cuda_check(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice), "H2D");
}
void d2h(void* dst, const void* src, size_t bytes) {
    if (bytes) cuda_check(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost), "D2H");
}

void check_packed(const PackedWeights& w, const ConvParams& p, WeightLayout want) {
    if (w.layout != want) throw ShapeMismatch("packed weights have the wrong layout for this pass");
    if (w.c != p.channels || w.k != p.filters || w.s != p.taps) {
        throw ShapeMismatch("packed weights are S=" + std::to_string(w.s) + " K=" + std::to_string(w.k) +
                            " C=" + std::to_string(w.c) + ", conv params say S=" + std::to_string(p.taps) +
                            " K=" + std::to_string(p.filters) + " C=" + std::to_string(p.channels));
    }
}

}  // namespace

idx_t output_width(const ConvParams& p, idx_t w_padded) {
    const c1d_desc d = make_desc(p, 1, w_padded);
    int64_t q = 0;
    check(c1d_output_width(&d, &q));
    return q;
}

ConvShapes conv_shapes(const ConvParams& p, idx_t w_padded) {
    ConvShapes s;
    s.receptive = p.dilation * (p.taps - 1);
    s.q = output_width(p, w_padded);
    s.w_padded = w_padded;
    return s;
}

std::int64_t conv_flops(const ConvParams& p, idx_t batch, idx_t q) {
    return std::int64_t{2} * batch * p.filters * p.channels * p.taps * q;
}

Tensor3Df conv1d_forward(const Tensor3Df& in, const PackedWeights& w, const ConvParams& p, int /*threads*/) {
    check_packed(w, p, WeightLayout::ForwardSKC);
    if (in.c != p.channels)
        throw ShapeMismatch("input has " + std::to_string(in.c) + " channels, conv expects " +
                            std::to_string(p.channels));
    const c1d_desc d = make_desc(p, in.n, in.w);
    int64_t q = 0;
    check(c1d_output_width(&d, &q));
    Tensor3Df out(in.n, p.filters, q);
    if (in.n == 0) return out;
    const WeightKCS kcs = unpack_weights(w);
    DevBuf dx(sizeof(float) * in.data.size()), dw(sizeof(float) * kcs.data.size()),
        dy(sizeof(float) * out.data.size());
    h2d(dx.p, in.data.data(), sizeof(float) * in.data.size());
    h2d(dw.p, kcs.data.data(), sizeof(float) * kcs.data.size());
    check(c1d_forward(&d, dx.p, static_cast<const float*>(dw.p), static_cast<float*>(dy.p), nullptr, 0, nullptr));
    d2h(out.data.data(), dy.p, sizeof(float) * out.data.size());
    return out;
}

Tensor3Df conv1d_backward_data(const Tensor3Df& grad_out, const PackedWeights& w, const ConvParams& p,
                               int /*threads*/) {
    check_packed(w, p, WeightLayout::BackwardSCK);
    if (grad_out.c != p.filters)
        throw ShapeMismatch("grad_out has " + std::to_string(grad_out.c) + " channels, conv has K=" +
                            std::to_string(p.filters));
    const idx_t receptive = p.dilation * (p.taps - 1);
    const idx_t w_out = grad_out.w + receptive;
    const c1d_desc d = make_desc(p, grad_out.n, w_out);
    int64_t q = 0;
    check(c1d_output_width(&d, &q));
    Tensor3Df grad_d(grad_out.n, p.channels, w_out);
    if (grad_out.n == 0) return grad_d;
    const WeightKCS kcs = unpack_weights(w);
    DevBuf dg(sizeof(float) * grad_out.data.size()), dw(sizeof(float) * kcs.data.size()),
        dd(sizeof(float) * grad_d.data.size());
    h2d(dg.p, grad_out.data.data(), sizeof(float) * grad_out.data.size());
    h2d(dw.p, kcs.data.data(), sizeof(float) * kcs.data.size());
    check(c1d_backward_data(&d, dg.p, static_cast<const float*>(dw.p), static_cast<float*>(dd.p), nullptr, 0,
                            nullptr));
    d2h(grad_d.data.data(), dd.p, sizeof(float) * grad_d.data.size());
    return grad_d;
}

WeightKCS conv1d_backward_weight(const Tensor3Df& grad_out, const Tensor3Df& in, const ConvParams& p,
                                 int /*threads*/) {
    if (in.n != grad_out.n) throw ShapeMismatch("batch sizes differ between input and grad_out");
    if (in.c != p.channels || grad_out.c != p.filters) throw ShapeMismatch("channel counts do not match conv params");
    const idx_t q = grad_out.w;
    const idx_t receptive = p.dilation * (p.taps - 1);
    if (in.w != q + receptive)
        throw ShapeMismatch("input width " + std::to_string(in.w) + " != Q + d*(S-1) = " +
                            std::to_string(q + receptive));
    const c1d_desc d = make_desc(p, in.n, in.w);
    int64_t qq = 0;
    check(c1d_output_width(&d, &qq));
    WeightKCS grad(p.filters, p.channels, p.taps);
    DevBuf dx(sizeof(float) * in.data.size()), dg(sizeof(float) * grad_out.data.size()),
        dw(sizeof(float) * grad.data.size());
    h2d(dx.p, in.data.data(), sizeof(float) * in.data.size());
    h2d(dg.p, grad_out.data.data(), sizeof(float) * grad_out.data.size());
    check(c1d_backward_weight(&d, dx.p, dg.p, static_cast<float*>(dw.p), nullptr, 0, nullptr));
    d2h(grad.data.data(), dw.p, sizeof(float) * grad.data.size());
    return grad;
}

}  // namespace conv1d
