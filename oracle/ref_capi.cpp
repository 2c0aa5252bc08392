// ref_capi.cpp — extern "C" shim over the UNMODIFIED reference library so Python tests and
// bench.py can run the reference's own CPU code path.
//
// TEST INFRASTRUCTURE ONLY (oracle side). Built by oracle/Makefile together with the reference
// sources where they lie under /root/reference/proj/src into oracle/_ref/libconv1d_ref*.so;
// no reference source is copied into this repository. Wrapped entry points:
//   conv1d_forward / conv1d_backward_data / conv1d_backward_weight   proj/src/conv.cpp:165-326
//   pack_weights_forward / pack_weights_backward / unpack_weights     proj/src/tensor.cpp:5-58
//   naive_forward / naive_backward_data / naive_backward_weight       proj/src/reference.cpp:23-104
//   norm_rel_error                                                    proj/src/reference.cpp:151-162
//   measure_kernel (the reference timing method)                      proj/src/bench.cpp:172-234
//   Rng / fp32_to_bf16                                                proj/include/conv1d/{rng,bf16}.hpp
//   DemoNet forward / backward / train_step, gather/scatter params    proj/src/train.cpp:257-353
//   mse_loss / bce_with_logits / sgd_step / auroc                     proj/src/train.cpp:106-171
//   generate_synthetic_dataset                                        proj/src/train.cpp:62-98
#include <cstdint>
#include <cstring>
#include <exception>
#include <vector>

#include "conv1d/bench.hpp"
#include "conv1d/bf16.hpp"
#include "conv1d/conv.hpp"
#include "conv1d/errors.hpp"
#include "conv1d/reference.hpp"
#include "conv1d/rng.hpp"
#include "conv1d/tensor.hpp"
#include "conv1d/train.hpp"

using namespace conv1d;

namespace {

// Status codes mirror include/c1d.h (C1D_OK, C1D_ERR_SHAPE_MISMATCH, C1D_ERR_ODD_DIMS,
// C1D_ERR_TOO_NARROW); anything else becomes 99.
template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const ShapeMismatch&) {
        return 1;
    } catch (const OddDims&) {
        return 2;
    } catch (const TooNarrow&) {
        return 3;
    } catch (const std::exception&) {
        return 99;
    }
}

ConvParams make_params(int64_t c, int64_t k, int64_t s, int64_t d, int precision, int64_t block_w) {
    ConvParams p;
    p.channels = c;
    p.filters = k;
    p.taps = s;
    p.dilation = d;
    p.precision = precision == 1 ? Precision::Bf16 : Precision::Fp32;
    p.block_w = block_w;
    return p;
}

Tensor3Df make_tensor(const float* data, int64_t n, int64_t c, int64_t w) {
    Tensor3Df t(n, c, w);
    std::memcpy(t.data.data(), data, sizeof(float) * static_cast<size_t>(n * c * w));
    return t;
}

WeightKCS make_kcs(const float* data, int64_t k, int64_t c, int64_t s) {
    WeightKCS w(k, c, s);
    std::memcpy(w.data.data(), data, sizeof(float) * static_cast<size_t>(k * c * s));
    return w;
}

}  // namespace

extern "C" {

int ref_forward(const float* in, int64_t n, int64_t c, int64_t w_in, const float* w_kcs, int64_t k,
                int64_t s, int64_t d, int precision, int64_t block_w, int threads, float* out) {
    return guarded([&] {
        const ConvParams p = make_params(c, k, s, d, precision, block_w);
        const Tensor3Df y =
            conv1d_forward(make_tensor(in, n, c, w_in), pack_weights_forward(make_kcs(w_kcs, k, c, s)), p,
                           threads);
        std::memcpy(out, y.data.data(), sizeof(float) * y.data.size());
    });
}

int ref_backward_data(const float* go, int64_t n, int64_t k, int64_t q, const float* w_kcs, int64_t c,
                      int64_t s, int64_t d, int precision, int64_t block_w, int threads, float* gin) {
    return guarded([&] {
        const ConvParams p = make_params(c, k, s, d, precision, block_w);
        const Tensor3Df g = conv1d_backward_data(
            make_tensor(go, n, k, q), pack_weights_backward(make_kcs(w_kcs, k, c, s)), p, threads);
        std::memcpy(gin, g.data.data(), sizeof(float) * g.data.size());
    });
}

int ref_backward_weight(const float* go, const float* in, int64_t n, int64_t c, int64_t k, int64_t s,
                        int64_t d, int64_t q, int precision, int64_t block_w, int threads, float* gw) {
    return guarded([&] {
        const ConvParams p = make_params(c, k, s, d, precision, block_w);
        const int64_t w_in = q + d * (s - 1);
        const WeightKCS g =
            conv1d_backward_weight(make_tensor(go, n, k, q), make_tensor(in, n, c, w_in), p, threads);
        std::memcpy(gw, g.data.data(), sizeof(float) * g.data.size());
    });
}

int ref_output_width(int64_t c, int64_t k, int64_t s, int64_t d, int precision, int64_t w_padded,
                     int64_t* q) {
    return guarded([&] { *q = output_width(make_params(c, k, s, d, precision, 64), w_padded); });
}

int64_t ref_conv_flops(int64_t n, int64_t c, int64_t k, int64_t s, int64_t q) {
    return conv_flops(make_params(c, k, s, 1, 0, 64), n, q);
}

void ref_pack_forward(const float* kcs, int64_t k, int64_t c, int64_t s, float* out) {
    const PackedWeights p = pack_weights_forward(make_kcs(kcs, k, c, s));
    std::memcpy(out, p.data.data(), sizeof(float) * p.data.size());
}

void ref_pack_backward(const float* kcs, int64_t k, int64_t c, int64_t s, float* out) {
    const PackedWeights p = pack_weights_backward(make_kcs(kcs, k, c, s));
    std::memcpy(out, p.data.data(), sizeof(float) * p.data.size());
}

void ref_naive_forward(const float* in, int64_t n, int64_t c, int64_t w_in, const float* w_kcs, int64_t k,
                       int64_t s, int64_t d, float* out) {
    const Tensor3Df y = naive_forward(make_tensor(in, n, c, w_in), make_kcs(w_kcs, k, c, s),
                                      make_params(c, k, s, d, 0, 64));
    std::memcpy(out, y.data.data(), sizeof(float) * y.data.size());
}

void ref_naive_backward_data(const float* go, int64_t n, int64_t k, int64_t q, const float* w_kcs,
                             int64_t c, int64_t s, int64_t d, float* gin) {
    const Tensor3Df g = naive_backward_data(make_tensor(go, n, k, q), make_kcs(w_kcs, k, c, s),
                                            make_params(c, k, s, d, 0, 64));
    std::memcpy(gin, g.data.data(), sizeof(float) * g.data.size());
}

void ref_naive_backward_weight(const float* go, const float* in, int64_t n, int64_t c, int64_t k,
                               int64_t s, int64_t d, int64_t q, float* gw) {
    const int64_t w_in = q + d * (s - 1);
    const WeightKCS g = naive_backward_weight(make_tensor(go, n, k, q), make_tensor(in, n, c, w_in),
                                              make_params(c, k, s, d, 0, 64));
    std::memcpy(gw, g.data.data(), sizeof(float) * g.data.size());
}

double ref_norm_rel_error(const float* got, const float* want, int64_t count) {
    return norm_rel_error({got, static_cast<size_t>(count)}, {want, static_cast<size_t>(count)});
}

uint16_t ref_fp32_to_bf16(float x) { return fp32_to_bf16(x).bits; }

void* ref_rng_new(uint64_t seed) { return new Rng(seed); }
void ref_rng_free(void* r) { delete static_cast<Rng*>(r); }
uint64_t ref_rng_next_u64(void* r) { return static_cast<Rng*>(r)->next_u64(); }
double ref_rng_next_double(void* r) { return static_cast<Rng*>(r)->next_double(); }
double ref_rng_next_normal(void* r) { return static_cast<Rng*>(r)->next_normal(); }
uint64_t ref_rng_next_below(void* r, uint64_t bound) { return static_cast<Rng*>(r)->next_below(bound); }
void ref_rng_fill_uniform(void* r, float* out, int64_t count, float lo, float hi) {
    static_cast<Rng*>(r)->fill_uniform({out, static_cast<size_t>(count)}, lo, hi);
}

// pass: 0 forward, 1 backward_data, 2 backward_weight. Returns mean seconds or a negative
// status on error.
double ref_measure_kernel(int64_t n, int64_t c, int64_t k, int64_t s, int64_t d, int64_t q, int precision,
                          int pass, int iterations, int warmup, int threads, uint64_t seed) {
    double secs = -1.0;
    const int rc = guarded([&] {
        BenchShape shape;
        shape.batch = n;
        shape.channels = c;
        shape.filters = k;
        shape.taps = s;
        shape.dilation = d;
        shape.q = q;
        shape.precision = precision == 1 ? Precision::Bf16 : Precision::Fp32;
        const Pass ps = pass == 0 ? Pass::Forward : pass == 1 ? Pass::BackwardData : Pass::BackwardWeight;
        secs = measure_kernel(shape, ps, iterations, warmup, threads, seed);
    });
    return rc == 0 ? secs : -static_cast<double>(rc);
}

// Parse a sweep CSV with the reference's own reader (bench.cpp:336-370): record count, or -1 when
// it rejects the file. Lets tests pin paper_2104_08002_b200/sweep.py's writer to the schema.
int64_t ref_parse_csv_count(const char* path) {
    try {
        return static_cast<int64_t>(parse_csv(path).size());
    } catch (const std::exception&) {
        return -1;
    }
}

// ---- the reference network (train.cpp), for pinning the GPU network step ----
void* ref_demonet_new(int blocks, int64_t hidden, int64_t taps, int64_t dilation, int precision, uint64_t seed) {
    try {
        return new DemoNet(blocks, hidden, taps, dilation, precision == 1 ? Precision::Bf16 : Precision::Fp32,
                           seed);
    } catch (const std::exception&) {
        return nullptr;
    }
}
void ref_demonet_free(void* h) { delete static_cast<DemoNet*>(h); }
// precision actually used by layer i (make_layer's even-dims rule, train.cpp:233-239): 0 FP32, 1 BF16
int ref_demonet_layer_precision(void* h, int i) {
    auto layers = static_cast<DemoNet*>(h)->layers();
    if (i < 0 || i >= static_cast<int>(layers.size())) return -1;
    return layers[static_cast<size_t>(i)]->p.precision == Precision::Bf16 ? 1 : 0;
}
int64_t ref_demonet_param_count(void* h) { return static_cast<int64_t>(gather_params(*static_cast<DemoNet*>(h)).size()); }
void ref_demonet_gather_params(void* h, float* out) {
    const std::vector<float> v = gather_params(*static_cast<DemoNet*>(h));
    std::memcpy(out, v.data(), sizeof(float) * v.size());
}
int ref_demonet_scatter_params(void* h, const float* in, int64_t count) {
    return guarded([&] { scatter_params(*static_cast<DemoNet*>(h), {in, static_cast<size_t>(count)}); });
}
void ref_demonet_gather_grads(void* h, float* out) {
    const std::vector<float> v = gather_grads(*static_cast<DemoNet*>(h));
    std::memcpy(out, v.data(), sizeof(float) * v.size());
}
// forward only: pred and logits, each (n, 1, width_padded - 2*pad)
int ref_demonet_forward(void* h, const float* x, int64_t n, int64_t w_padded, int threads, float* pred,
                        float* logits) {
    return guarded([&] {
        const DemoNet::Output o = static_cast<DemoNet*>(h)->forward(make_tensor(x, n, 1, w_padded), threads);
        std::memcpy(pred, o.pred.data.data(), sizeof(float) * o.pred.data.size());
        std::memcpy(logits, o.logits.data.data(), sizeof(float) * o.logits.data.size());
    });
}
// one train_step (forward, mse + bce_weight*bce, full backward; gradients left in the layers)
int ref_demonet_train_step(void* h, const float* x, const float* clean, const float* mask, int64_t n,
                           int64_t w_padded, int64_t width, float bce_weight, int threads, double* loss) {
    return guarded([&] {
        *loss = train_step(*static_cast<DemoNet*>(h), make_tensor(x, n, 1, w_padded), make_tensor(clean, n, 1, width),
                           make_tensor(mask, n, 1, width), bce_weight, threads);
    });
}
void ref_demonet_step(void* h, float lr) { static_cast<DemoNet*>(h)->step(lr); }

double ref_mse_loss(const float* pred, const float* target, int64_t count, float* grad) {
    const LossResult r = mse_loss({pred, static_cast<size_t>(count)}, {target, static_cast<size_t>(count)});
    std::memcpy(grad, r.grad.data(), sizeof(float) * r.grad.size());
    return r.value;
}
double ref_bce_with_logits(const float* logits, const float* mask, int64_t count, float* grad) {
    const LossResult r = bce_with_logits({logits, static_cast<size_t>(count)}, {mask, static_cast<size_t>(count)});
    std::memcpy(grad, r.grad.data(), sizeof(float) * r.grad.size());
    return r.value;
}
void ref_sgd_step(float* params, const float* grads, int64_t count, float lr) {
    sgd_step({params, static_cast<size_t>(count)}, {grads, static_cast<size_t>(count)}, lr);
}
double ref_auroc(const float* scores, const float* labels, int64_t count) {
    return auroc({scores, static_cast<size_t>(count)}, {labels, static_cast<size_t>(count)});
}
int ref_synthetic_dataset(uint64_t seed, int64_t count, int64_t width, float* noisy, float* clean, float* mask) {
    return guarded([&] {
        const SyntheticDataset ds = generate_synthetic_dataset(seed, count, width);
        std::memcpy(noisy, ds.noisy.data.data(), sizeof(float) * ds.noisy.data.size());
        std::memcpy(clean, ds.clean.data.data(), sizeof(float) * ds.clean.data.size());
        std::memcpy(mask, ds.mask.data.data(), sizeof(float) * ds.mask.data.size());
    });
}

}  // extern "C"
