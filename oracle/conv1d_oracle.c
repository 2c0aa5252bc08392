/*
 * conv1d_oracle.c — CPU restatement of the reference conv1d algorithm.
 *
 * TEST INFRASTRUCTURE ONLY. This file is the parity checker for the B200 kernels; only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it. The product
 * path (paper_2104_08002_b200/) never links or calls it.
 *
 * Every function restates one piece of the reference implementation under
 * /root/reference/proj (paths below are relative to that tree):
 *   - xoshiro256** + splitmix64 seeding, next_double/next_float/next_below/next_normal,
 *     fill_uniform                                     include/conv1d/rng.hpp:14-58
 *   - RNE fp32->bf16 with quiet NaN, exact widening    include/conv1d/bf16.hpp:20-42
 *   - output_width / conv_flops / parameter checks     src/conv.cpp:33-57,142-163
 *   - pack_weights_forward / _backward / unpack        src/tensor.cpp:5-58
 *   - zero_pad_width / same_pad_width                  src/tensor.cpp:60-82
 *   - naive_forward / naive_backward_data /
 *     naive_backward_weight (double accumulation)      src/reference.cpp:23-104
 *   - norm_rel_error                                   src/reference.cpp:151-162
 * New samplers not present in the reference Rng (Poisson via Knuth's product method and
 * Bernoulli via a threshold on next_double) back the config-5 network inputs.
 *
 * Parity is pinned: tests/test_oracle.py checks this file against golden vectors produced by
 * the reference itself (tests/golden/make_golden.py, via oracle/_ref/libconv1d_ref.so).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#define ORC_OK 0
#define ORC_SHAPE_MISMATCH 1
#define ORC_ODD_DIMS 2
#define ORC_TOO_NARROW 3

/* ---------------------------------------------------------------- rng (rng.hpp:12-64) */
typedef struct {
    uint64_t s[4];
} orc_rng;

static uint64_t rotl64(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }

void orc_rng_seed(orc_rng* r, uint64_t seed) {
    uint64_t x = seed;
    for (int i = 0; i < 4; ++i) { /* splitmix64, rng.hpp:14-24 */
        x += 0x9e3779b97f4a7c15ull;
        uint64_t z = x;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        r->s[i] = z ^ (z >> 31);
    }
}

uint64_t orc_rng_next_u64(orc_rng* r) { /* xoshiro256**, rng.hpp:26-36 */
    uint64_t* s = r->s;
    const uint64_t result = rotl64(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return result;
}

double orc_rng_next_double(orc_rng* r) { return (double)(orc_rng_next_u64(r) >> 11) * 0x1.0p-53; }

float orc_rng_next_float(orc_rng* r, float lo, float hi) {
    return lo + (float)orc_rng_next_double(r) * (hi - lo);
}

uint64_t orc_rng_next_below(orc_rng* r, uint64_t bound) { return orc_rng_next_u64(r) % bound; }

double orc_rng_next_normal(orc_rng* r) { /* Box-Muller, one value per call, rng.hpp:50-54 */
    const double kPi = 3.14159265358979323846;
    const double u1 = (double)((orc_rng_next_u64(r) >> 11) + 1) * 0x1.0p-53;
    const double u2 = orc_rng_next_double(r);
    return sqrt(-2.0 * log(u1)) * cos(2.0 * kPi * u2);
}

void orc_fill_uniform(orc_rng* r, float* out, int64_t n, float lo, float hi) {
    for (int64_t i = 0; i < n; ++i) out[i] = orc_rng_next_float(r, lo, hi);
}

void orc_fill_normal(orc_rng* r, float* out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) out[i] = (float)orc_rng_next_normal(r);
}

/* New sampler (no reference counterpart): Knuth's product-of-uniforms Poisson draw. */
uint32_t orc_rng_next_poisson(orc_rng* r, double lambda) {
    const double limit = exp(-lambda);
    double prod = orc_rng_next_double(r);
    uint32_t k = 0;
    while (prod > limit) {
        ++k;
        prod *= orc_rng_next_double(r);
    }
    return k;
}

void orc_fill_poisson(orc_rng* r, float* out, int64_t n, double lambda) {
    for (int64_t i = 0; i < n; ++i) out[i] = (float)orc_rng_next_poisson(r, lambda);
}

/* New sampler: Bernoulli(p) as next_double() < p. */
void orc_fill_bernoulli(orc_rng* r, float* out, int64_t n, double p) {
    for (int64_t i = 0; i < n; ++i) out[i] = orc_rng_next_double(r) < p ? 1.0f : 0.0f;
}

/* Counter-based samplers of the device path (paper_2104_08002_b200/csrc/train.cu, c1d.h
 * c1d_fill_poisson / c1d_fill_bernoulli), restated for bit-exact checks: element i owns the
 * splitmix64 stream state = mix64(seed ^ mix64(i + golden)). New code, no reference counterpart. */
static uint64_t orc_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static double orc_splitmix_next(uint64_t* s) {
    *s += 0x9E3779B97F4A7C15ull;
    return (double)(orc_mix64(*s) >> 11) * 0x1.0p-53;
}
void orc_sample_poisson(float* out, int64_t n, double lambda, uint64_t seed) {
    const double limit = exp(-lambda);
    for (int64_t i = 0; i < n; ++i) {
        uint64_t st = orc_mix64(seed ^ orc_mix64((uint64_t)i + 0x9E3779B97F4A7C15ull));
        double prod = orc_splitmix_next(&st);
        uint32_t k = 0;
        while (prod > limit) {
            ++k;
            prod *= orc_splitmix_next(&st);
        }
        out[i] = (float)k;
    }
}
void orc_sample_bernoulli(float* out, int64_t n, double p, uint64_t seed) {
    for (int64_t i = 0; i < n; ++i) {
        uint64_t st = orc_mix64(seed ^ orc_mix64((uint64_t)i + 0x9E3779B97F4A7C15ull));
        out[i] = orc_splitmix_next(&st) < p ? 1.0f : 0.0f;
    }
}

/* ---------------------------------------------------------------- bf16 (bf16.hpp:20-42) */
uint16_t orc_fp32_to_bf16(float x) {
    uint32_t u;
    memcpy(&u, &x, sizeof u);
    if ((u & 0x7f800000u) == 0x7f800000u) {
        if ((u & 0x007fffffu) != 0) return (uint16_t)((u >> 16) | 0x0040u); /* quiet NaN */
        return (uint16_t)(u >> 16);                                      /* +-inf */
    }
    u += 0x7fffu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}

float orc_bf16_to_fp32(uint16_t b) {
    const uint32_t u = (uint32_t)b << 16;
    float f;
    memcpy(&f, &u, sizeof f);
    return f;
}

void orc_round_bf16(const float* in, float* out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) out[i] = orc_bf16_to_fp32(orc_fp32_to_bf16(in[i]));
}

void orc_to_bf16_bits(const float* in, uint16_t* out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) out[i] = orc_fp32_to_bf16(in[i]);
}

/* ---------------------------------------------------------------- geometry (conv.cpp) */
/* validate_params (conv.cpp:33-50); precision 1 = bf16 enforces the even-dims rule. */
int orc_validate_params(int64_t c, int64_t k, int64_t s, int64_t d, int precision, int64_t block_w) {
    if (c < 1 || k < 1 || s < 1 || d < 1 || block_w < 1) return ORC_SHAPE_MISMATCH;
    if (precision == 1 && (c % 2 != 0 || k % 2 != 0 || block_w % 2 != 0)) return ORC_ODD_DIMS;
    return ORC_OK;
}

/* output_width (conv.cpp:142-151): Q = W - d(S-1), TooNarrow when W <= d(S-1). */
int orc_output_width(int64_t c, int64_t k, int64_t s, int64_t d, int64_t w_padded, int64_t* q) {
    const int e = orc_validate_params(c, k, s, d, 0, 64);
    if (e) return e;
    const int64_t receptive = d * (s - 1);
    if (w_padded <= receptive) return ORC_TOO_NARROW;
    *q = w_padded - receptive;
    return ORC_OK;
}

int64_t orc_conv_flops(int64_t n, int64_t c, int64_t k, int64_t s, int64_t q) {
    return (int64_t)2 * n * k * c * s * q; /* conv.cpp:161-163 */
}

/* same_pad_width (tensor.cpp:76-82): -1 when d(S-1) is odd. */
int64_t orc_same_pad_width(int64_t s, int64_t d) {
    const int64_t r = d * (s - 1);
    return (r % 2 != 0) ? -1 : r / 2;
}

/* ---------------------------------------------------------------- packing (tensor.cpp:5-58) */
void orc_pack_forward(const float* kcs, int64_t k, int64_t c, int64_t s, float* skc) {
    for (int64_t t = 0; t < s; ++t)
        for (int64_t a = 0; a < k; ++a)
            for (int64_t b = 0; b < c; ++b) skc[(t * k + a) * c + b] = kcs[(a * c + b) * s + t];
}

void orc_pack_backward(const float* kcs, int64_t k, int64_t c, int64_t s, float* sck) {
    for (int64_t t = 0; t < s; ++t) {
        const int64_t src = s - 1 - t; /* slot t holds original tap S-1-t, transposed to C x K */
        for (int64_t b = 0; b < c; ++b)
            for (int64_t a = 0; a < k; ++a) sck[(t * c + b) * k + a] = kcs[(a * c + b) * s + src];
    }
}

/* layout 0 = ForwardSKC, 1 = BackwardSCK */
void orc_unpack(const float* packed, int layout, int64_t k, int64_t c, int64_t s, float* kcs) {
    for (int64_t t = 0; t < s; ++t)
        for (int64_t a = 0; a < k; ++a)
            for (int64_t b = 0; b < c; ++b) {
                if (layout == 0)
                    kcs[(a * c + b) * s + t] = packed[(t * k + a) * c + b];
                else
                    kcs[(a * c + b) * s + (s - 1 - t)] = packed[(t * c + b) * k + a];
            }
}

void orc_zero_pad_width(const float* in, int64_t n, int64_t c, int64_t w, int64_t left, int64_t right,
                        float* out) {
    const int64_t wo = w + left + right;
    memset(out, 0, sizeof(float) * (size_t)(n * c * wo));
    for (int64_t i = 0; i < n * c; ++i) memcpy(out + i * wo + left, in + i * w, sizeof(float) * (size_t)w);
}

/* ---------------------------------------------------------------- naive passes (reference.cpp) */
/* out(n,k,x) = sum_c sum_s in(n,c,x+d*s) * w(k,c,s), double accumulation, c outer / s inner. */
void orc_naive_forward(const float* in, int64_t n, int64_t c, int64_t w_in, const float* w, int64_t k,
                       int64_t s, int64_t d, float* out) {
    const int64_t q = w_in - d * (s - 1);
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t i = 0; i < n; ++i)
        for (int64_t kk = 0; kk < k; ++kk)
            for (int64_t x = 0; x < q; ++x) {
                double acc = 0.0;
                for (int64_t cc = 0; cc < c; ++cc) {
                    const float* row = in + (i * c + cc) * w_in + x;
                    const float* wr = w + (kk * c + cc) * s;
                    for (int64_t t = 0; t < s; ++t) acc += (double)row[d * t] * (double)wr[t];
                }
                out[(i * k + kk) * q + x] = (float)acc;
            }
}

/* grad_in(n,c,x) = sum_k sum_s grad_out(n,k,x-d*s) * w(k,c,s), out-of-range terms zero. */
void orc_naive_backward_data(const float* go, int64_t n, int64_t k, int64_t q, const float* w, int64_t c,
                             int64_t s, int64_t d, float* gin) {
    const int64_t width = q + d * (s - 1);
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t i = 0; i < n; ++i)
        for (int64_t cc = 0; cc < c; ++cc)
            for (int64_t x = 0; x < width; ++x) {
                double acc = 0.0;
                for (int64_t kk = 0; kk < k; ++kk) {
                    const float* row = go + (i * k + kk) * q;
                    const float* wr = w + (kk * c + cc) * s;
                    for (int64_t t = 0; t < s; ++t) {
                        const int64_t src = x - d * t;
                        if (src < 0 || src >= q) continue;
                        acc += (double)row[src] * (double)wr[t];
                    }
                }
                gin[(i * c + cc) * width + x] = (float)acc;
            }
}

/* grad_w(k,c,s) = sum_n sum_q in(n,c,q+d*s) * grad_out(n,k,q). */
void orc_naive_backward_weight(const float* go, const float* in, int64_t n, int64_t c, int64_t k,
                               int64_t s, int64_t d, int64_t q, float* gw) {
    const int64_t w_in = q + d * (s - 1);
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t kk = 0; kk < k; ++kk)
        for (int64_t cc = 0; cc < c; ++cc)
            for (int64_t t = 0; t < s; ++t) {
                double acc = 0.0;
                for (int64_t i = 0; i < n; ++i) {
                    const float* xr = in + (i * c + cc) * w_in + d * t;
                    const float* gr = go + (i * k + kk) * q;
                    for (int64_t x = 0; x < q; ++x) acc += (double)xr[x] * (double)gr[x];
                }
                gw[(kk * c + cc) * s + t] = (float)acc;
            }
}

/* Worst |got - want| over max(max|want|, 1)  (reference.cpp:151-162). */
double orc_norm_rel_error(const float* got, const float* want, int64_t n) {
    double norm = 1.0, worst = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double a = fabs((double)want[i]);
        if (a > norm) norm = a;
    }
    for (int64_t i = 0; i < n; ++i) {
        const double diff = fabs((double)got[i] - (double)want[i]);
        if (diff / norm > worst) worst = diff / norm;
    }
    return worst;
}
