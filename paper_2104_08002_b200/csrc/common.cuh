// common.cuh — shared device helpers for the conv1d kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace c1d {

// fp32 -> bf16 bits, round-to-nearest-even, NaN -> quiet NaN, inf kept. Bit-identical to the
// reference conv1d::fp32_to_bf16 (proj/include/conv1d/bf16.hpp:29-40).
__host__ __device__ __forceinline__ uint16_t fp32_to_bf16_bits(float x) {
#ifdef __CUDA_ARCH__
    uint32_t u = __float_as_uint(x);
#else
    uint32_t u;
    __builtin_memcpy(&u, &x, 4);
#endif
    if ((u & 0x7f800000u) == 0x7f800000u) {
        if ((u & 0x007fffffu) != 0) return static_cast<uint16_t>((u >> 16) | 0x0040u);
        return static_cast<uint16_t>(u >> 16);
    }
    u += 0x7fffu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}

__host__ __device__ __forceinline__ float bf16_bits_to_fp32(uint16_t b) {
    const uint32_t u = static_cast<uint32_t>(b) << 16;
#ifdef __CUDA_ARCH__
    return __uint_as_float(u);
#else
    float f;
    __builtin_memcpy(&f, &u, 4);
    return f;
#endif
}

__device__ __forceinline__ float round_to_bf16(float x) { return bf16_bits_to_fp32(fp32_to_bf16_bits(x)); }

// Load one element of an FP32 or BF16 tensor as float; `round` applies the BF16 rounding the
// reference performs on FP32 inputs in BF16 mode.
template <typename T>
__device__ __forceinline__ float load_as_float(const T* p, int64_t i, bool round);
template <>
__device__ __forceinline__ float load_as_float<float>(const float* p, int64_t i, bool round) {
    const float v = __ldg(p + i);
    return round ? round_to_bf16(v) : v;
}
template <>
__device__ __forceinline__ float load_as_float<uint16_t>(const uint16_t* p, int64_t i, bool) {
    return bf16_bits_to_fp32(__ldg(p + i));
}

__host__ __device__ constexpr int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace c1d
