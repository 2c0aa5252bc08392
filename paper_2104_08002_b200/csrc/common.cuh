// common.cuh — shared device helpers for the conv1d kernels.
#pragma once
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include <utility>

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

// Four consecutive elements p[i .. i+3] as floats with one vector load (i must be a multiple of 4
// and p 16-B (float) / 8-B (bf16) aligned): the 1-tap kernels' HBM-bound streams.
template <typename T>
__device__ __forceinline__ void load4_as_float(const T* p, int64_t i, bool round, float (&v)[4]);
template <>
__device__ __forceinline__ void load4_as_float<float>(const float* p, int64_t i, bool round, float (&v)[4]) {
    const float4 t = __ldg(reinterpret_cast<const float4*>(p + i));
    v[0] = t.x, v[1] = t.y, v[2] = t.z, v[3] = t.w;
    if (round)
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = round_to_bf16(v[j]);
}
template <>
__device__ __forceinline__ void load4_as_float<uint16_t>(const uint16_t* p, int64_t i, bool, float (&v)[4]) {
    const uint2 t = __ldg(reinterpret_cast<const uint2*>(p + i));
    v[0] = bf16_bits_to_fp32(static_cast<uint16_t>(t.x & 0xffffu));
    v[1] = bf16_bits_to_fp32(static_cast<uint16_t>(t.x >> 16));
    v[2] = bf16_bits_to_fp32(static_cast<uint16_t>(t.y & 0xffffu));
    v[3] = bf16_bits_to_fp32(static_cast<uint16_t>(t.y >> 16));
}

__host__ __device__ constexpr int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---- programmatic dependent launch (PDL) ------------------------------------------------------
// The hot kernels launch with programmatic stream serialization: a kernel's CTAs may become
// resident while the previous kernel in the stream is finishing, run their prologue (barrier
// init, TMEM allocation, tensor-map prefetch), and block in pdl_wait() until that kernel has
// completed and its memory is visible. Every kernel launched through launch_pdl() calls
// pdl_wait() before its first global-memory access; pdl_trigger() lets the next kernel start
// launching (its own pdl_wait() still waits for this kernel's completion).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

inline bool pdl_enabled() {
    static const bool on = getenv("C1D_NO_PDL") == nullptr;  // dev A/B switch
    return on;
}

// Dev A/B switches read by the planners: each environment variable is read once per process (the
// planners run on every call, and getenv walks the environment).
enum class DevSwitch { kNoWres, kNoDbuf, kNoTail, kNoWs, kD8Carry, kNoStagger, kCount };
inline bool dev_switch(DevSwitch s) {
    static const bool on[static_cast<int>(DevSwitch::kCount)] = {
        getenv("C1D_NO_WRES") != nullptr, getenv("C1D_NO_DBUF") != nullptr, getenv("C1D_NO_TAIL") != nullptr,
        getenv("C1D_NO_WS") != nullptr, getenv("C1D_D8_CARRY") != nullptr, getenv("C1D_NO_STAGGER") != nullptr};
    return on[static_cast<int>(s)];
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace c1d
