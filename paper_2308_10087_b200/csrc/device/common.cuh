// Shared device helpers for the sm_100a stage engine.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace gp {

constexpr uint32_t kColBits = 26;                  // packed edge: col | chunk << 26
constexpr uint32_t kColMask = (1u << kColBits) - 1;
constexpr uint32_t kMaxChunks = 64;                // done-set is a u64 bitmask
constexpr uint32_t kMaxWidth = 128;                // one float4 per lane per row

// splitmix64 finaliser (rng.hpp:9-14); the GPU derives every dropout decision
// from it exactly like DropMask::make (nn.hpp:112-127).
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t a, uint64_t b) { return mix64(mix64(a) ^ b); }
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t a, uint64_t b, uint64_t c) {
    return mix64(mix64(a, b) ^ c);
}

// Dropout mask of (epoch t, global layer l) over an N x cols input.
// keep(v, j) <=> hash_unit(mix64(key, v*cols + j)) < keep_prob, where
// key = mix64(seed, t, l) (nn.hpp:123-125). With k2 = mix64(key) the per-element
// hash is mix64(k2 ^ i); hash_unit(h) < keep <=> (h >> 11) < ceil(keep * 2^53),
// an exact integer test (hash_unit = (h>>11) * 2^-53, rng.hpp:27-29).
struct DropKey {
    uint64_t k2 = 0;
    uint64_t thr = 0;
    float scale = 1.f;      // float(1 / keep) (nn.hpp:120)
    uint32_t cols = 0;
    uint32_t enabled = 0;
};

__device__ __forceinline__ bool drop_keep(const DropKey& m, uint64_t idx) {
    return (mix64(m.k2 ^ idx) >> 11) < m.thr;
}

// DropMask::apply (nn.hpp:134-137): kept ? x * scale : 0, one IEEE multiply.
__device__ __forceinline__ float drop_apply(const DropKey& m, uint32_t v_orig, uint32_t j, float x) {
    if (!m.enabled) return x;
    const uint64_t idx = uint64_t(v_orig) * m.cols + j;
    return drop_keep(m, idx) ? __fmul_rn(x, m.scale) : 0.0f;
}

// Bit-exact counterparts of the reference's scalar float arithmetic: x86-64
// SSE, mul and add rounded separately (no FMA contraction at -O2).
__device__ __forceinline__ float mul_add(float acc, float a, float b) {
    return __fadd_rn(acc, __fmul_rn(a, b));
}

__device__ __forceinline__ float4 f4_zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }

__device__ __forceinline__ float4 shfl4(float4 v, int src) {
    float4 r;
    r.x = __shfl_sync(0xffffffffu, v.x, src);
    r.y = __shfl_sync(0xffffffffu, v.y, src);
    r.z = __shfl_sync(0xffffffffu, v.z, src);
    r.w = __shfl_sync(0xffffffffu, v.w, src);
    return r;
}

__device__ __forceinline__ float f4_get(const float4& v, int q) {
    return q == 0 ? v.x : (q == 1 ? v.y : (q == 2 ? v.z : v.w));
}

}  // namespace gp
