// Device helpers shared by the HBM-bound kernels (ops.cu) and the sequence-parallel NVLS norm
// kernels (tp_nvls.cu): counter-based dropout decisions, bf16x8 pack/unpack, block sums.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "ops.h"

namespace gptb200 {
namespace rowops {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

struct DropDev {
  uint64_t key;
  uint32_t thr;
  float scale;
  int64_t base;
  bool on;
};

inline DropDev make_drop(const DropKey& k) {
  DropDev d{};
  d.on = k.p > 0.f;
  if (!d.on) return d;
  // identical to orc_dropout_keep's key schedule (host-side mix64 restated)
  auto mix = [](uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  };
  d.key = mix(k.seed ^ 0xD6E8FEB86659FD93ULL ^ (static_cast<uint64_t>(static_cast<uint32_t>(k.step)) << 40) ^
              (static_cast<uint64_t>(static_cast<uint32_t>(k.layer & 0xFFFF)) << 16) ^
              static_cast<uint64_t>(static_cast<uint32_t>(k.site)));
  d.thr = static_cast<uint32_t>(static_cast<double>(k.p) * 65536.0);
  d.scale = static_cast<float>(1.0 / (1.0 - static_cast<double>(k.p)));
  d.base = k.elem_base;
  return d;
}

// Dropout decision of one element: one 64-bit hash per 4 consecutive global elements, element e
// uses the 16-bit field (e % 4) (restated in oracle/gpt_oracle.c orc_dropout_keep).
__device__ __forceinline__ bool keep(const DropDev& d, int64_t elem) {
  const uint64_t e = static_cast<uint64_t>(d.base + elem);
  return static_cast<uint32_t>((mix64(d.key + (e >> 2)) >> (16 * (e & 3))) & 0xFFFFu) >= d.thr;
}

// Keep bits of 8 consecutive elements starting at `elem` (global index a multiple of 4): 2 hashes.
__device__ __forceinline__ uint32_t keep8(const DropDev& d, int64_t elem) {
  const uint64_t e = static_cast<uint64_t>(d.base + elem);
  uint32_t bits = 0;
#pragma unroll
  for (int hgrp = 0; hgrp < 2; ++hgrp) {
    const uint64_t h = mix64(d.key + ((e >> 2) + hgrp));
#pragma unroll
    for (int i = 0; i < 4; ++i)
      bits |= (static_cast<uint32_t>((h >> (16 * i)) & 0xFFFFu) >= d.thr ? 1u : 0u) << (4 * hgrp + i);
  }
  return bits;
}

__device__ __forceinline__ void unpack8(const uint4& v, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}

__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint4 v;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return v;
}

__device__ __forceinline__ float round_bf16(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

// Sum of `N` values across the block (blockDim.x multiple of 32, <= 1024).
template <int N>
__device__ __forceinline__ void block_sum(float (&v)[N], float* red /* >= 32*N */) {
#pragma unroll
  for (int i = 0; i < N; ++i)
    for (int off = 16; off; off >>= 1) v[i] += __shfl_xor_sync(0xffffffff, v[i], off);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < N; ++i) red[i * 32 + warp] = v[i];
  __syncthreads();
#pragma unroll
  for (int i = 0; i < N; ++i) {
    float t = lane < nw ? red[i * 32 + lane] : 0.f;
    for (int off = 16; off; off >>= 1) t += __shfl_xor_sync(0xffffffff, t, off);
    v[i] = t;
  }
}

}  // namespace rowops
}  // namespace gptb200
