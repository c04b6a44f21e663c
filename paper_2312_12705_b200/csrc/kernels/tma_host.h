// Host-side TMA descriptor encoding shared by the tcgen05 kernels.
#pragma once

#include <cuda.h>

#include <cstdint>

namespace gptb200 {

// 2D bf16 tensor map over a row-major [outer][inner] matrix with leading dimension ld
// (elements), box {box_inner, box_outer}, 128B swizzle (box_inner * 2 <= 128).
bool make_tmap_bf16(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld,
                    uint32_t box_inner, uint32_t box_outer);

// Same with 64B swizzle (box_inner * 2 <= 64): the 32-column tail chunk of a 160-wide head.
bool make_tmap_bf16_sw64(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld,
                         uint32_t box_inner, uint32_t box_outer);

// 2D fp32 tensor map [outer][inner] (ld in elements), box {box_inner, box_outer}; no swizzle by
// default, 128B swizzle with sw128 (box_inner * 4 == 128).
bool make_tmap_f32(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld, uint32_t box_inner,
                   uint32_t box_outer, bool sw128 = false);

// SM count of the current device (cached per device).
int device_sm_count();

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device): the attribute is per
// device, so a process driving sessions on several GPUs (or threads) sets it on each. Thread-safe.
// Returns 0 or the CUDA error code.
int ensure_dynamic_smem(const void* kernel, int bytes);

// Launch-variant counters (process-wide, all devices): which kernel variant each dispatcher
// chose, so tests can assert that a step at the production shapes ran the headline variants.
enum KernelVariant {
  KV_GEMM_SINGLE = 0,      // single-CTA 128xBN tiles
  KV_GEMM_PAIR_256,        // CTA-pair (cta_group::2) 256x256 tiles
  KV_GEMM_PAIR_512,        // CTA-pair 256x512 tiles
  KV_GEMM_KSPLIT,          // K-sliced accumulating fp32 GEMM (weight gradients)
  KV_ATTN_FWD_PERSISTENT,  // tcgen05 forward, persistent (hd <= 128)
  KV_ATTN_FWD_PER_BLOCK,   // tcgen05 forward, CTA per (q block, head)
  KV_ATTN_BWD_PER_BLOCK,   // tcgen05 backward, CTA per (kv block, head)
  KV_ATTN_BWD_PERSISTENT,  // tcgen05 backward, persistent
  KV_ATTN_BWD_HD64,        // tcgen05 backward, hd 64 kernel
  KV_ATTN_BWD_HD160,       // tcgen05 backward, hd 160 kernel
  KV_LN_BWD_STREAM,        // persistent bulk-copy LayerNorm backward (single HBM pass)
  KV_LN_BWD_FUSED,         // 32-row fused LayerNorm backward
  KV_LN_BWD_TWO_PASS,      // warp-per-row + column-sum LayerNorm backward
  KV_ATTN_FWD_TWO_Q,       // tcgen05 forward, two query tiles per CTA (hd 64 / 128, large grids)
  KV_NUM
};
void count_variant(int v);
void read_variants(int64_t* out, int n);
void reset_variants();

}  // namespace gptb200
