// Host-side TMA descriptor encoding shared by the tcgen05 kernels.
#pragma once

#include <cuda.h>

#include <cstdint>

namespace gptb200 {

// 2D bf16 tensor map over a row-major [outer][inner] matrix with leading dimension ld
// (elements), box {box_inner, box_outer}, 128B swizzle (box_inner * 2 <= 128).
bool make_tmap_bf16(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld,
                    uint32_t box_inner, uint32_t box_outer);

// 2D fp32 tensor map [outer][inner] (ld in elements), box {box_inner, box_outer}; no swizzle by
// default, 128B swizzle with sw128 (box_inner * 4 == 128).
bool make_tmap_f32(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld, uint32_t box_inner,
                   uint32_t box_outer, bool sw128 = false);

int device_sm_count();

}  // namespace gptb200
