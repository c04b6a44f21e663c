// Host-side TMA descriptor encoding shared by the tcgen05 kernels.
#pragma once

#include <cuda.h>

#include <cstdint>

namespace gptb200 {

// 2D bf16 tensor map over a row-major [outer][inner] matrix with leading dimension ld
// (elements), box {box_inner, box_outer}, 128B swizzle (box_inner * 2 <= 128).
bool make_tmap_bf16(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld,
                    uint32_t box_inner, uint32_t box_outer);

// 2D fp32 tensor map [outer][inner] (ld in elements), box {box_inner, box_outer}, no swizzle
// (used as the destination of bulk reduce-add).
bool make_tmap_f32(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld, uint32_t box_inner,
                   uint32_t box_outer);

int device_sm_count();

}  // namespace gptb200
