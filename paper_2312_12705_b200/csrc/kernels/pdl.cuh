// Programmatic dependent launch (PDL) between consecutive kernels of the step stream.
//
// A kernel launched with launch_pdl() may start while the previous kernel in the stream is still
// draining: its CTAs run their smem / TMEM / mbarrier / tensor-map prologue, then block in
// pdl_wait() (griddepcontrol.wait: the previous grid has completed and its memory is visible)
// before touching global memory. pdl_trigger() (griddepcontrol.launch_dependents) lets the next
// grid be scheduled once every CTA of this grid has issued it, so the next kernel's launch and
// prologue overlap this kernel's tail. Every kernel launched through launch_pdl() must call
// pdl_wait() before its first global-memory access. GPTB200_PDL=0 turns the attribute off (A/B).
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

namespace gptb200 {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("GPTB200_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace gptb200
