// L2 fp32 reduction throughput on B200 (the attention backward's dQ flush): 32 KB per "tile" per CTA,
// as scalar coalesced red.add (one 128-byte request per warp instruction), red.add.v4 (512 B per warp
// instruction) and cp.reduce.async.bulk (smem -> global add, one 32 KB bulk op per tile).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/red_bench tools/red_bench.cu && tools/red_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void red_scalar(float* dst, int tiles, int regions, int warps) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int t = 0; t < tiles; ++t) {
    float* base = dst + static_cast<size_t>((blockIdx.x + t) % regions) * 8192;  // 32 KB region
    for (int i = warp; i < 256; i += warps) atomicAdd(base + i * 32 + lane, 1.0f);
  }
}

__global__ void red_v4(float* dst, int tiles, int regions, int warps) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int t = 0; t < tiles; ++t) {
    float* base = dst + static_cast<size_t>((blockIdx.x + t) % regions) * 8192;
    for (int i = warp; i < 64; i += warps) {
      float* p = base + i * 128 + lane * 4;
      asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f)
                   : "memory");
    }
  }
}

__global__ void red_bulk(float* dst, int tiles, int regions, int chunks) {
  extern __shared__ __align__(128) float sm[];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = 1.f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
    const int cb = 32768 / chunks;
    for (int t = 0; t < tiles; ++t) {
      float* base = dst + static_cast<size_t>((blockIdx.x + t) % regions) * 8192;
      for (int c = 0; c < chunks; ++c)
        asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(
                         reinterpret_cast<char*>(base) + c * cb),
                     "r"(s + c * cb), "r"(cb)
                     : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int regions_max = 4096;
  float* dst;
  cudaMalloc(&dst, static_cast<size_t>(regions_max) * 32768);
  cudaMemset(dst, 0, static_cast<size_t>(regions_max) * 32768);
  cudaFuncSetAttribute(red_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int tiles = 200;
  for (int grid : {1, sms / 2, sms, 2 * sms}) {
    for (int regions : {16, 1024}) {
      for (int variant = 0; variant < 6; ++variant) {
        const int warps = variant == 0 ? 4 : variant == 1 ? 8 : variant == 2 ? 4 : 8;
        auto launch = [&] {
          if (variant == 0 || variant == 1) red_scalar<<<grid, warps * 32>>>(dst, tiles, regions, warps);
          else if (variant == 2 || variant == 3) red_v4<<<grid, warps * 32>>>(dst, tiles, regions, warps);
          else red_bulk<<<grid, 128, 32768>>>(dst, tiles, regions, variant == 4 ? 1 : 8);
        };
        launch();
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double bytes = static_cast<double>(grid) * tiles * 32768;
        const char* names[] = {"scalar 4w", "scalar 8w", "v4 4w", "v4 8w", "bulk 1x32K", "bulk 8x4K"};
        std::printf("grid %4d regions %4d %-10s: %8.1f GB/s  %7.0f ns per 32 KB tile per CTA\n", grid, regions,
                    names[variant], bytes / ms / 1e6, ms * 1e6 / tiles);
      }
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  std::printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
