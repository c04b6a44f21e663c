// tcgen05.mma issue-rate microbenchmark (B200): cycles per K=16 MMA for M=128 and N in {64,128,256},
// both operands from shared memory (SS) or A from TMEM (TS), optionally with 8 warps streaming
// st.shared in parallel (the attention backward's P/dS stores). Operand contents are garbage; only
// the pipe rate matters. One CTA per SM, all SMs busy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2312_12705_b200/csrc -o tools/mma_bench tools/mma_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "kernels/sm100_ptx.cuh"

using namespace gptb200;

constexpr int kIters = 2048;

template <int N, bool TS, bool STORES>
__global__ void __launch_bounds__(320, 1) mma_rate(unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) ptx::tmem_alloc<512>(&tslot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t a = ptx::smem_u32(sm), b = a + 65536;
  if (warp == 0) {
    constexpr uint32_t id = ptx::idesc_bf16_f32(128, N, false, false);
    const unsigned long long t0 = clock64();
    for (int i = 0; i < kIters; ++i) {
      const uint32_t k = (i & 7) * 32;
      if constexpr (TS)
        ptx::mma_bf16_ts_w(tmem + 256, tmem + (i & 7) * 8, ptx::smem_desc_sw128(b + k, 16, 1024), id, 1u);
      else
        ptx::mma_bf16_ss_w(tmem + 256, ptx::smem_desc_sw128(a + k, 16, 1024), ptx::smem_desc_sw128(b + k, 16, 1024),
                           id, 1u);
    }
    ptx::mma_commit_w(&bar);
    ptx::mbar_wait(&bar, 0);
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  } else if (STORES && warp >= 2) {
    // 8 warps: 16-byte stores over a 32 KB region (the attention backward's P^T/dS^T tile)
    uint4* p = reinterpret_cast<uint4*>(sm + 131072);
    const int t = threadIdx.x - 64;
    for (int i = 0; i < kIters / 4; ++i) {
#pragma unroll
      for (int u = 0; u < 8; ++u) p[(t * 8 + (u ^ (t & 7))) & 2047] = make_uint4(i, u, t, 0);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

template <int N, bool TS, bool STORES>
void run(const char* name, int sms, unsigned long long* d) {
  auto k = mma_rate<N, TS, STORES>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  k<<<sms, 320, 200 * 1024>>>(d);
  k<<<sms, 320, 200 * 1024>>>(d);
  cudaDeviceSynchronize();
  unsigned long long h[256];
  cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < sms; ++i) s += h[i];
  const double cyc = s / sms / kIters;
  const double floor = 128.0 * N / 256.0;
  std::printf("%-28s N=%3d: %6.1f cycles per K=16 MMA (floor %5.1f) -> %.2f of the tensor floor\n", name, N, cyc,
              floor, floor / cyc);
}


int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d;
  cudaMalloc(&d, 256 * 8);
  run<64, false, false>("SS", sms, d);
  run<128, false, false>("SS", sms, d);
  run<256, false, false>("SS", sms, d);
  run<64, true, false>("TS (A in TMEM)", sms, d);
  run<128, true, false>("TS (A in TMEM)", sms, d);
  run<256, true, false>("TS (A in TMEM)", sms, d);
  run<64, false, true>("SS + 8 warps st.shared", sms, d);
  run<128, false, true>("SS + 8 warps st.shared", sms, d);
  run<64, true, true>("TS + 8 warps st.shared", sms, d);
  std::printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}

