#include "kernels/tp_nvls.h"

#include <nccl_device.h>

#include <cstdint>
#include <cstdlib>

namespace gptb200 {

struct NvlsContext {
  void* base = nullptr;
  size_t bytes = 0;
  ncclWindow_t win = nullptr;
  ncclDevComm dev{};
  int max_ctas = 0;
  int nranks = 1;
};

namespace {

constexpr int kThreads = 512;
constexpr int kUnroll = 4;

__device__ __forceinline__ uint4 mc_ld_reduce_bf16x8(const uint4* p) {
  uint4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}

__device__ __forceinline__ void mc_st_bf16x8(uint4* p, uint4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.bf16x2 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}

// One CTA-indexed barrier before (every rank's partial sums are complete: each rank arrives
// after the producing kernel on its stream) and after (every rank's multicast stores landed
// before any rank reads its copy or overwrites the buffer).
__global__ void __launch_bounds__(kThreads) nvls_allreduce_kernel(ncclDevComm dev, ncclWindow_t win, size_t offset,
                                                                  size_t vec_per_rank) {
  ncclCoopCta coop;
  ncclLsaBarrierSession<ncclCoopCta> bar(coop, dev, ncclTeamTagLsa(), blockIdx.x, /*multimem=*/true);
  bar.sync(coop, cuda::memory_order_acq_rel);
  uint4* mc = static_cast<uint4*>(ncclGetLsaMultimemPointer(win, offset, dev)) +
              static_cast<size_t>(dev.lsaRank) * vec_per_rank;
  const size_t stride = static_cast<size_t>(gridDim.x) * kThreads;
  size_t i = static_cast<size_t>(blockIdx.x) * kThreads + threadIdx.x;
  for (; i + (kUnroll - 1) * stride < vec_per_rank; i += kUnroll * stride) {
    uint4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) v[u] = mc_ld_reduce_bf16x8(mc + i + u * stride);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) mc_st_bf16x8(mc + i + u * stride, v[u]);
  }
  for (; i < vec_per_rank; i += stride) mc_st_bf16x8(mc + i, mc_ld_reduce_bf16x8(mc + i));
  bar.sync(coop, cuda::memory_order_acq_rel);
}

}  // namespace

NvlsContext* nvls_create(ncclComm_t comm, size_t bytes, int max_ctas) {
  const char* env = std::getenv("GPTB200_TP_NVLS");
  if (env && env[0] == '0') return nullptr;
  int n = 0;
  if (ncclCommCount(comm, &n) != ncclSuccess || n < 2) return nullptr;
  if (ncclTeamLsa(comm).nRanks != n) return nullptr;  // TP group spans NVLink domains
  auto* c = new NvlsContext;
  c->nranks = n;
  c->max_ctas = max_ctas;
  c->bytes = (bytes + (2u << 20) - 1) / (2u << 20) * (2u << 20);
  if (ncclMemAlloc(&c->base, c->bytes) != ncclSuccess) {
    delete c;
    return nullptr;
  }
  if (ncclCommWindowRegister(comm, c->base, c->bytes, &c->win, NCCL_WIN_COLL_SYMMETRIC) != ncclSuccess) {
    ncclMemFree(c->base);
    delete c;
    return nullptr;
  }
  ncclDevCommRequirements reqs{};
  reqs.lsaMultimem = true;
  reqs.lsaBarrierCount = max_ctas;
  if (ncclDevCommCreate(comm, &reqs, &c->dev) != ncclSuccess) {
    ncclCommWindowDeregister(comm, c->win);
    ncclMemFree(c->base);
    delete c;
    return nullptr;
  }
  return c;
}

void nvls_destroy(NvlsContext* c, ncclComm_t comm) {
  if (!c) return;
  ncclDevCommDestroy(comm, &c->dev);
  ncclCommWindowDeregister(comm, c->win);
  ncclMemFree(c->base);
  delete c;
}

void* nvls_base(const NvlsContext* c) { return c ? c->base : nullptr; }
size_t nvls_bytes(const NvlsContext* c) { return c ? c->bytes : 0; }

int nvls_allreduce_bf16(NvlsContext* c, void* buf, size_t n, cudaStream_t st, int ctas) {
  if (!c) return 1;
  const auto off = static_cast<size_t>(static_cast<char*>(buf) - static_cast<char*>(c->base));
  if (static_cast<char*>(buf) < static_cast<char*>(c->base) || off + n * 2 > c->bytes || off % 16 ||
      n % (8 * static_cast<size_t>(c->nranks)))
    return 1;
  const size_t vec_per_rank = n / 8 / c->nranks;
  if (ctas <= 0 || ctas > c->max_ctas) ctas = c->max_ctas;
  nvls_allreduce_kernel<<<ctas, kThreads, 0, st>>>(c->dev, c->win, off, vec_per_rank);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

}  // namespace gptb200
