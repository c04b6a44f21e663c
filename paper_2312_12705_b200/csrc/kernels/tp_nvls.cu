#include "kernels/tp_nvls.h"

#include <nccl_device.h>

#include "kernels/rowops.cuh"

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
  int device = 0;
  // Deadlock-free grid caps per VPT instantiation (0 = not computed yet), see sp_grid().
  int fwd_cap[17] = {};
  int bwd_cap[17] = {};
  int ar_cap = 0;
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

using namespace rowops;

__device__ __forceinline__ void mc_st_bf16x8_v(void* p, uint4 v) { mc_st_bf16x8(static_cast<uint4*>(p), v); }

constexpr int kSpThreads = 256;

// one CTA per own row (grid-stride), 256 threads x VPT 8-wide column vectors
template <int VPT>
__global__ void __launch_bounds__(kSpThreads) sp_ln_fwd_kernel(ncclDevComm dev, ncclWindow_t win, SpLnFwdArgs a,
                                                               DropDev dr) {
  __shared__ float red[64];
  ncclCoopCta coop;
  ncclLsaBarrierSession<ncclCoopCta> bar(coop, dev, ncclTeamTagLsa(), a.bar_base + blockIdx.x,
                                         /*multimem=*/true);
  bar.sync(coop, cuda::memory_order_acq_rel);  // partials complete; every reader of the ln buffer done
  const bf16* ymc = a.y_off >= 0 ? static_cast<const bf16*>(ncclGetLsaMultimemPointer(win, a.y_off, dev)) : nullptr;
  bf16* lnmc = a.ln_off >= 0 ? static_cast<bf16*>(ncclGetLsaMultimemPointer(win, a.ln_off, dev)) : nullptr;
  const int d = a.d;
  for (int i = blockIdx.x; i < a.nrows; i += gridDim.x) {
    const int R = a.row0 + i;
    const size_t goff = static_cast<size_t>(R) * d, loff = static_cast<size_t>(i) * d;
    const bf16* rsrc = a.resid_pos_table ? a.resid + static_cast<size_t>(R % a.seq) * d : a.resid + loff;
    // issue every load of the row (the in-switch reductions take microseconds) before using any
    uint4 yraw[VPT], rraw[VPT];
#pragma unroll
    for (int v = 0; v < VPT; ++v) {
      const int c0 = (v * kSpThreads + threadIdx.x) * 8;
      if (c0 >= d) break;
      if (ymc) yraw[v] = mc_ld_reduce_bf16x8(reinterpret_cast<const uint4*>(ymc + goff + c0));
    }
#pragma unroll
    for (int v = 0; v < VPT; ++v) {
      const int c0 = (v * kSpThreads + threadIdx.x) * 8;
      if (c0 >= d) break;
      rraw[v] = *reinterpret_cast<const uint4*>(rsrc + c0);
    }
    float h[VPT][8];
    float sum = 0.f;
#pragma unroll
    for (int v = 0; v < VPT; ++v) {
      const int c0 = (v * kSpThreads + threadIdx.x) * 8;
      if (c0 >= d) break;
      float r[8];
      unpack8(rraw[v], r);
      if (ymc) {
        float y[8];
        unpack8(yraw[v], y);
        if (a.bias) {
          float b[8];
          unpack8(*reinterpret_cast<const uint4*>(a.bias + c0), b);
#pragma unroll
          for (int k = 0; k < 8; ++k) y[k] += b[k];
        }
        if (a.resid_pos_table) {  // embedding: dropout(word + position)
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            y[k] += r[k];
            r[k] = 0.f;
          }
        }
        if (dr.on) {
          const uint32_t kb = keep8(dr, static_cast<int64_t>(goff) + c0);
#pragma unroll
          for (int k = 0; k < 8; ++k) y[k] = (kb >> k) & 1u ? y[k] * dr.scale : 0.f;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) h[v][k] = round_bf16(r[k] + y[k]);
        if (a.h_out) *reinterpret_cast<uint4*>(a.h_out + loff + c0) = pack8(h[v]);
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) h[v][k] = r[k];
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) sum += h[v][k];
    }
    if (a.gamma) {
      float s1[1] = {sum};
      block_sum<1>(s1, red);
      const float mean = s1[0] / d;
      float q[1] = {0.f};
#pragma unroll
      for (int v = 0; v < VPT; ++v) {
        const int c0 = (v * kSpThreads + threadIdx.x) * 8;
        if (c0 >= d) break;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float t = h[v][k] - mean;
          q[0] += t * t;
        }
      }
      block_sum<1>(q, red);
      const float rstd = rsqrtf(q[0] / d + 1e-5f);
      if (threadIdx.x == 0) {
        a.mean[i] = mean;
        a.rstd[i] = rstd;
      }
#pragma unroll
      for (int v = 0; v < VPT; ++v) {
        const int c0 = (v * kSpThreads + threadIdx.x) * 8;
        if (c0 >= d) break;
        float g[8], b[8], o[8];
        unpack8(*reinterpret_cast<const uint4*>(a.gamma + c0), g);
        unpack8(*reinterpret_cast<const uint4*>(a.beta + c0), b);
#pragma unroll
        for (int k = 0; k < 8; ++k) o[k] = (h[v][k] - mean) * rstd * g[k] + b[k];
        mc_st_bf16x8_v(lnmc + goff + c0, pack8(o));
      }
    }
  }
  bar.sync(coop, cuda::memory_order_acq_rel);  // allgathered rows visible on every rank
}

template <int VPT>
__global__ void __launch_bounds__(kSpThreads) sp_ln_bwd_kernel(ncclDevComm dev, ncclWindow_t win, SpLnBwdArgs a,
                                                               DropDev dr) {
  __shared__ float red[64];
  ncclCoopCta coop;
  ncclLsaBarrierSession<ncclCoopCta> bar(coop, dev, ncclTeamTagLsa(), a.bar_base + blockIdx.x,
                                         /*multimem=*/true);
  bar.sync(coop, cuda::memory_order_acq_rel);
  const bf16* dymc = a.dy_off >= 0 ? static_cast<const bf16*>(ncclGetLsaMultimemPointer(win, a.dy_off, dev)) : nullptr;
  bf16* dyloc = a.dy_off >= 0 ? static_cast<bf16*>(ncclGetLocalPointer(win, a.dy_off)) : nullptr;
  bf16* dxdmc = a.dxd_off >= 0 ? static_cast<bf16*>(ncclGetLsaMultimemPointer(win, a.dxd_off, dev)) : nullptr;
  const int d = a.d;
  for (int i = blockIdx.x; i < a.nrows; i += gridDim.x) {
    const int R = a.row0 + i;
    const size_t goff = static_cast<size_t>(R) * d, loff = static_cast<size_t>(i) * d;
    float dx[VPT][8];
    if (dymc) {
      const float mu = a.mean[i], rs = a.rstd[i];
      float s[2] = {0.f, 0.f};
      uint4 dyraw[VPT];  // every in-switch reduction of the row in flight before the first use
#pragma unroll
      for (int v = 0; v < VPT; ++v) {
        const int c0 = (v * kSpThreads + threadIdx.x) * 8;
        if (c0 >= d) break;
        dyraw[v] = mc_ld_reduce_bf16x8(reinterpret_cast<const uint4*>(dymc + goff + c0));
      }
#pragma unroll
      for (int v = 0; v < VPT; ++v) {
        const int c0 = (v * kSpThreads + threadIdx.x) * 8;
        if (c0 >= d) break;
        const uint4 dyv = dyraw[v];
        *reinterpret_cast<uint4*>(dyloc + goff + c0) = dyv;  // reduced row kept for the column sums
        float x[8], dy[8], g[8];
        unpack8(dyv, dy);
        unpack8(*reinterpret_cast<const uint4*>(a.x + loff + c0), x);
        unpack8(*reinterpret_cast<const uint4*>(a.gamma + c0), g);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float gy = dy[k] * g[k];
          s[0] += gy;
          s[1] += gy * (x[k] - mu) * rs;
          dx[v][k] = gy;
        }
      }
      block_sum<2>(s, red);
      const float m1 = s[0] / d, m2 = s[1] / d;
#pragma unroll
      for (int v = 0; v < VPT; ++v) {
        const int c0 = (v * kSpThreads + threadIdx.x) * 8;
        if (c0 >= d) break;
        float x[8];
        unpack8(*reinterpret_cast<const uint4*>(a.x + loff + c0), x);
#pragma unroll
        for (int k = 0; k < 8; ++k) dx[v][k] = rs * (dx[v][k] - m1 - (x[k] - mu) * rs * m2);
      }
    } else {
#pragma unroll
      for (int v = 0; v < VPT; ++v)
#pragma unroll
        for (int k = 0; k < 8; ++k) dx[v][k] = 0.f;
    }
#pragma unroll
    for (int v = 0; v < VPT; ++v) {
      const int c0 = (v * kSpThreads + threadIdx.x) * 8;
      if (c0 >= d) break;
      if (a.resid_grad) {
        float r[8];
        unpack8(*reinterpret_cast<const uint4*>(a.resid_grad + loff + c0), r);
#pragma unroll
        for (int k = 0; k < 8; ++k) dx[v][k] += r[k];
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) dx[v][k] = round_bf16(dx[v][k]);
      if (a.dx) *reinterpret_cast<uint4*>(a.dx + loff + c0) = pack8(dx[v]);
      if (dxdmc) {
        float o[8];
        const uint32_t kb = dr.on ? keep8(dr, static_cast<int64_t>(goff) + c0) : 0xFFu;
#pragma unroll
        for (int k = 0; k < 8; ++k) o[k] = dr.on ? ((kb >> k) & 1u ? dx[v][k] * dr.scale : 0.f) : dx[v][k];
        mc_st_bf16x8_v(dxdmc + goff + c0, pack8(o));
      }
    }
  }
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
  cudaGetDevice(&c->device);
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
  reqs.lsaBarrierCount = kNvlsBarrierSets * max_ctas;
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

int64_t nvls_offset(const NvlsContext* c, const void* p) {
  if (!c || !p) return -1;
  const char* b = static_cast<const char*>(c->base);
  const char* q = static_cast<const char*>(p);
  return (q >= b && q < b + c->bytes) ? static_cast<int64_t>(q - b) : -1;
}

namespace {
// Every CTA of an SP kernel waits at an LSA barrier for the CTA with the same index on every peer,
// so a kernel only makes progress once ALL its CTAs are resident on every rank. Kernels of the two
// barrier sets (step / SP stream and the recompute stream) and NCCL's own spin-waiting kernels
// (DP reduce-scatter / allgather, TP grad allreduce on the comm stream) can be in flight together:
// if one rank's SMs fill with set-0 CTAs while a peer's fill with set-1 or NCCL CTAs, the wait is
// cyclic. Cap each set at half of the CTAs the GPU can hold for this kernel outside a reserve of
// SMs for NCCL, so all concurrently active spin-waiting grids are co-resident whatever the order.
constexpr int kNcclReservedSms = 24;

template <typename Kernel>
int deadlock_free_cap(Kernel k, int device, int threads = kSpThreads) {
  int sms = 0, per_sm = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || sms <= 0) return 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, threads, 0) != cudaSuccess || per_sm <= 0)
    per_sm = 1;
  const int usable = sms > 2 * kNcclReservedSms ? sms - kNcclReservedSms : sms / 2;
  return per_sm * (usable / kNvlsBarrierSets) > 0 ? per_sm * (usable / kNvlsBarrierSets) : 1;
}

int sp_grid(NvlsContext* c, int nrows, int vpt, bool fwd) {
  int& cap = fwd ? c->fwd_cap[vpt] : c->bwd_cap[vpt];
  if (cap == 0) {
    switch (vpt) {
#define CAP(V) \
  case V: cap = fwd ? deadlock_free_cap(sp_ln_fwd_kernel<V>, c->device) : deadlock_free_cap(sp_ln_bwd_kernel<V>, c->device); break;
      CAP(1) CAP(2) CAP(3) CAP(4) CAP(5) CAP(6) CAP(7) CAP(8) CAP(9) CAP(10) CAP(11) CAP(12) CAP(13) CAP(14)
      CAP(15) CAP(16)
#undef CAP
      default: cap = 1;
    }
    if (cap > c->max_ctas) cap = c->max_ctas;
  }
  return nrows < cap ? nrows : cap;
}
}  // namespace

int sp_ln_fwd(NvlsContext* c, const SpLnFwdArgs& a_in, cudaStream_t st) {
  if (!c || a_in.nrows <= 0 || a_in.d % 8 != 0 || a_in.d > 16 * kSpThreads * 8) return 1;
  if (a_in.lane_set < 0 || a_in.lane_set >= kNvlsBarrierSets) return 1;
  SpLnFwdArgs a = a_in;
  a.bar_base = a.lane_set * c->max_ctas;
  if (a.drop.p > 0.f && a.drop.elem_base % 8 != 0) return 1;
  if (a.gamma && (a.ln_off < 0 || !a.beta || !a.mean || !a.rstd)) return 1;
  const int vpt = (a.d / 8 + kSpThreads - 1) / kSpThreads;
  const DropDev dr = make_drop(a.drop);
  const int grid = sp_grid(c, a.nrows, vpt, true);
  switch (vpt) {
#define SPF(V) case V: sp_ln_fwd_kernel<V><<<grid, kSpThreads, 0, st>>>(c->dev, c->win, a, dr); break;
    SPF(1) SPF(2) SPF(3) SPF(4) SPF(5) SPF(6) SPF(7) SPF(8) SPF(9) SPF(10) SPF(11) SPF(12) SPF(13) SPF(14)
    SPF(15) SPF(16)
#undef SPF
    default: return 1;
  }
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

int sp_ln_bwd(NvlsContext* c, const SpLnBwdArgs& a_in, cudaStream_t st) {
  if (!c || a_in.nrows <= 0 || a_in.d % 8 != 0 || a_in.d > 16 * kSpThreads * 8 || !a_in.workspace) return 1;
  if (a_in.lane_set < 0 || a_in.lane_set >= kNvlsBarrierSets) return 1;
  SpLnBwdArgs a = a_in;
  a.bar_base = a.lane_set * c->max_ctas;
  if (a.drop.p > 0.f && a.drop.elem_base % 8 != 0) return 1;
  if (a.dy_off >= 0 && (!a.x || !a.gamma || !a.mean || !a.rstd)) return 1;
  const int vpt = (a.d / 8 + kSpThreads - 1) / kSpThreads;
  const DropDev dr = make_drop(a.drop);
  const int grid = sp_grid(c, a.nrows, vpt, false);
  switch (vpt) {
#define SPB(V) case V: sp_ln_bwd_kernel<V><<<grid, kSpThreads, 0, st>>>(c->dev, c->win, a, dr); break;
    SPB(1) SPB(2) SPB(3) SPB(4) SPB(5) SPB(6) SPB(7) SPB(8) SPB(9) SPB(10) SPB(11) SPB(12) SPB(13) SPB(14)
    SPB(15) SPB(16)
#undef SPB
    default: return 1;
  }
  if (cudaPeekAtLastError() != cudaSuccess) return 2;
  // column sums over the own rows (reduced dy in this rank's copy of P, dxd rows in its copy)
  LnBwdArgs cb;
  cb.rows = a.nrows;
  cb.d = a.d;
  cb.x = a.x;
  cb.dy = a.dy_off >= 0 ? reinterpret_cast<const bf16*>(static_cast<const char*>(c->base) + a.dy_off) +
                              static_cast<size_t>(a.row0) * a.d
                        : nullptr;
  cb.mean = a.mean;
  cb.rstd = a.rstd;
  cb.dgamma = a.dgamma;
  cb.dbeta = a.dbeta;
  cb.dbias = a.dbias;
  cb.workspace = a.workspace;
  const bf16* dbias_src = a.dxd_off >= 0 ? reinterpret_cast<const bf16*>(static_cast<const char*>(c->base) + a.dxd_off) +
                                               static_cast<size_t>(a.row0) * a.d
                                         : nullptr;
  if (a.dbias && !dbias_src) return 1;
  return ln_bwd_cols(cb, dbias_src, st) == 0 ? 0 : 2;
}

int nvls_allreduce_bf16(NvlsContext* c, void* buf, size_t n, cudaStream_t st, int ctas) {
  if (!c) return 1;
  const auto off = static_cast<size_t>(static_cast<char*>(buf) - static_cast<char*>(c->base));
  if (static_cast<char*>(buf) < static_cast<char*>(c->base) || off + n * 2 > c->bytes || off % 16 ||
      n % (8 * static_cast<size_t>(c->nranks)))
    return 1;
  const size_t vec_per_rank = n / 8 / c->nranks;
  if (c->ar_cap == 0) {
    c->ar_cap = deadlock_free_cap(nvls_allreduce_kernel, c->device, kThreads);
    if (c->ar_cap > c->max_ctas) c->ar_cap = c->max_ctas;
  }
  if (ctas <= 0 || ctas > c->ar_cap) ctas = c->ar_cap;
  nvls_allreduce_kernel<<<ctas, kThreads, 0, st>>>(c->dev, c->win, off, vec_per_rank);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

}  // namespace gptb200
