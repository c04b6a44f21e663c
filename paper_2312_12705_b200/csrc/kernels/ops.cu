// K7-K12: HBM-bound kernels of the GPT block. Every kernel moves 16-byte vectors with
// coalesced row-contiguous access; row reductions are warp-shuffle + one smem pass; column
// reductions (LN/bias grads) go through per-block fp32 partials and a second deterministic pass.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "ops.h"
#include "rowops.cuh"
#include "pdl.cuh"
#include "sm100_ptx.cuh"
#include "tma_host.h"

namespace gptb200 {

namespace {

using namespace rowops;
using namespace ptx;

// Paired fp32 arithmetic (sm_100 FFMA2 / FMUL2 / FADD2: two fp32 lanes per instruction). The
// LayerNorm backward is instruction-bound at d = 2048, so its per-element math runs in pairs.
__device__ __forceinline__ uint64_t f2pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 f2unpack(uint64_t v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ uint64_t f2fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t f2mul(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t f2add(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// two packed bf16 -> an fp32 pair
__device__ __forceinline__ uint64_t bf2_to_f2(uint32_t w) {
  return f2pack(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
}


// vectors-per-thread choice: threads = (d/8)/vpt, a multiple of 32 and <= 1024
int pick_vpt(int d) {
  const int nvec = d / 8;
  for (int vpt = 1; vpt <= 8; ++vpt)
    if (nvec % vpt == 0 && (nvec / vpt) % 32 == 0 && nvec / vpt <= 1024) return vpt;
  return 0;
}

// ---------------------------------------------------------------- residual + dropout + LN
template <int VPT>
__global__ void resid_ln_kernel(ResidLnArgs a, DropDev dr) {
  __shared__ float red[64];
  const int row = blockIdx.x;
  const int d = a.d;
  float h[VPT][8];
  const size_t roff = static_cast<size_t>(row) * d;
  const bf16* rsrc = a.resid_pos_table ? a.resid + static_cast<size_t>(row % a.seq) * d : a.resid + roff;
#pragma unroll
  for (int v = 0; v < VPT; ++v) {
    const int c0 = (v * blockDim.x + threadIdx.x) * 8;
    float r[8];
    unpack8(*reinterpret_cast<const uint4*>(rsrc + c0), r);
    if (a.y) {
      float y[8];
      unpack8(*reinterpret_cast<const uint4*>(a.y + roff + c0), y);
      if (a.bias) {
        float b[8];
        unpack8(*reinterpret_cast<const uint4*>(a.bias + c0), b);
#pragma unroll
        for (int i = 0; i < 8; ++i) y[i] += b[i];
      }
      if (a.resid_pos_table) {  // embedding: dropout(word + position), Megatron's embedding dropout
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          y[i] += r[i];
          r[i] = 0.f;
        }
      }
      if (dr.on) {
        const uint32_t kb = keep8(dr, static_cast<int64_t>(roff) + c0);
#pragma unroll
        for (int i = 0; i < 8; ++i) y[i] = (kb >> i) & 1u ? y[i] * dr.scale : 0.f;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) h[v][i] = round_bf16(r[i] + y[i]);
      if (a.h_out) *reinterpret_cast<uint4*>(a.h_out + roff + c0) = pack8(h[v]);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) h[v][i] = r[i];
    }
  }
  if (!a.gamma) return;
  float s[1] = {0.f};
#pragma unroll
  for (int v = 0; v < VPT; ++v)
#pragma unroll
    for (int i = 0; i < 8; ++i) s[0] += h[v][i];
  block_sum<1>(s, red);
  const float mean = s[0] / d;
  float q[1] = {0.f};
#pragma unroll
  for (int v = 0; v < VPT; ++v)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float t = h[v][i] - mean;
      q[0] += t * t;
    }
  block_sum<1>(q, red);
  const float rstd = rsqrtf(q[0] / d + 1e-5f);
  if (threadIdx.x == 0) {
    a.mean[row] = mean;
    a.rstd[row] = rstd;
  }
#pragma unroll
  for (int v = 0; v < VPT; ++v) {
    const int c0 = (v * blockDim.x + threadIdx.x) * 8;
    float g[8], b[8], o[8];
    unpack8(*reinterpret_cast<const uint4*>(a.gamma + c0), g);
    unpack8(*reinterpret_cast<const uint4*>(a.beta + c0), b);
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i] = (h[v][i] - mean) * rstd * g[i] + b[i];
    *reinterpret_cast<uint4*>(a.ln_out + roff + c0) = pack8(o);
  }
}

// Warp-per-row variant for d <= 4096 (d % 256 == 0): lane owns VPL 16-byte vectors at columns
// (v*32 + lane)*8; both row reductions are warp shuffles (no block barriers).
template <int VPL>
__global__ void __launch_bounds__(256, 2) resid_ln_warp_kernel(ResidLnArgs a, DropDev dr) {
  pdl_trigger();  // launched through launch_pdl (pdl.cuh)
  pdl_wait();
  const int row = blockIdx.x * 8 + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (row >= a.rows) return;
  const int d = a.d;
  const size_t roff = static_cast<size_t>(row) * d;
  const bf16* rsrc = a.resid_pos_table ? a.resid + static_cast<size_t>(row % a.seq) * d : a.resid + roff;
  uint4 hp[VPL], yv[VPL];  // all row loads in flight first; hp then holds the new residual (bf16)
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    const int c0 = (v * 32 + lane) * 8;
    hp[v] = *reinterpret_cast<const uint4*>(rsrc + c0);
    if (a.y) yv[v] = *reinterpret_cast<const uint4*>(a.y + roff + c0);
  }
  uint64_t S = f2pack(0.f, 0.f);  // running row sum, fp32 pair
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    const int c0 = (v * 32 + lane) * 8;
    if (a.y) {
      float r[8], y[8];
      unpack8(hp[v], r);
      unpack8(yv[v], y);
      if (a.bias) {
        float b[8];
        unpack8(*reinterpret_cast<const uint4*>(a.bias + c0), b);
#pragma unroll
        for (int i = 0; i < 8; ++i) y[i] += b[i];
      }
      if (a.resid_pos_table) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          y[i] += r[i];
          r[i] = 0.f;
        }
      }
      if (dr.on) {
        const uint32_t kb = keep8(dr, static_cast<int64_t>(roff) + c0);
#pragma unroll
        for (int i = 0; i < 8; ++i) y[i] = (kb >> i) & 1u ? y[i] * dr.scale : 0.f;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) r[i] += y[i];
      hp[v] = pack8(r);
      if (a.h_out) *reinterpret_cast<uint4*>(a.h_out + roff + c0) = hp[v];
    }
    const uint32_t hw[4] = {hp[v].x, hp[v].y, hp[v].z, hp[v].w};
#pragma unroll
    for (int e2 = 0; e2 < 4; ++e2) S = f2add(S, bf2_to_f2(hw[e2]));
  }
  if (!a.gamma) return;
  const float2 sp = f2unpack(S);
  float sum = sp.x + sp.y;
  for (int off = 16; off; off >>= 1) sum += __shfl_xor_sync(0xffffffff, sum, off);
  const float mean = sum / d;
  const uint64_t NMEAN = f2pack(-mean, -mean);
  uint64_t Q = f2pack(0.f, 0.f);
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    const uint32_t hw[4] = {hp[v].x, hp[v].y, hp[v].z, hp[v].w};
#pragma unroll
    for (int e2 = 0; e2 < 4; ++e2) {
      const uint64_t T = f2add(bf2_to_f2(hw[e2]), NMEAN);
      Q = f2fma(T, T, Q);
    }
  }
  const float2 qp = f2unpack(Q);
  float q = qp.x + qp.y;
  for (int off = 16; off; off >>= 1) q += __shfl_xor_sync(0xffffffff, q, off);
  const float rstd = rsqrtf(q / d + 1e-5f);
  if (lane == 0) {
    a.mean[row] = mean;
    a.rstd[row] = rstd;
  }
  const uint64_t RS = f2pack(rstd, rstd), NMR = f2pack(-mean * rstd, -mean * rstd);
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    const int c0 = (v * 32 + lane) * 8;
    const uint4 gv = *reinterpret_cast<const uint4*>(a.gamma + c0);
    const uint4 bv = *reinterpret_cast<const uint4*>(a.beta + c0);
    const uint32_t hw[4] = {hp[v].x, hp[v].y, hp[v].z, hp[v].w};
    const uint32_t gw[4] = {gv.x, gv.y, gv.z, gv.w}, bw[4] = {bv.x, bv.y, bv.z, bv.w};
    float o[8];
#pragma unroll
    for (int e2 = 0; e2 < 4; ++e2) {  // (h*rstd - mean*rstd) * g + b
      const uint64_t O = f2fma(f2fma(bf2_to_f2(hw[e2]), RS, NMR), bf2_to_f2(gw[e2]), bf2_to_f2(bw[e2]));
      const float2 op = f2unpack(O);
      o[2 * e2] = op.x;
      o[2 * e2 + 1] = op.y;
    }
    *reinterpret_cast<uint4*>(a.ln_out + roff + c0) = pack8(o);
  }
}

// ---------------------------------------------------------------- LN backward (+residual, dropout')

// Phase A, rows of d <= 4096: one warp per row, shuffle-only reductions (no block barriers).
template <int VPL>
__global__ void __launch_bounds__(256, 4) ln_bwd_warp_kernel(LnBwdArgs a, DropDev dr) {
  const int row = blockIdx.x * 8 + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (row >= a.rows) return;
  const int d = a.d;
  const size_t roff = static_cast<size_t>(row) * d;
  float m1 = 0.f, m2 = 0.f, mu = 0.f, rs = 0.f;
  if (a.dy) {  // pass 1: the two row sums (x, dy re-read in pass 2 hit L1/L2)
    mu = a.mean[row];
    rs = a.rstd[row];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
      const int c0 = (v * 32 + lane) * 8;
      float x[8], dy[8], g[8];
      unpack8(*reinterpret_cast<const uint4*>(a.x + roff + c0), x);
      unpack8(*reinterpret_cast<const uint4*>(a.dy + roff + c0), dy);
      unpack8(*reinterpret_cast<const uint4*>(a.gamma + c0), g);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float gy = dy[i] * g[i];
        s1 += gy;
        s2 += gy * (x[i] - mu) * rs;
      }
    }
    for (int off = 16; off; off >>= 1) {
      s1 += __shfl_xor_sync(0xffffffff, s1, off);
      s2 += __shfl_xor_sync(0xffffffff, s2, off);
    }
    m1 = s1 / d;
    m2 = s2 / d;
  }
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    const int c0 = (v * 32 + lane) * 8;
    float dx[8];
    if (a.dy) {
      float x[8], dy[8], g[8];
      unpack8(*reinterpret_cast<const uint4*>(a.x + roff + c0), x);
      unpack8(*reinterpret_cast<const uint4*>(a.dy + roff + c0), dy);
      unpack8(*reinterpret_cast<const uint4*>(a.gamma + c0), g);
#pragma unroll
      for (int i = 0; i < 8; ++i) dx[i] = rs * (dy[i] * g[i] - m1 - (x[i] - mu) * rs * m2);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) dx[i] = 0.f;
    }
    if (a.resid_grad) {
      float r[8];
      unpack8(*reinterpret_cast<const uint4*>(a.resid_grad + roff + c0), r);
#pragma unroll
      for (int i = 0; i < 8; ++i) dx[i] += r[i];
    }
    const uint4 dxp = pack8(dx);
    if (a.dx) *reinterpret_cast<uint4*>(a.dx + roff + c0) = dxp;
    if (a.dxd && (dr.on || a.dxd != a.dx)) {
      uint4 op = dxp;
      if (dr.on) {
        float o[8];
        unpack8(dxp, o);
        const uint32_t kb = keep8(dr, static_cast<int64_t>(roff) + c0);
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = (kb >> i) & 1u ? o[i] * dr.scale : 0.f;
        op = pack8(o);
      }
      *reinterpret_cast<uint4*>(a.dxd + roff + c0) = op;
    }
  }
}

// Wide rows (d > 8192): phase A computes dx / dxd per row (no column state), phase B the column
// sums over 128-row chunks (column accumulators do not fit in registers at d = 12288 / 25600).
template <int VPT>
__global__ void ln_bwd_rows_kernel(LnBwdArgs a, DropDev dr) {
  __shared__ float red[64];
  const int d = a.d;
  const int row = blockIdx.x;
  const size_t roff = static_cast<size_t>(row) * d;
  float dx[VPT][8];
  if (a.dy) {
    const float mu = a.mean[row], rs = a.rstd[row];
    float s[2] = {0.f, 0.f};
#pragma unroll
    for (int v = 0; v < VPT; ++v) {
      const int c0 = (v * blockDim.x + threadIdx.x) * 8;
      float x[8], dy[8], g[8];
      unpack8(*reinterpret_cast<const uint4*>(a.x + roff + c0), x);
      unpack8(*reinterpret_cast<const uint4*>(a.dy + roff + c0), dy);
      unpack8(*reinterpret_cast<const uint4*>(a.gamma + c0), g);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float xh = (x[i] - mu) * rs, gy = dy[i] * g[i];
        s[0] += gy;
        s[1] += gy * xh;
        dx[v][i] = gy;  // stash g*dy; xh recomputed below
      }
    }
    block_sum<2>(s, red);
    const float m1 = s[0] / d, m2 = s[1] / d;
#pragma unroll
    for (int v = 0; v < VPT; ++v) {
      const int c0 = (v * blockDim.x + threadIdx.x) * 8;
      float x[8];
      unpack8(*reinterpret_cast<const uint4*>(a.x + roff + c0), x);
#pragma unroll
      for (int i = 0; i < 8; ++i) dx[v][i] = rs * (dx[v][i] - m1 - (x[i] - mu) * rs * m2);
    }
  } else {
#pragma unroll
    for (int v = 0; v < VPT; ++v)
#pragma unroll
      for (int i = 0; i < 8; ++i) dx[v][i] = 0.f;
  }
#pragma unroll
  for (int v = 0; v < VPT; ++v) {
    const int c0 = (v * blockDim.x + threadIdx.x) * 8;
    if (a.resid_grad) {
      float r[8];
      unpack8(*reinterpret_cast<const uint4*>(a.resid_grad + roff + c0), r);
#pragma unroll
      for (int i = 0; i < 8; ++i) dx[v][i] += r[i];
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) dx[v][i] = round_bf16(dx[v][i]);
    if (a.dx) *reinterpret_cast<uint4*>(a.dx + roff + c0) = pack8(dx[v]);
    if (a.dxd && (dr.on || a.dxd != a.dx)) {
      float o[8];
#pragma unroll
      const uint32_t kb = dr.on ? keep8(dr, static_cast<int64_t>(roff) + c0) : 0xFFu;
      for (int i = 0; i < 8; ++i) o[i] = dr.on ? ((kb >> i) & 1u ? dx[v][i] * dr.scale : 0.f) : dx[v][i];
      *reinterpret_cast<uint4*>(a.dxd + roff + c0) = pack8(o);
    }
  }
}

// Single-HBM-pass LayerNorm backward: a CTA owns kLnFuseRows rows. Pass 1 (warp per row): the
// two row reductions. Pass 2 (thread per 8 columns, rows walked in order): dx, dropout'(dx) and
// the dgamma/dbeta/dbias column partials in registers; x and dy come back from L2 (the CTA's
// 32-row slab was just read). HBM: 10 B/element instead of 16 for the two-kernel form.
constexpr int kLnFuseRows = 32;

__global__ void __launch_bounds__(256) ln_bwd_fused_kernel(LnBwdArgs a, DropDev dr, float* __restrict__ ws) {
  __shared__ float sm1[kLnFuseRows], sm2[kLnFuseRows], smu[kLnFuseRows], srs[kLnFuseRows];
  const int d = a.d;
  const int r0 = blockIdx.x * kLnFuseRows;
  const int nr = min(kLnFuseRows, a.rows - r0);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (a.dy) {
    for (int rr = warp; rr < nr; rr += 8) {
      const int row = r0 + rr;
      const size_t roff = static_cast<size_t>(row) * d;
      const float mu = a.mean[row], rs = a.rstd[row];
      float s1 = 0.f, s2 = 0.f;
      for (int c0 = lane * 8; c0 < d; c0 += 256) {
        float x[8], dy[8], g[8];
        unpack8(*reinterpret_cast<const uint4*>(a.x + roff + c0), x);
        unpack8(*reinterpret_cast<const uint4*>(a.dy + roff + c0), dy);
        unpack8(*reinterpret_cast<const uint4*>(a.gamma + c0), g);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float gy = dy[i] * g[i];
          s1 += gy;
          s2 += gy * (x[i] - mu) * rs;
        }
      }
      for (int off = 16; off; off >>= 1) {
        s1 += __shfl_xor_sync(0xffffffff, s1, off);
        s2 += __shfl_xor_sync(0xffffffff, s2, off);
      }
      if (lane == 0) {
        sm1[rr] = s1 / d;
        sm2[rr] = s2 / d;
        smu[rr] = mu;
        srs[rr] = rs;
      }
    }
  }
  __syncthreads();
  for (int c0 = threadIdx.x * 8; c0 < d; c0 += 256 * 8) {
    float g[8], ag[8], ab[8], as[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) ag[i] = ab[i] = as[i] = 0.f;
    if (a.dy) unpack8(*reinterpret_cast<const uint4*>(a.gamma + c0), g);
#pragma unroll 2
    for (int rr = 0; rr < nr; ++rr) {
      const size_t o = static_cast<size_t>(r0 + rr) * d + c0;
      float dx[8];
      if (a.dy) {
        const float mu = smu[rr], rs = srs[rr], m1 = sm1[rr], m2 = sm2[rr];
        float x[8], dy[8];
        unpack8(*reinterpret_cast<const uint4*>(a.x + o), x);
        unpack8(*reinterpret_cast<const uint4*>(a.dy + o), dy);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float xh = (x[i] - mu) * rs;
          dx[i] = rs * (dy[i] * g[i] - m1 - xh * m2);
          ag[i] += dy[i] * xh;
          ab[i] += dy[i];
        }
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) dx[i] = 0.f;
      }
      if (a.resid_grad) {
        float r[8];
        unpack8(*reinterpret_cast<const uint4*>(a.resid_grad + o), r);
#pragma unroll
        for (int i = 0; i < 8; ++i) dx[i] += r[i];
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) dx[i] = round_bf16(dx[i]);
      if (a.dx) *reinterpret_cast<uint4*>(a.dx + o) = pack8(dx);
      float od[8];
      const uint32_t kb = dr.on ? keep8(dr, static_cast<int64_t>(o)) : 0xFFu;
#pragma unroll
      for (int i = 0; i < 8; ++i) od[i] = dr.on ? ((kb >> i) & 1u ? dx[i] * dr.scale : 0.f) : dx[i];
      if (a.dxd && (dr.on || a.dxd != a.dx)) *reinterpret_cast<uint4*>(a.dxd + o) = pack8(od);
      if (a.dbias) {
        const uint4 q = pack8(od);  // bias grad sums the bf16 values that were stored
        float qv[8];
        unpack8(q, qv);
#pragma unroll
        for (int i = 0; i < 8; ++i) as[i] += qv[i];
      }
    }
    float* w = ws + static_cast<size_t>(blockIdx.x) * 3 * d;
    *reinterpret_cast<float4*>(w + c0) = make_float4(ag[0], ag[1], ag[2], ag[3]);
    *reinterpret_cast<float4*>(w + c0 + 4) = make_float4(ag[4], ag[5], ag[6], ag[7]);
    *reinterpret_cast<float4*>(w + d + c0) = make_float4(ab[0], ab[1], ab[2], ab[3]);
    *reinterpret_cast<float4*>(w + d + c0 + 4) = make_float4(ab[4], ab[5], ab[6], ab[7]);
    *reinterpret_cast<float4*>(w + 2 * d + c0) = make_float4(as[0], as[1], as[2], as[3]);
    *reinterpret_cast<float4*>(w + 2 * d + c0 + 4) = make_float4(as[4], as[5], as[6], as[7]);
  }
}

// Persistent, bulk-copy-staged LayerNorm backward (rows fill the GPU, d <= 4096, rows % R == 0).
// Each CTA walks the R-row slabs blockIdx.x, blockIdx.x + gridDim.x, ...; x and dy of a slab are
// contiguous, so one cp.async.bulk per tensor (x, dy and resid_grad) moves them into a shared-memory ring
// (mbarrier tx-count completion). Pass 1 (8 / R warps per row): the two row reductions from
// shared memory; pass 2 (thread per 8 columns): dx, dropout'(dx), dgamma/dbeta/dbias partials,
// accumulated in registers across all of the CTA's slabs. x and dy cross HBM exactly once (the
// 32-row fused form re-reads them from L2 and, with ~1000 resident slabs = 256 MB > L2, partly
// from HBM). Partials: ws[gridDim.x][3][d], reduced by reduce_partials_kernel in fixed order.
constexpr int kLnStages = 3;

template <int R, int NG>
__global__ void __launch_bounds__(256, 2) ln_bwd_stream_kernel(LnBwdArgs a, DropDev dr, float* __restrict__ ws,
                                                              int nslabs, int nst) {
  constexpr int W = 8 / R;  // warps per row in pass 1
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ uint64_t full[kLnStages];  // nst <= kLnStages stages in use
  __shared__ float part[R][W][2];
  __shared__ float smu[R], srs[R];
  const int d = a.d;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const uint32_t tile = static_cast<uint32_t>(R) * d * 2;  // bytes of one tensor's slab
  pdl_trigger();  // launched through launch_pdl (pdl.cuh): barrier init below is smem-only, but keep it simple
  pdl_wait();
  const int my = (nslabs - static_cast<int>(blockIdx.x) + static_cast<int>(gridDim.x) - 1) / gridDim.x;
  const int ntens = a.resid_grad ? 3 : 2;  // x, dy (, resid_grad) slabs per stage
  const size_t stage_bytes = static_cast<size_t>(ntens) * tile;
  auto sx = [&](int st) { return reinterpret_cast<const bf16*>(ring + st * stage_bytes); };
  auto sdy = [&](int st) { return reinterpret_cast<const bf16*>(ring + st * stage_bytes + tile); };
  auto srg = [&](int st) { return reinterpret_cast<const bf16*>(ring + st * stage_bytes + 2 * tile); };
  auto issue = [&](int i) {
    const int st = i % nst;
    const size_t off = static_cast<size_t>(blockIdx.x + static_cast<size_t>(i) * gridDim.x) * R * d;
    fence_proxy_async();
    mbar_arrive_expect_tx(&full[st], ntens * tile);
    bulk_load(ring + st * stage_bytes, a.x + off, tile, &full[st]);
    bulk_load(ring + st * stage_bytes + tile, a.dy + off, tile, &full[st]);
    if (a.resid_grad) bulk_load(ring + st * stage_bytes + 2 * tile, a.resid_grad + off, tile, &full[st]);
  };
  if (tid == 0) {
    for (int st = 0; st < nst; ++st) mbar_init(&full[st], 1);
    fence_mbar_init();
    for (int i = 0; i < nst && i < my; ++i) issue(i);
  }
  uint64_t g2[NG][4], AG[NG][4], AB[NG][4];  // gamma and the dgamma / dbeta partials, fp32 pairs
  uint64_t AS[NG][4];  // dbias partials
#pragma unroll
  for (int k = 0; k < NG; ++k) {
    const int c0 = tid * 8 + k * 2048;
    uint4 gv = make_uint4(0u, 0u, 0u, 0u);
    if (c0 < d) gv = *reinterpret_cast<const uint4*>(a.gamma + c0);
    const uint32_t gw[4] = {gv.x, gv.y, gv.z, gv.w};
#pragma unroll
    for (int e2 = 0; e2 < 4; ++e2) {
      g2[k][e2] = bf2_to_f2(gw[e2]);
      AG[k][e2] = AB[k][e2] = AS[k][e2] = f2pack(0.f, 0.f);
    }
  }
  __syncthreads();
  const int pr = warp / W, psub = warp % W;
  for (int i = 0; i < my; ++i) {
    const int st = i % nst;
    const int row0 = (blockIdx.x + i * gridDim.x) * R;
    mbar_wait(&full[st], (i / nst) & 1);
    const bf16* xs = sx(st);
    const bf16* dys = sdy(st);
    {  // pass 1: row reductions
      const int row = row0 + pr;
      const float mu = a.mean[row], rs = a.rstd[row];
      const uint64_t RS = f2pack(rs, rs), NMR = f2pack(-mu * rs, -mu * rs);
      uint64_t S1 = f2pack(0.f, 0.f), S2 = S1;
      for (int c0 = (psub * 32 + lane) * 8; c0 < d; c0 += W * 256) {
        const uint4 xv = *reinterpret_cast<const uint4*>(xs + pr * d + c0);
        const uint4 dv = *reinterpret_cast<const uint4*>(dys + pr * d + c0);
        const uint4 gv = *reinterpret_cast<const uint4*>(a.gamma + c0);
        const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w}, dw[4] = {dv.x, dv.y, dv.z, dv.w};
        const uint32_t gw[4] = {gv.x, gv.y, gv.z, gv.w};
#pragma unroll
        for (int e2 = 0; e2 < 4; ++e2) {
          const uint64_t GY = f2mul(bf2_to_f2(dw[e2]), bf2_to_f2(gw[e2]));
          S1 = f2add(S1, GY);
          S2 = f2fma(GY, f2fma(bf2_to_f2(xw[e2]), RS, NMR), S2);
        }
      }
      const float2 s1p = f2unpack(S1), s2p = f2unpack(S2);
      float s1 = s1p.x + s1p.y, s2 = s2p.x + s2p.y;
      for (int off = 16; off; off >>= 1) {
        s1 += __shfl_xor_sync(0xffffffff, s1, off);
        s2 += __shfl_xor_sync(0xffffffff, s2, off);
      }
      if (lane == 0) {
        part[pr][psub][0] = s1;
        part[pr][psub][1] = s2;
        if (psub == 0) {
          smu[pr] = mu;
          srs[pr] = rs;
        }
      }
    }
    __syncthreads();
    // pass 2: thread per 8 columns
#pragma unroll
    for (int k = 0; k < NG; ++k) {
      const int c0 = tid * 8 + k * 2048;
      if (c0 >= d) continue;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        float m1 = 0.f, m2 = 0.f;
#pragma unroll
        for (int w = 0; w < W; ++w) {
          m1 += part[r][w][0];
          m2 += part[r][w][1];
        }
        m1 /= d;
        m2 /= d;
        const float mu = smu[r], rs = srs[r];
        const size_t o = static_cast<size_t>(row0 + r) * d + c0;
        // dx = rs * (dy*g - xh*m2) - m1*rs, xh = x*rs - mu*rs; dgamma += dy*xh, dbeta += dy
        const uint64_t RS = f2pack(rs, rs), NMR = f2pack(-mu * rs, -mu * rs), NM2 = f2pack(-m2, -m2);
        const uint64_t NM1RS = f2pack(-m1 * rs, -m1 * rs);
        const uint4 xv = *reinterpret_cast<const uint4*>(xs + r * d + c0);
        const uint4 dv = *reinterpret_cast<const uint4*>(dys + r * d + c0);
        uint4 rv = make_uint4(0u, 0u, 0u, 0u);
        if (a.resid_grad) rv = *reinterpret_cast<const uint4*>(srg(st) + r * d + c0);
        const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w}, dw[4] = {dv.x, dv.y, dv.z, dv.w};
        const uint32_t rw[4] = {rv.x, rv.y, rv.z, rv.w};
        uint32_t dxw[4];
#pragma unroll
        for (int e2 = 0; e2 < 4; ++e2) {
          const uint64_t DY = bf2_to_f2(dw[e2]);
          const uint64_t XH = f2fma(bf2_to_f2(xw[e2]), RS, NMR);
          uint64_t DX = f2fma(f2fma(XH, NM2, f2mul(DY, g2[k][e2])), RS, NM1RS);
          AG[k][e2] = f2fma(DY, XH, AG[k][e2]);
          AB[k][e2] = f2add(AB[k][e2], DY);
          if (a.resid_grad) DX = f2add(DX, bf2_to_f2(rw[e2]));
          const float2 dxp = f2unpack(DX);
          dxw[e2] = pack_bf16(dxp.x, dxp.y);  // round-to-nearest bf16 pair (what is stored)
        }
        if (a.dx) *reinterpret_cast<uint4*>(a.dx + o) = make_uint4(dxw[0], dxw[1], dxw[2], dxw[3]);
        uint32_t odw[4] = {dxw[0], dxw[1], dxw[2], dxw[3]};
        if (dr.on) {
          const uint32_t kb = keep8(dr, static_cast<int64_t>(o));
#pragma unroll
          for (int e2 = 0; e2 < 4; ++e2) {
            const float2 f = unpack_bf16(dxw[e2]);
            odw[e2] = pack_bf16((kb >> (2 * e2)) & 1u ? f.x * dr.scale : 0.f,
                                (kb >> (2 * e2 + 1)) & 1u ? f.y * dr.scale : 0.f);
          }
        }
        if (a.dxd && (dr.on || a.dxd != a.dx))
          *reinterpret_cast<uint4*>(a.dxd + o) = make_uint4(odw[0], odw[1], odw[2], odw[3]);
        if (a.dbias) {  // bias grad sums the bf16 values that were stored
#pragma unroll
          for (int e2 = 0; e2 < 4; ++e2) AS[k][e2] = f2add(AS[k][e2], bf2_to_f2(odw[e2]));
        }
      }
    }
    __syncthreads();  // stage st and the row partials are free again
    if (tid == 0 && i + nst < my) issue(i + nst);
  }
#pragma unroll
  for (int k = 0; k < NG; ++k) {
    const int c0 = tid * 8 + k * 2048;
    if (c0 >= d) continue;
    float* w = ws + static_cast<size_t>(blockIdx.x) * 3 * d;
    float ag[8], ab[8], as[8];
#pragma unroll
    for (int e2 = 0; e2 < 4; ++e2) {
      const float2 gp = f2unpack(AG[k][e2]), bp = f2unpack(AB[k][e2]), sp = f2unpack(AS[k][e2]);
      ag[2 * e2] = gp.x;
      ag[2 * e2 + 1] = gp.y;
      ab[2 * e2] = bp.x;
      ab[2 * e2 + 1] = bp.y;
      as[2 * e2] = sp.x;
      as[2 * e2 + 1] = sp.y;
    }
    *reinterpret_cast<float4*>(w + c0) = make_float4(ag[0], ag[1], ag[2], ag[3]);
    *reinterpret_cast<float4*>(w + c0 + 4) = make_float4(ag[4], ag[5], ag[6], ag[7]);
    *reinterpret_cast<float4*>(w + d + c0) = make_float4(ab[0], ab[1], ab[2], ab[3]);
    *reinterpret_cast<float4*>(w + d + c0 + 4) = make_float4(ab[4], ab[5], ab[6], ab[7]);
    *reinterpret_cast<float4*>(w + 2 * d + c0) = make_float4(as[0], as[1], as[2], as[3]);
    *reinterpret_cast<float4*>(w + 2 * d + c0 + 4) = make_float4(as[4], as[5], as[6], as[7]);
  }
}

constexpr int kLnColRows = 64;

// Phase B: column sums over 64-row chunks of (dy*xhat, dy, dxd); one thread = 8 columns,
// 4 rows in flight per iteration. partial[chunk][3][d].
__global__ void __launch_bounds__(256) ln_bwd_cols_kernel(LnBwdArgs a, const bf16* __restrict__ dxd_src,
                                                          float* __restrict__ ws) {
  const int c0 = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
  const int d = a.d;
  if (c0 >= d) return;
  const int r0 = blockIdx.y * kLnColRows, r1 = min(r0 + kLnColRows, a.rows);
  float g[8], bb[8], sb[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) g[i] = bb[i] = sb[i] = 0.f;
#pragma unroll 4
  for (int r = r0; r < r1; ++r) {
    const size_t o = static_cast<size_t>(r) * d + c0;
    if (a.dy) {
      const float mu = a.mean[r], rs = a.rstd[r];
      float x[8], dy[8];
      unpack8(*reinterpret_cast<const uint4*>(a.x + o), x);
      unpack8(*reinterpret_cast<const uint4*>(a.dy + o), dy);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        g[i] += dy[i] * (x[i] - mu) * rs;
        bb[i] += dy[i];
      }
    }
    if (dxd_src) {
      float v[8];
      unpack8(*reinterpret_cast<const uint4*>(dxd_src + o), v);
#pragma unroll
      for (int i = 0; i < 8; ++i) sb[i] += v[i];
    }
  }
  float* w = ws + static_cast<size_t>(blockIdx.y) * 3 * d;
  *reinterpret_cast<float4*>(w + c0) = make_float4(g[0], g[1], g[2], g[3]);
  *reinterpret_cast<float4*>(w + c0 + 4) = make_float4(g[4], g[5], g[6], g[7]);
  *reinterpret_cast<float4*>(w + d + c0) = make_float4(bb[0], bb[1], bb[2], bb[3]);
  *reinterpret_cast<float4*>(w + d + c0 + 4) = make_float4(bb[4], bb[5], bb[6], bb[7]);
  *reinterpret_cast<float4*>(w + 2 * d + c0) = make_float4(sb[0], sb[1], sb[2], sb[3]);
  *reinterpret_cast<float4*>(w + 2 * d + c0 + 4) = make_float4(sb[4], sb[5], sb[6], sb[7]);
}

// out_k[c] += sum_b ws[b*stride + k*n + c] for k = 0..2 (outputs may be null). Block (32, 32):
// 32 consecutive columns x 32 partial-row lanes (lane ty sums rows ty, ty+32, ...), then a fixed
// tree over the 32 lanes: deterministic, and 1024 threads per 32 columns keep enough loads in
// flight for the ~1000-row partial matrices of the big-M steps.
constexpr int kRedLanes = 32;
__global__ void __launch_bounds__(32 * kRedLanes) reduce_partials_kernel(const float* __restrict__ ws, int nblocks,
                                                                          int stride, int n, float* out0, float* out1,
                                                                          float* out2) {
  __shared__ float red[3][kRedLanes][33];
  pdl_trigger();  // launched through launch_pdl (pdl.cuh)
  pdl_wait();
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + tx;
  float s0 = 0.f, s1 = 0.f, s2 = 0.f;
  if (c < n) {
#pragma unroll 4
    for (int b = ty; b < nblocks; b += kRedLanes) {
      const float* w = ws + static_cast<size_t>(b) * stride;
      s0 += w[c];
      if (out1) s1 += w[n + c];
      if (out2) s2 += w[2 * n + c];
    }
  }
  red[0][ty][tx] = s0;
  red[1][ty][tx] = s1;
  red[2][ty][tx] = s2;
  __syncthreads();
  for (int off = kRedLanes / 2; off > 0; off >>= 1) {  // fixed pairwise tree over the lanes
    if (ty < off) {
      red[0][ty][tx] += red[0][ty + off][tx];
      red[1][ty][tx] += red[1][ty + off][tx];
      red[2][ty][tx] += red[2][ty + off][tx];
    }
    __syncthreads();
  }
  if (ty == 0 && c < n) {
    if (out0) out0[c] += red[0][0][tx];
    if (out1) out1[c] += red[1][0][tx];
    if (out2) out2[c] += red[2][0][tx];
  }
}

// ---------------------------------------------------------------- column sums
constexpr int kColsumRows = 128;

__global__ void colsum_kernel(const bf16* __restrict__ X, int rows, int n, float* __restrict__ ws) {
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) * 2;
  if (c >= n) return;
  const int r0 = blockIdx.y * kColsumRows, r1 = min(r0 + kColsumRows, rows);
  float s0 = 0.f, s1 = 0.f;
  for (int r = r0; r < r1; ++r) {
    float2 v = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(X + static_cast<size_t>(r) * n + c));
    s0 += v.x;
    s1 += v.y;
  }
  ws[static_cast<size_t>(blockIdx.y) * n + c] = s0;
  ws[static_cast<size_t>(blockIdx.y) * n + c + 1] = s1;
}

// ---------------------------------------------------------------- embedding
__global__ void embed_lookup_kernel(const int32_t* __restrict__ tok, int rows, const bf16* __restrict__ wte,
                                    int vstart, int vrows, int d, bf16* __restrict__ out) {
  const int vpr = d / 8;
  const size_t n = static_cast<size_t>(rows) * vpr;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(i / vpr), c = static_cast<int>(i % vpr) * 8;
    const int t = tok[r] - vstart;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (t >= 0 && t < vrows) v = *reinterpret_cast<const uint4*>(wte + static_cast<size_t>(t) * d + c);
    *reinterpret_cast<uint4*>(out + static_cast<size_t>(r) * d + c) = v;
  }
}

__global__ void embed_bwd_wte_kernel(const int32_t* __restrict__ tok, int rows, const bf16* __restrict__ g,
                                     int vstart, int vrows, int d, float* __restrict__ dwte) {
  const int r = blockIdx.x;
  const int t = tok[r] - vstart;
  if (t < 0 || t >= vrows) return;
  for (int c = threadIdx.x * 2; c < d; c += blockDim.x * 2) {
    float2 v = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(g + static_cast<size_t>(r) * d + c));
    atomicAdd(dwte + static_cast<size_t>(t) * d + c, v.x);
    atomicAdd(dwte + static_cast<size_t>(t) * d + c + 1, v.y);
  }
}

__global__ void embed_bwd_wpe_kernel(const bf16* __restrict__ g, int rows, int d, int seq, float* __restrict__ dwpe) {
  const size_t n = static_cast<size_t>(seq) * d;
  const int nseq = rows / seq;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t pos = i / d, c = i % d;
    float s = 0.f;
    for (int b = 0; b < nseq; ++b) s += __bfloat162float(g[(static_cast<size_t>(b) * seq + pos) * d + c]);
    dwpe[i] += s;
  }
}

// ---------------------------------------------------------------- cross entropy
constexpr float kLog2eF = 1.4426950408889634f;

__global__ void xent_stats_kernel(const bf16* __restrict__ logits, int vcols, const int32_t* __restrict__ labels,
                                  int vstart, float* __restrict__ stats) {
  __shared__ float redm[32], reds[32];
  const int row = blockIdx.x;
  const bf16* x = logits + static_cast<size_t>(row) * vcols;
  float m = -INFINITY, s = 0.f;
  for (int c = threadIdx.x * 8; c < vcols; c += blockDim.x * 8) {
    float f[8];
    unpack8(*reinterpret_cast<const uint4*>(x + c), f);
    float lm = f[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) lm = fmaxf(lm, f[i]);
    const float nm = fmaxf(m, lm);
    float acc = s * exp2f((m - nm) * kLog2eF);
#pragma unroll
    for (int i = 0; i < 8; ++i) acc += exp2f((f[i] - nm) * kLog2eF);
    s = acc;
    m = nm;
  }
  for (int off = 16; off; off >>= 1) {
    const float om = __shfl_xor_sync(0xffffffff, m, off), os = __shfl_xor_sync(0xffffffff, s, off);
    const float nm = fmaxf(m, om);
    s = (m == -INFINITY ? 0.f : s * exp2f((m - nm) * kLog2eF)) + (om == -INFINITY ? 0.f : os * exp2f((om - nm) * kLog2eF));
    m = nm;
  }
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  if (lane == 0) {
    redm[warp] = m;
    reds[warp] = s;
  }
  __syncthreads();
  if (warp == 0) {
    m = lane < nw ? redm[lane] : -INFINITY;
    s = lane < nw ? reds[lane] : 0.f;
    for (int off = 16; off; off >>= 1) {
      const float om = __shfl_xor_sync(0xffffffff, m, off), os = __shfl_xor_sync(0xffffffff, s, off);
      const float nm = fmaxf(m, om);
      s = (m == -INFINITY ? 0.f : s * exp2f((m - nm) * kLog2eF)) + (om == -INFINITY ? 0.f : os * exp2f((om - nm) * kLog2eF));
      m = nm;
    }
    if (lane == 0) {
      const int t = labels[row] - vstart;
      stats[static_cast<size_t>(row) * 3 + 0] = m;
      stats[static_cast<size_t>(row) * 3 + 1] = s;
      stats[static_cast<size_t>(row) * 3 + 2] = (t >= 0 && t < vcols) ? __bfloat162float(x[t]) : 0.f;
    }
  }
}

// Row statistics from the LM-head GEMM's (max, sum exp) partials per 64 columns (GemmParams::
// rowstat_part): the same (max, sum exp(x - max), target logit) as xent_stats_kernel without re-reading
// the [rows, vcols] logits (only the target logit of each row).
__global__ void xent_stats_parts_kernel(const bf16* __restrict__ logits, const float2* __restrict__ parts, int vcols,
                                        const int32_t* __restrict__ labels, int vstart, float* __restrict__ stats) {
  __shared__ float redm[32], reds[32];
  const int row = blockIdx.x;
  const int np = vcols / 64;
  const float2* pr = parts + static_cast<size_t>(row) * np;
  auto combine = [](float& m, float& s, float om, float os) {
    const float nm = fmaxf(m, om);
    s = (m == -INFINITY ? 0.f : s * exp2f((m - nm) * kLog2eF)) + (om == -INFINITY ? 0.f : os * exp2f((om - nm) * kLog2eF));
    m = nm;
  };
  float m = -INFINITY, s = 0.f;
  for (int i = threadIdx.x; i < np; i += blockDim.x) {
    const float2 v = pr[i];
    combine(m, s, v.x, v.y);
  }
  for (int off = 16; off; off >>= 1)
    combine(m, s, __shfl_xor_sync(0xffffffff, m, off), __shfl_xor_sync(0xffffffff, s, off));
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  if (lane == 0) {
    redm[warp] = m;
    reds[warp] = s;
  }
  __syncthreads();
  if (warp == 0) {
    m = lane < nw ? redm[lane] : -INFINITY;
    s = lane < nw ? reds[lane] : 0.f;
    for (int off = 16; off; off >>= 1)
      combine(m, s, __shfl_xor_sync(0xffffffff, m, off), __shfl_xor_sync(0xffffffff, s, off));
    if (lane == 0) {
      const int t = labels[row] - vstart;
      stats[static_cast<size_t>(row) * 3 + 0] = m;
      stats[static_cast<size_t>(row) * 3 + 1] = s;
      stats[static_cast<size_t>(row) * 3 + 2] =
          (t >= 0 && t < vcols) ? __bfloat162float(logits[static_cast<size_t>(row) * vcols + t]) : 0.f;
    }
  }
}

__global__ void xent_finish_kernel(bf16* __restrict__ logits, int rows, int vcols, const int32_t* __restrict__ labels,
                                   int vstart, const float* __restrict__ all_stats, int tp, float scale,
                                   float* __restrict__ row_loss) {
  const int row = blockIdx.x;
  float gm = -INFINITY;
  for (int i = 0; i < tp; ++i) gm = fmaxf(gm, all_stats[(static_cast<size_t>(i) * rows + row) * 3]);
  float gs = 0.f, tgt = 0.f;
  for (int i = 0; i < tp; ++i) {
    const float* st = all_stats + (static_cast<size_t>(i) * rows + row) * 3;
    gs += st[1] * exp2f((st[0] - gm) * kLog2eF);
    tgt += st[2];
  }
  if (threadIdx.x == 0 && row_loss) row_loss[row] = logf(gs) + gm - tgt;
  const float inv = 1.f / gs;
  const int t = labels[row] - vstart;
  bf16* x = logits + static_cast<size_t>(row) * vcols;
  for (int c = threadIdx.x * 8; c < vcols; c += blockDim.x * 8) {
    float f[8];
    unpack8(*reinterpret_cast<const uint4*>(x + c), f);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float p = exp2f((f[i] - gm) * kLog2eF) * inv;
      if (c + i == t) p -= 1.f;
      f[i] = p * scale;
    }
    *reinterpret_cast<uint4*>(x + c) = pack8(f);
  }
}

// ---------------------------------------------------------------- Adam / init / casts
__global__ void adam_kernel(AdamArgs a) {
  const int64_t n4 = a.n / 4;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float4 p = reinterpret_cast<float4*>(a.master)[i];
    float4 m = reinterpret_cast<float4*>(a.m)[i];
    float4 v = reinterpret_cast<float4*>(a.v)[i];
    const float4 g = reinterpret_cast<const float4*>(a.grad)[i];
    float pp[4] = {p.x, p.y, p.z, p.w}, mm[4] = {m.x, m.y, m.z, m.w}, vv[4] = {v.x, v.y, v.z, v.w};
    const float gg[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      mm[k] = a.beta1 * mm[k] + (1.f - a.beta1) * gg[k];
      vv[k] = a.beta2 * vv[k] + (1.f - a.beta2) * gg[k] * gg[k];
      const float mh = mm[k] / a.bc1, vh = vv[k] / a.bc2;
      pp[k] -= a.lr * (mh / (sqrtf(vh) + a.eps) + a.weight_decay * pp[k]);
    }
    reinterpret_cast<float4*>(a.master)[i] = make_float4(pp[0], pp[1], pp[2], pp[3]);
    reinterpret_cast<float4*>(a.m)[i] = make_float4(mm[0], mm[1], mm[2], mm[3]);
    reinterpret_cast<float4*>(a.v)[i] = make_float4(vv[0], vv[1], vv[2], vv[3]);
    uint2 o;
    __nv_bfloat162 lo = __floats2bfloat162_rn(pp[0], pp[1]), hi = __floats2bfloat162_rn(pp[2], pp[3]);
    o.x = *reinterpret_cast<uint32_t*>(&lo);
    o.y = *reinterpret_cast<uint32_t*>(&hi);
    reinterpret_cast<uint2*>(a.param)[i] = o;
  }
}

__global__ void init_kernel(InitArgs a) {
  const int64_t n = a.rows * a.cols;
  const uint64_t key = mix64(a.seed ^ (static_cast<uint64_t>(static_cast<uint32_t>(a.tensor_id)) << 48));
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (a.scale == 0.f) {
      a.dst[i] = a.constant;
      continue;
    }
    const int64_t r = i / a.cols, c = i % a.cols;
    const int64_t gr = (r / a.rseg) * a.rstride + a.roff + r % a.rseg;
    const uint64_t gidx = static_cast<uint64_t>(gr * a.gcols + a.coff + c);
    int64_t s = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) s += static_cast<int64_t>(mix64(key + gidx * 4u + static_cast<uint64_t>(k)) >> 40);
    const int32_t ci = static_cast<int32_t>(s - (static_cast<int64_t>(2) << 24));
    a.dst[i] = __fmul_rn(__int2float_rn(ci), a.scale);
  }
}

__global__ void cast_f32_bf16_kernel(const float* __restrict__ s, bf16* __restrict__ d, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    d[i] = __float2bfloat16_rn(s[i]);
}

__global__ void cast_bf16_f32_kernel(const bf16* __restrict__ s, float* __restrict__ d, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    d[i] = __bfloat162float(s[i]);
}

__global__ void split_tokens_kernel(const int32_t* __restrict__ tok, int n, int s, int32_t* __restrict__ in,
                                    int32_t* __restrict__ lab) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const int b = r / s, i = r % s;
    in[r] = tok[b * (s + 1) + i];
    lab[r] = tok[b * (s + 1) + i + 1];
  }
}

__global__ void accumulate_sum_kernel(const float* __restrict__ x, int n, float* acc) {
  __shared__ float red[32];
  float s = 0.f;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += x[i];
  float v[1] = {s};
  block_sum<1>(v, red);
  if (threadIdx.x == 0) *acc += v[0];
}

int device_sms() { return device_sm_count(); }

int grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  if (g > 148 * 16) g = 148 * 16;
  return static_cast<int>(g < 1 ? 1 : g);
}

int status() { return cudaGetLastError() == cudaSuccess ? 0 : 3; }

}  // namespace

int resid_ln_fwd(const ResidLnArgs& a, cudaStream_t st) {
  const int vpt = pick_vpt(a.d);
  if (vpt == 0 || a.rows <= 0) return 1;
  if (a.drop.p > 0.f && a.drop.elem_base % 8 != 0) return 1;  // keep8 works on 8-aligned groups
  if (a.gamma && (!a.ln_out || !a.mean || !a.rstd)) return 1;
  const int threads = a.d / 8 / vpt;
  const DropDev dr = make_drop(a.drop);
  if (a.d % 256 == 0 && a.d <= 4096) {
    const int blocks = (a.rows + 7) / 8;
    switch (a.d / 256) {
#define WCASE(V) case V: launch_pdl(resid_ln_warp_kernel<V>, dim3(blocks), dim3(256), 0, st, a, dr); return status();
      WCASE(1) WCASE(2) WCASE(3) WCASE(4) WCASE(5) WCASE(6) WCASE(7) WCASE(8)
      WCASE(9) WCASE(10) WCASE(11) WCASE(12) WCASE(13) WCASE(14) WCASE(15) WCASE(16)
#undef WCASE
      default: break;
    }
  }
  switch (vpt) {
#define CASE(V) case V: resid_ln_kernel<V><<<a.rows, threads, 0, st>>>(a, dr); break;
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
#undef CASE
    default: return 1;
  }
  return status();
}

size_t ln_bwd_workspace_floats(int rows, int d) {
  return static_cast<size_t>((rows + kLnFuseRows - 1) / kLnFuseRows) * 3 * d;
}

int ln_bwd(const LnBwdArgs& a, cudaStream_t st) {
  const int vpt = pick_vpt(a.d);
  if (vpt == 0 || a.rows <= 0 || !a.workspace) return 1;
  if (a.drop.p > 0.f && a.dxd != nullptr && a.dxd == a.dx) return 1;  // would clobber dx
  if (a.drop.p > 0.f && a.drop.elem_base % 8 != 0) return 1;
  if (a.dy && (!a.gamma || !a.mean || !a.rstd || !a.x)) return 1;
  const DropDev dr = make_drop(a.drop);
  // fused single HBM pass when the row count alone fills the GPU (>= 2 waves of 32-row slabs);
  // wide-row / few-row shapes keep the row-parallel two-pass form
  const int blocks = (a.rows + kLnFuseRows - 1) / kLnFuseRows;
  static const bool two_pass_only = std::getenv("GPTB200_LN_BWD_TWO_PASS") != nullptr;  // A/B switch
  static const bool no_stream = std::getenv("GPTB200_LN_BWD_NO_STREAM") != nullptr;     // A/B switch
  const int R = a.d <= 2048 ? 4 : 2;
  if (blocks >= 2 * device_sms() && !two_pass_only && !no_stream && a.dy && a.d % 256 == 0 && a.d <= 4096 &&
      a.rows % R == 0) {
    const int nslabs = a.rows / R;
    const int grid = std::min(nslabs, 2 * device_sms());  // <= rows / 32: fits the workspace
    // ~96 KB ring (2 CTAs per SM): 3 stages of x/dy, or 2 stages of x/dy/resid_grad
    const int ntens = a.resid_grad ? 3 : 2;
    const int nst = a.resid_grad ? 2 : 3;
    const size_t smem = static_cast<size_t>(nst) * ntens * R * a.d * 2;
    // the largest ring either variant asks for
    constexpr int max_smem = 3 * 2 * 4 * 2048 * 2;
    if (ensure_dynamic_smem(reinterpret_cast<const void*>(ln_bwd_stream_kernel<4, 1>), max_smem) != 0 ||
        ensure_dynamic_smem(reinterpret_cast<const void*>(ln_bwd_stream_kernel<2, 2>), max_smem) != 0)
      return 3;
    count_variant(KV_LN_BWD_STREAM);
    if (R == 4)
      launch_pdl(ln_bwd_stream_kernel<4, 1>, dim3(grid), dim3(256), smem, st, a, dr, a.workspace, nslabs, nst);
    else
      launch_pdl(ln_bwd_stream_kernel<2, 2>, dim3(grid), dim3(256), smem, st, a, dr, a.workspace, nslabs, nst);
    const bool any = a.dgamma || a.dbeta || a.dbias;
    if (any)
      launch_pdl(reduce_partials_kernel, dim3((a.d + 31) / 32), dim3(32 * kRedLanes), 0, st, a.workspace, grid, 3 * a.d, a.d, a.dgamma,
                                                                          a.dbeta, a.dbias);
    return status();
  }
  if (blocks >= 2 * device_sms() && !two_pass_only) {
    count_variant(KV_LN_BWD_FUSED);
    ln_bwd_fused_kernel<<<blocks, 256, 0, st>>>(a, dr, a.workspace);
    const bool any = (a.dy && (a.dgamma || a.dbeta)) || a.dbias;
    if (any)
      launch_pdl(reduce_partials_kernel, dim3((a.d + 31) / 32), dim3(32 * kRedLanes), 0, st, a.workspace, blocks, 3 * a.d, a.d,
                                                                a.dy ? a.dgamma : nullptr, a.dy ? a.dbeta : nullptr,
                                                                a.dbias);
    return status();
  }
  count_variant(KV_LN_BWD_TWO_PASS);
  // phase A: dx (+ dropout'(dx)) per row
  if (a.dx || a.dxd) {
    if (a.d % 256 == 0 && a.d <= 4096) {
      const int blocks = (a.rows + 7) / 8;
      switch (a.d / 256) {
#define WCASE(V) case V: ln_bwd_warp_kernel<V><<<blocks, 256, 0, st>>>(a, dr); break;
        WCASE(1) WCASE(2) WCASE(3) WCASE(4) WCASE(5) WCASE(6) WCASE(7) WCASE(8)
        WCASE(9) WCASE(10) WCASE(11) WCASE(12) WCASE(13) WCASE(14) WCASE(15) WCASE(16)
#undef WCASE
        default: return 1;
      }
    } else {
      const int threads = a.d / 8 / vpt;
      switch (vpt) {
#define CASE(V) case V: ln_bwd_rows_kernel<V><<<a.rows, threads, 0, st>>>(a, dr); break;
        CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
#undef CASE
        default: return 1;
      }
    }
  }
  // phase B: column sums
  if (a.dbias) {
    const bf16* src = a.dxd ? a.dxd : (a.dx ? a.dx : nullptr);
    if (!src && !a.dy && !dr.on) src = a.resid_grad;  // no LN, no dropout: dxd == resid_grad
    if (!src) return 1;
    return ln_bwd_cols(a, src, st);
  }
  return ln_bwd_cols(a, nullptr, st);
}

int ln_bwd_cols(const LnBwdArgs& a, const bf16* dbias_src, cudaStream_t st) {
  const bool any = (a.dy && (a.dgamma || a.dbeta)) || (a.dbias && dbias_src);
  if (!any) return status();
  if (!a.workspace || a.rows <= 0 || a.d % 8 != 0) return 1;
  const int chunks = (a.rows + kLnColRows - 1) / kLnColRows;
  dim3 grid((a.d / 8 + 255) / 256, chunks);
  ln_bwd_cols_kernel<<<grid, 256, 0, st>>>(a, a.dbias ? dbias_src : nullptr, a.workspace);
  launch_pdl(reduce_partials_kernel, dim3((a.d + 31) / 32), dim3(32 * kRedLanes), 0, st, a.workspace, chunks, 3 * a.d, a.d,
                                                            a.dy ? a.dgamma : nullptr, a.dy ? a.dbeta : nullptr,
                                                            a.dbias ? a.dbias : nullptr);
  return status();
}

int reduce_col_partials(const float* partial, int nblocks, int n, float* out, cudaStream_t st) {
  if (nblocks <= 0 || n <= 0) return 1;
  launch_pdl(reduce_partials_kernel, dim3((n + 31) / 32), dim3(32 * kRedLanes), 0, st, partial, nblocks, n, n, out, nullptr, nullptr);
  return status();
}

size_t colsum_workspace_floats(int rows, int n) {
  return static_cast<size_t>((rows + kColsumRows - 1) / kColsumRows) * n;
}

int colsum_bf16(const bf16* X, int rows, int n, float* out, float* ws, cudaStream_t st) {
  if (n % 2 != 0 || rows <= 0) return 1;
  const int splits = (rows + kColsumRows - 1) / kColsumRows;
  dim3 grid((n / 2 + 255) / 256, splits);
  colsum_kernel<<<grid, 256, 0, st>>>(X, rows, n, ws);
  launch_pdl(reduce_partials_kernel, dim3((n + 31) / 32), dim3(32 * kRedLanes), 0, st, ws, splits, n, n, out, nullptr, nullptr);
  return status();
}

int embed_lookup(const int32_t* tokens, int rows, const bf16* wte, int vstart, int vrows, int d,
                 bf16* out, cudaStream_t st) {
  if (d % 8) return 1;
  embed_lookup_kernel<<<grid_for(static_cast<int64_t>(rows) * d / 8, 256), 256, 0, st>>>(tokens, rows, wte, vstart,
                                                                                       vrows, d, out);
  return status();
}

int embed_bwd(const int32_t* tokens, int rows, const bf16* g, int vstart, int vrows, int d, int seq,
              float* dwte, float* dwpe, cudaStream_t st) {
  embed_bwd_wte_kernel<<<rows, 256, 0, st>>>(tokens, rows, g, vstart, vrows, d, dwte);
  if (dwpe)
    embed_bwd_wpe_kernel<<<grid_for(static_cast<int64_t>(seq) * d, 256), 256, 0, st>>>(g, rows, d, seq, dwpe);
  return status();
}

int xent_stats(const bf16* logits, int rows, int vcols, const int32_t* labels, int vstart, float* stats,
               cudaStream_t st) {
  if (vcols % 8) return 1;
  xent_stats_kernel<<<rows, 512, 0, st>>>(logits, vcols, labels, vstart, stats);
  return status();
}

int xent_stats_from_parts(const bf16* logits, const float2* parts, int rows, int vcols, const int32_t* labels,
                          int vstart, float* stats, cudaStream_t st) {
  if (vcols % 64) return 1;
  xent_stats_parts_kernel<<<rows, 256, 0, st>>>(logits, parts, vcols, labels, vstart, stats);
  return status();
}

int xent_finish(bf16* logits, int rows, int vcols, const int32_t* labels, int vstart, const float* all_stats,
                int tp, float scale, float* row_loss, cudaStream_t st) {
  xent_finish_kernel<<<rows, 512, 0, st>>>(logits, rows, vcols, labels, vstart, all_stats, tp, scale, row_loss);
  return status();
}

int adam_step(const AdamArgs& a, cudaStream_t st) {
  if (a.n % 4) return 1;
  adam_kernel<<<grid_for(a.n / 4, 256), 256, 0, st>>>(a);
  return status();
}

int init_tensor(const InitArgs& a, cudaStream_t st) {
  init_kernel<<<grid_for(a.rows * a.cols, 256), 256, 0, st>>>(a);
  return status();
}

int split_tokens(const int32_t* tok, int nseq, int s, int32_t* inputs, int32_t* labels, cudaStream_t st) {
  const int n = nseq * s;
  split_tokens_kernel<<<grid_for(n, 256), 256, 0, st>>>(tok, n, s, inputs, labels);
  return status();
}

int accumulate_sum(const float* x, int n, float* acc, cudaStream_t st) {
  accumulate_sum_kernel<<<1, 1024, 0, st>>>(x, n, acc);
  return status();
}

int cast_f32_bf16(const float* s, bf16* d, int64_t n, cudaStream_t st) {
  cast_f32_bf16_kernel<<<grid_for(n, 256), 256, 0, st>>>(s, d, n);
  return status();
}

int cast_bf16_f32(const bf16* s, float* d, int64_t n, cudaStream_t st) {
  cast_bf16_f32_kernel<<<grid_for(n, 256), 256, 0, st>>>(s, d, n);
  return status();
}

}  // namespace gptb200
