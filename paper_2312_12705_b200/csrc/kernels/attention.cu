// K5/K6: causal flash attention forward and backward (online softmax, warp-shuffle row
// reductions), bf16 in/out with fp32 accumulation, head dims 64/128/160.
//
// Layout (one TP rank): qkv[M, 3*dt] with M = b*s tokens and dt = heads_local*hd; q heads occupy
// columns [0, dt), k heads [dt, 2dt), v heads [2dt, 3dt), each head hd contiguous. Output o[M, dt];
// lse[b, heads_local, s] in log2 units (lse2 = max2 + log2(sum)), consumed by the backward pass.
// This is the FA2 algorithm on warp-level m16n8k16 tensor-core MMA; scores never touch HBM.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "attention.h"
#include "mma_sync.cuh"

namespace gptb200 {

using namespace wmma16;

namespace {

constexpr float kLog2e = 1.4426950408889634f;

// ----------------------------------------------------------------------------- forward
// CTA = 128 query rows of one (sequence, head); 8 warps x 16 rows; KV tiles of 64 rows,
// double-buffered through cp.async. Rows padded by 8 elements -> conflict-free ldmatrix.
template <int HD>
struct FwdCfg {
  static constexpr int BM = 128, BN = 64, LD = HD + 8;
  static constexpr int kSmem = (BM + 4 * BN) * LD * 2;
};

template <int HD>
__global__ void __launch_bounds__(256, 1)
    flash_fwd_kernel(const __nv_bfloat16* __restrict__ qkv, __nv_bfloat16* __restrict__ out,
                     float* __restrict__ lse, int s, int ht, float scale_log2) {
  using Cfg = FwdCfg<HD>;
  constexpr int BM = Cfg::BM, BN = Cfg::BN, LD = Cfg::LD;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(smem_raw);
  __nv_bfloat16* sK = sQ + BM * LD;  // [2][BN][LD]
  __nv_bfloat16* sV = sK + 2 * BN * LD;

  const int q_blk = gridDim.x - 1 - blockIdx.x;  // heaviest causal blocks first
  const int b = blockIdx.y / ht, h = blockIdx.y % ht;
  const int dt = ht * HD, ldq = 3 * dt;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const size_t row0 = static_cast<size_t>(b) * s;
  const int q0 = q_blk * BM;
  const __nv_bfloat16* gQ = qkv + (row0 + q0) * ldq + h * HD;
  const __nv_bfloat16* gK = qkv + row0 * ldq + dt + h * HD;
  const __nv_bfloat16* gV = qkv + row0 * ldq + 2 * dt + h * HD;
  constexpr int CPR = HD / 8;  // 16B chunks per row

  for (int i = threadIdx.x; i < BM * CPR; i += 256) {
    int r = i / CPR, c = i % CPR;
    cp_async16(ptx_smem(sQ + r * LD + c * 8), gQ + static_cast<size_t>(r) * ldq + c * 8);
  }
  auto load_kv = [&](int j, int buf) {
    const __nv_bfloat16* k = gK + static_cast<size_t>(j * BN) * ldq;
    const __nv_bfloat16* v = gV + static_cast<size_t>(j * BN) * ldq;
    for (int i = threadIdx.x; i < BN * CPR; i += 256) {
      int r = i / CPR, c = i % CPR;
      cp_async16(ptx_smem(sK + (buf * BN + r) * LD + c * 8), k + static_cast<size_t>(r) * ldq + c * 8);
      cp_async16(ptx_smem(sV + (buf * BN + r) * LD + c * 8), v + static_cast<size_t>(r) * ldq + c * 8);
    }
  };
  load_kv(0, 0);
  cp_async_commit();

  float o_acc[HD / 8][4];
#pragma unroll
  for (int n = 0; n < HD / 8; ++n)
#pragma unroll
    for (int e = 0; e < 4; ++e) o_acc[n][e] = 0.f;
  float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};
  uint32_t qf[HD / 16][4];

  const int n_tiles = (q0 + BM) / BN;
  const int my_row_lo = q0 + warp * 16;  // first query row of this warp
  const int g = lane / 4, t4 = lane % 4;

  for (int j = 0; j < n_tiles; ++j) {
    const int buf = j & 1;
    if (j + 1 < n_tiles) load_kv(j + 1, buf ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (j == 0) {
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk)
        ldsm_x4(qf[kk], ptx_smem(sQ + (warp * 16 + a_row(lane)) * LD + kk * 16 + a_col(lane)));
    }
    const int kv0 = j * BN;
    if (kv0 <= my_row_lo + 15) {  // otherwise the whole tile is masked for this warp
      float sc[BN / 8][4];
#pragma unroll
      for (int n = 0; n < BN / 8; ++n)
#pragma unroll
        for (int e = 0; e < 4; ++e) sc[n][e] = 0.f;
      const __nv_bfloat16* kb = sK + buf * BN * LD;
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
#pragma unroll
        for (int np = 0; np < BN / 16; ++np) {
          uint32_t bf[4];
          ldsm_x4(bf, ptx_smem(kb + (np * 16 + bn_row(lane)) * LD + kk * 16 + bn_col(lane)));
          mma_bf16(sc[2 * np], qf[kk], bf[0], bf[1]);
          mma_bf16(sc[2 * np + 1], qf[kk], bf[2], bf[3]);
        }
      }
      // scale, causal mask, online softmax (rows g and g+8 of this warp's 16)
      const bool diag = kv0 + BN - 1 > my_row_lo;
      float mx[2] = {m_run[0], m_run[1]};
#pragma unroll
      for (int n = 0; n < BN / 8; ++n)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float v = sc[n][e] * scale_log2;
          if (diag) {
            int col = kv0 + n * 8 + 2 * t4 + (e & 1);
            int row = my_row_lo + g + (e >> 1) * 8;
            if (col > row) v = -INFINITY;
          }
          sc[n][e] = v;
          mx[e >> 1] = fmaxf(mx[e >> 1], v);
        }
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffff, mx[r], 1));
        mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffff, mx[r], 2));
      }
      float corr[2], rs[2] = {0.f, 0.f};
#pragma unroll
      for (int r = 0; r < 2; ++r) corr[r] = exp2f(m_run[r] - mx[r]);  // m_run=-inf -> 0
      uint32_t pf[BN / 16][4];
#pragma unroll
      for (int n = 0; n < BN / 8; ++n) {
        float p0 = exp2f(sc[n][0] - mx[0]), p1 = exp2f(sc[n][1] - mx[0]);
        float p2 = exp2f(sc[n][2] - mx[1]), p3 = exp2f(sc[n][3] - mx[1]);
        rs[0] += p0 + p1;
        rs[1] += p2 + p3;
        pf[n / 2][(n & 1) * 2 + 0] = pack_bf16(p0, p1);
        pf[n / 2][(n & 1) * 2 + 1] = pack_bf16(p2, p3);
      }
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        l_run[r] = l_run[r] * corr[r] + rs[r];
        m_run[r] = mx[r];
      }
#pragma unroll
      for (int n = 0; n < HD / 8; ++n) {
        o_acc[n][0] *= corr[0];
        o_acc[n][1] *= corr[0];
        o_acc[n][2] *= corr[1];
        o_acc[n][3] *= corr[1];
      }
      const __nv_bfloat16* vb = sV + buf * BN * LD;
#pragma unroll
      for (int kk = 0; kk < BN / 16; ++kk) {
        // A fragment of P for kv columns [16kk, 16kk+16): n-tiles 2kk (a0,a1) and 2kk+1 (a2,a3)
        uint32_t a[4] = {pf[kk][0], pf[kk][1], pf[kk][2], pf[kk][3]};
#pragma unroll
        for (int np = 0; np < HD / 16; ++np) {
          uint32_t bf[4];
          ldsm_x4_t(bf, ptx_smem(vb + (kk * 16 + bt_row(lane)) * LD + np * 16 + bt_col(lane)));
          mma_bf16(o_acc[2 * np], a, bf[0], bf[1]);
          mma_bf16(o_acc[2 * np + 1], a, bf[2], bf[3]);
        }
      }
    }
    __syncthreads();
  }
  // epilogue: normalise, write o and lse
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    l_run[r] += __shfl_xor_sync(0xffffffff, l_run[r], 1);
    l_run[r] += __shfl_xor_sync(0xffffffff, l_run[r], 2);
  }
  const float inv0 = 1.f / l_run[0], inv1 = 1.f / l_run[1];
  const int r0 = q0 + warp * 16 + g;
  __nv_bfloat16* o0 = out + (row0 + r0) * static_cast<size_t>(dt) + h * HD;
  __nv_bfloat16* o1 = o0 + 8 * static_cast<size_t>(dt);
#pragma unroll
  for (int n = 0; n < HD / 8; ++n) {
    *reinterpret_cast<uint32_t*>(o0 + n * 8 + 2 * t4) = pack_bf16(o_acc[n][0] * inv0, o_acc[n][1] * inv0);
    *reinterpret_cast<uint32_t*>(o1 + n * 8 + 2 * t4) = pack_bf16(o_acc[n][2] * inv1, o_acc[n][3] * inv1);
  }
  if (t4 == 0) {
    float* L = lse + (static_cast<size_t>(b) * ht + h) * s;
    L[r0] = m_run[0] + log2f(l_run[0]);
    L[r0 + 8] = m_run[1] + log2f(l_run[1]);
  }
}

// ----------------------------------------------------------------------------- backward
// Preprocess: D[b,h,q] = sum_c dO[q,c] * O[q,c]; zero the fp32 dQ accumulator.
template <int HD>
__global__ void flash_bwd_pre_kernel(const __nv_bfloat16* __restrict__ o,
                                     const __nv_bfloat16* __restrict__ dout, float* __restrict__ D,
                                     float* __restrict__ dq_acc, int s, int ht, int M) {
  const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  const int dt = ht * HD;
  if (warp_global >= M * ht) return;
  const int row = warp_global / ht, h = warp_global % ht;
  const __nv_bfloat16* op = o + static_cast<size_t>(row) * dt + h * HD;
  const __nv_bfloat16* dp = dout + static_cast<size_t>(row) * dt + h * HD;
  float acc = 0.f;
  for (int c = lane * 2; c < HD; c += 64) {
    float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(op + c));
    float2 bb = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(dp + c));
    acc += a.x * bb.x + a.y * bb.y;
  }
  for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffff, acc, off);
  const int b = row / s, q = row % s;
  if (lane == 0) D[(static_cast<size_t>(b) * ht + h) * s + q] = acc;
  float* dqa = dq_acc + static_cast<size_t>(row) * dt + h * HD;
  for (int c = lane; c < HD; c += 32) dqa[c] = 0.f;
}

// CTA = 64 kv rows of one (sequence, head), 4 warps x 16 kv rows; loops over 32-row q tiles
// from the diagonal to the end. dK/dV accumulate in registers; dQ through fp32 atomics.
template <int HD>
struct BwdCfg {
  static constexpr int BN = 64, BQ = 32, LD = HD + 8, LDS = BQ + 8;
  static constexpr int kSmem = (2 * BN * LD + 2 * 2 * BQ * LD + BN * LDS) * 2 + 2 * 2 * BQ * 4;
};

template <int HD>
__global__ void __launch_bounds__(128, 2)
    flash_bwd_kernel(const __nv_bfloat16* __restrict__ qkv, const __nv_bfloat16* __restrict__ dout,
                     const float* __restrict__ lse, const float* __restrict__ D,
                     float* __restrict__ dq_acc, __nv_bfloat16* __restrict__ dqkv, int s, int ht,
                     float scale_log2, float scale) {
  using Cfg = BwdCfg<HD>;
  constexpr int BN = Cfg::BN, BQ = Cfg::BQ, LD = Cfg::LD, LDS = Cfg::LDS;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  __nv_bfloat16* sK = reinterpret_cast<__nv_bfloat16*>(smem_raw);
  __nv_bfloat16* sV = sK + BN * LD;
  __nv_bfloat16* sQ = sV + BN * LD;          // [2][BQ][LD]
  __nv_bfloat16* sdO = sQ + 2 * BQ * LD;     // [2][BQ][LD]
  __nv_bfloat16* sdS = sdO + 2 * BQ * LD;    // [BN][LDS]  (dS^T)
  float* sL = reinterpret_cast<float*>(sdS + BN * LDS);  // [2][BQ]
  float* sD = sL + 2 * BQ;                               // [2][BQ]

  const int kv_blk = blockIdx.x;
  const int b = blockIdx.y / ht, h = blockIdx.y % ht;
  const int dt = ht * HD, ldq = 3 * dt;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int g = lane / 4, t4 = lane % 4;
  const size_t row0 = static_cast<size_t>(b) * s;
  const int kv0 = kv_blk * BN;
  constexpr int CPR = HD / 8;

  const __nv_bfloat16* gQ = qkv + row0 * ldq + h * HD;
  const __nv_bfloat16* gK = qkv + (row0 + kv0) * ldq + dt + h * HD;
  const __nv_bfloat16* gV = qkv + (row0 + kv0) * ldq + 2 * dt + h * HD;
  const __nv_bfloat16* gdO = dout + row0 * dt + h * HD;
  const float* gL = lse + (static_cast<size_t>(b) * ht + h) * s;
  const float* gD = D + (static_cast<size_t>(b) * ht + h) * s;

  for (int i = threadIdx.x; i < BN * CPR; i += 128) {
    int r = i / CPR, c = i % CPR;
    cp_async16(ptx_smem(sK + r * LD + c * 8), gK + static_cast<size_t>(r) * ldq + c * 8);
    cp_async16(ptx_smem(sV + r * LD + c * 8), gV + static_cast<size_t>(r) * ldq + c * 8);
  }
  auto load_q = [&](int qt, int buf) {
    const int qr = qt * BQ;
    for (int i = threadIdx.x; i < BQ * CPR; i += 128) {
      int r = i / CPR, c = i % CPR;
      cp_async16(ptx_smem(sQ + (buf * BQ + r) * LD + c * 8), gQ + static_cast<size_t>(qr + r) * ldq + c * 8);
      cp_async16(ptx_smem(sdO + (buf * BQ + r) * LD + c * 8), gdO + static_cast<size_t>(qr + r) * dt + c * 8);
    }
    if (threadIdx.x < BQ) {
      sL[buf * BQ + threadIdx.x] = gL[qr + threadIdx.x];
      sD[buf * BQ + threadIdx.x] = gD[qr + threadIdx.x];
    }
  };
  const int qt_first = kv0 / BQ;
  const int qt_end = s / BQ;
  load_q(qt_first, 0);
  cp_async_commit();

  float dk[HD / 8][4], dv[HD / 8][4];
#pragma unroll
  for (int n = 0; n < HD / 8; ++n)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[n][e] = dv[n][e] = 0.f;

  const int my_kv = kv0 + warp * 16;  // first kv row of this warp

  for (int qt = qt_first; qt < qt_end; ++qt) {
    const int buf = (qt - qt_first) & 1;
    if (qt + 1 < qt_end) load_q(qt + 1, buf ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const int q0 = qt * BQ;
    const __nv_bfloat16* q_s = sQ + buf * BQ * LD;
    const __nv_bfloat16* do_s = sdO + buf * BQ * LD;
    // S^T = K Q^T and dP^T = V dO^T   (16 kv x 32 q per warp)
    float st[BQ / 8][4], dpt[BQ / 8][4];
#pragma unroll
    for (int n = 0; n < BQ / 8; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) st[n][e] = dpt[n][e] = 0.f;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      uint32_t ka[4], va[4];
      ldsm_x4(ka, ptx_smem(sK + (warp * 16 + a_row(lane)) * LD + kk * 16 + a_col(lane)));
      ldsm_x4(va, ptx_smem(sV + (warp * 16 + a_row(lane)) * LD + kk * 16 + a_col(lane)));
#pragma unroll
      for (int np = 0; np < BQ / 16; ++np) {
        uint32_t qb[4], ob[4];
        ldsm_x4(qb, ptx_smem(q_s + (np * 16 + bn_row(lane)) * LD + kk * 16 + bn_col(lane)));
        ldsm_x4(ob, ptx_smem(do_s + (np * 16 + bn_row(lane)) * LD + kk * 16 + bn_col(lane)));
        mma_bf16(st[2 * np], ka, qb[0], qb[1]);
        mma_bf16(st[2 * np + 1], ka, qb[2], qb[3]);
        mma_bf16(dpt[2 * np], va, ob[0], ob[1]);
        mma_bf16(dpt[2 * np + 1], va, ob[2], ob[3]);
      }
    }
    // P^T, dS^T (rows = kv g / g+8 of this warp, cols = q)
    uint32_t pa[BQ / 16][4], dsa[BQ / 16][4];
#pragma unroll
    for (int n = 0; n < BQ / 8; ++n) {
      float p[4], ds[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int qc = n * 8 + 2 * t4 + (e & 1);
        const int kvr = my_kv + g + (e >> 1) * 8;
        float pv = exp2f(st[n][e] * scale_log2 - sL[buf * BQ + qc]);
        if (q0 + qc < kvr) pv = 0.f;
        p[e] = pv;
        ds[e] = pv * (dpt[n][e] - sD[buf * BQ + qc]);
      }
      pa[n / 2][(n & 1) * 2 + 0] = pack_bf16(p[0], p[1]);
      pa[n / 2][(n & 1) * 2 + 1] = pack_bf16(p[2], p[3]);
      dsa[n / 2][(n & 1) * 2 + 0] = pack_bf16(ds[0], ds[1]);
      dsa[n / 2][(n & 1) * 2 + 1] = pack_bf16(ds[2], ds[3]);
      // stash dS^T (bf16) for the dQ product
      __nv_bfloat16* dsrow = sdS + (warp * 16 + g) * LDS + n * 8 + 2 * t4;
      *reinterpret_cast<uint32_t*>(dsrow) = dsa[n / 2][(n & 1) * 2 + 0];
      *reinterpret_cast<uint32_t*>(dsrow + 8 * LDS) = dsa[n / 2][(n & 1) * 2 + 1];
    }
    // dV += P^T dO ; dK += dS^T Q     (k = q rows)
#pragma unroll
    for (int kk = 0; kk < BQ / 16; ++kk) {
#pragma unroll
      for (int np = 0; np < HD / 16; ++np) {
        uint32_t ob[4], qb[4];
        ldsm_x4_t(ob, ptx_smem(do_s + (kk * 16 + bt_row(lane)) * LD + np * 16 + bt_col(lane)));
        ldsm_x4_t(qb, ptx_smem(q_s + (kk * 16 + bt_row(lane)) * LD + np * 16 + bt_col(lane)));
        mma_bf16(dv[2 * np], pa[kk], ob[0], ob[1]);
        mma_bf16(dv[2 * np + 1], pa[kk], ob[2], ob[3]);
        mma_bf16(dk[2 * np], dsa[kk], qb[0], qb[1]);
        mma_bf16(dk[2 * np + 1], dsa[kk], qb[2], qb[3]);
      }
    }
    __syncthreads();  // sdS complete
    // dQ[q, :] += dS K : warp -> q m-tile (warp & 1), hd half (warp >> 1)
    {
      const int mt = warp & 1, half = warp >> 1;
      constexpr int NH = HD / 2;  // columns per warp
      float dq[NH / 8][4];
#pragma unroll
      for (int n = 0; n < NH / 8; ++n)
#pragma unroll
        for (int e = 0; e < 4; ++e) dq[n][e] = 0.f;
#pragma unroll
      for (int kk = 0; kk < BN / 16; ++kk) {
        uint32_t a[4];
        ldsm_x4_t(a, ptx_smem(sdS + (kk * 16 + at_row(lane)) * LDS + mt * 16 + at_col(lane)));
#pragma unroll
        for (int np = 0; np < NH / 16; ++np) {
          uint32_t kb[4];
          ldsm_x4_t(kb, ptx_smem(sK + (kk * 16 + bt_row(lane)) * LD + half * NH + np * 16 + bt_col(lane)));
          mma_bf16(dq[2 * np], a, kb[0], kb[1]);
          mma_bf16(dq[2 * np + 1], a, kb[2], kb[3]);
        }
      }
      float* d0 = dq_acc + (row0 + q0 + mt * 16 + g) * static_cast<size_t>(dt) + h * HD + half * NH;
      float* d1 = d0 + 8 * static_cast<size_t>(dt);
#pragma unroll
      for (int n = 0; n < NH / 8; ++n) {
        atomicAdd(d0 + n * 8 + 2 * t4, dq[n][0]);
        atomicAdd(d0 + n * 8 + 2 * t4 + 1, dq[n][1]);
        atomicAdd(d1 + n * 8 + 2 * t4, dq[n][2]);
        atomicAdd(d1 + n * 8 + 2 * t4 + 1, dq[n][3]);
      }
    }
    __syncthreads();  // before the next tile overwrites sQ/sdO/sdS
  }
  // write dK (scaled) and dV
  const size_t kr = row0 + my_kv + g;
  __nv_bfloat16* dk0 = dqkv + kr * ldq + dt + h * HD;
  __nv_bfloat16* dv0 = dqkv + kr * ldq + 2 * dt + h * HD;
#pragma unroll
  for (int n = 0; n < HD / 8; ++n) {
    *reinterpret_cast<uint32_t*>(dk0 + n * 8 + 2 * t4) = pack_bf16(dk[n][0] * scale, dk[n][1] * scale);
    *reinterpret_cast<uint32_t*>(dk0 + 8 * static_cast<size_t>(ldq) + n * 8 + 2 * t4) =
        pack_bf16(dk[n][2] * scale, dk[n][3] * scale);
    *reinterpret_cast<uint32_t*>(dv0 + n * 8 + 2 * t4) = pack_bf16(dv[n][0], dv[n][1]);
    *reinterpret_cast<uint32_t*>(dv0 + 8 * static_cast<size_t>(ldq) + n * 8 + 2 * t4) =
        pack_bf16(dv[n][2], dv[n][3]);
  }
}

// dq (bf16, scaled) into the q section of dqkv.
__global__ void flash_bwd_dq_kernel(const float* __restrict__ dq_acc, __nv_bfloat16* __restrict__ dqkv,
                                    int M, int dt, float scale) {
  const size_t n = static_cast<size_t>(M) * dt / 4;
  const int ldq = 3 * dt;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    size_t e = i * 4;
    size_t row = e / dt, col = e % dt;
    float4 v = reinterpret_cast<const float4*>(dq_acc)[i];
    uint2 pk;
    pk.x = pack_bf16(v.x * scale, v.y * scale);
    pk.y = pack_bf16(v.z * scale, v.w * scale);
    *reinterpret_cast<uint2*>(dqkv + row * ldq + col) = pk;
  }
}

template <int HD>
int fwd_impl(const AttnShape& a, const __nv_bfloat16* qkv, __nv_bfloat16* out, float* lse,
             cudaStream_t st) {
  using Cfg = FwdCfg<HD>;
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(flash_fwd_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem);
    init = true;
  }
  dim3 grid(a.seq / Cfg::BM, a.batch * a.heads);
  const float scale_log2 = kLog2e / sqrtf(static_cast<float>(HD));
  flash_fwd_kernel<HD><<<grid, 256, Cfg::kSmem, st>>>(qkv, out, lse, a.seq, a.heads, scale_log2);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

template <int HD>
int bwd_impl(const AttnShape& a, const __nv_bfloat16* qkv, const __nv_bfloat16* out,
             const __nv_bfloat16* dout, const float* lse, float* D, float* dq_acc,
             __nv_bfloat16* dqkv, cudaStream_t st, bool d_ready) {
  using Cfg = BwdCfg<HD>;
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(flash_bwd_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem);
    init = true;
  }
  const int M = a.batch * a.seq;
  const int warps = M * a.heads;
  if (d_ready)
    cudaMemsetAsync(dq_acc, 0, static_cast<size_t>(M) * a.heads * HD * sizeof(float), st);
  else
    flash_bwd_pre_kernel<HD><<<(warps + 7) / 8, 256, 0, st>>>(out, dout, D, dq_acc, a.seq, a.heads, M);
  const float scale = 1.f / sqrtf(static_cast<float>(HD));
  if (HD != 160) {
    // tcgen05 main kernel (attention_sm100.cu); TMEM cannot hold dK+dV+S+dP at hd=160
    const int r = flash_attn_bwd_tc_main(a, qkv, dout, lse, D, dq_acc, dqkv, st);
    if (r != 0) return r;
  } else {
    dim3 grid(a.seq / Cfg::BN, a.batch * a.heads);
    flash_bwd_kernel<HD><<<grid, 128, Cfg::kSmem, st>>>(qkv, dout, lse, D, dq_acc, dqkv, a.seq, a.heads,
                                                        scale * kLog2e, scale);
  }
  const int dt = a.heads * HD;
  flash_bwd_dq_kernel<<<1184, 256, 0, st>>>(dq_acc, dqkv, M, dt, scale);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

}  // namespace

int flash_attn_fwd(const AttnShape& a, const __nv_bfloat16* qkv, __nv_bfloat16* out, float* lse,
                   cudaStream_t st) {
  return flash_attn_fwd_tc(a, qkv, out, lse, st);
}

// mma.sync (FA2) forward, kept only as a cross-check for the tcgen05 kernel in the GPU tests.
int flash_attn_fwd_mma(const AttnShape& a, const __nv_bfloat16* qkv, __nv_bfloat16* out, float* lse,
                       cudaStream_t st) {
  if (a.seq % 128 != 0) return 1;
  switch (a.head_dim) {
    case 64: return fwd_impl<64>(a, qkv, out, lse, st);
    case 128: return fwd_impl<128>(a, qkv, out, lse, st);
    case 160: return fwd_impl<160>(a, qkv, out, lse, st);
    default: return 1;
  }
}

int flash_attn_bwd(const AttnShape& a, const __nv_bfloat16* qkv, const __nv_bfloat16* out,
                   const __nv_bfloat16* dout, const float* lse, float* D, float* dq_acc,
                   __nv_bfloat16* dqkv, cudaStream_t st, bool d_ready) {
  if (a.seq % 128 != 0) return 1;
  switch (a.head_dim) {
    case 64: return bwd_impl<64>(a, qkv, out, dout, lse, D, dq_acc, dqkv, st, false);
    case 128: return bwd_impl<128>(a, qkv, out, dout, lse, D, dq_acc, dqkv, st, d_ready);
    case 160: return bwd_impl<160>(a, qkv, out, dout, lse, D, dq_acc, dqkv, st, false);
    default: return 1;
  }
}

}  // namespace gptb200
