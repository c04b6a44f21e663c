// K5: causal flash-attention forward on the 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// CTA = one (sequence, head, 128-query block); 6 warps:
//   warp 0     TMA producer: Q once, then K_j / V_j tiles (128 kv rows) through a ring of stages
//   warp 1     TMEM owner + single-thread MMA issuer:  S_j = Q K_j^T  (M128 N128 K=hd) into one of
//              two TMEM S buffers, then O += P_j V_j (M128 N=hd K128) into the TMEM O accumulator
//   warps 2-5  softmax: thread i owns query row i (TMEM lane i) — the row max / sum need no
//              shuffles; P_j (bf16) goes to 128B-swizzled smem as the A operand of the PV MMA;
//              O is rescaled lazily (only when the running max grows by > 2^8) with tcgen05.ld/st;
//              epilogue O / l -> bf16 and lse2 = m + log2(l) (log2 units, as the backward expects).
// Issue order S_0, S_1, PV_0, S_2, PV_1, ... so the softmax of tile j+1 overlaps PV_j.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "attention.h"
#include "pdl.cuh"
#include "sm100_ptx.cuh"
#include "tma_host.h"

#include <cstdio>
#include <cstdlib>
#include <vector>

namespace gptb200 {

namespace {

constexpr int kBM = 128, kBN = 128;

#ifdef GPTB200_DEBUG_HANG
__device__ __forceinline__ void dwait(uint64_t* bar, uint32_t parity, int id) {
  uint32_t addr = ptx::smem_u32(bar);
  for (long long it = 0;; ++it) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, P1;\n\t}"
        : "=r"(done) : "r"(addr), "r"(parity) : "memory");
    if (done) return;
    if (it == (1ll << 22)) {
      printf("HANG block(%d,%d) thread %d barrier %d parity %u\n", blockIdx.x, blockIdx.y, threadIdx.x, id, parity);
      __trap();
    }
  }
}
#define WAIT(bar, par, id) dwait(bar, par, id)
#define WAIT_SPIN(bar, par, id) dwait(bar, par, id)
#else
#define WAIT(bar, par, id) ptx::mbar_wait(bar, par)
// the two-query-tile forward hands off between roles every few hundred cycles: a thread parked by
// the suspend-hinted wait resumes too late there (94 vs 798 TFLOP/s), so it spins
#define WAIT_SPIN(bar, par, id) ptx::mbar_wait_spin(bar, par)
#endif
// Timeline instrumentation of the backward kernels (debug builds only, -DGPTB200_ATTN_TRACE):
// clock64 stamps of one CTA's role events per query tile, dumped by the launcher to
// $GPTB200_ATTN_TRACE. Compiles to nothing in the release library.
#ifdef GPTB200_ATTN_TRACE
__device__ unsigned long long* g_attn_trace = nullptr;
constexpr int kTraceTiles = 64, kTraceEv = 24;
#define ATTN_TRACE(ev, j)                                                                              \
  do {                                                                                                 \
    if (g_attn_trace != nullptr && blockIdx.x == 0 && blockIdx.y == 0 && (threadIdx.x & 31) == 0 &&   \
        (j) < kTraceTiles)                                                                             \
      g_attn_trace[(j) * kTraceEv + (ev)] = clock64();                                                \
  } while (0)
#else
#define ATTN_TRACE(ev, j) \
  do {                    \
  } while (0)
#endif
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n)); }

// 2^x on the SFU, flush-to-zero (one MUFU.EX2; exp2f adds denormal range fix-ups we do not need).
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// P stays in TMEM (bf16 over the S columns it replaces) and PV reads its A operand from TMEM.
// CS softmax warps per TMEM lane quarter, each owning 128/CS score columns of its 32 query rows.
// A head of 160 columns is two 64-column SW128 chunks plus a 32-column SW64 tail chunk (its own
// tensor map), so Q / K / V tiles are 40 KB and K and V stay double-buffered.
template <int HD>
struct TcFwdCfg {
  static constexpr int NC = (HD + 63) / 64;             // 64-wide swizzle chunks of the head dim
  static constexpr int NF = HD / 64;                    // full SW128 chunks
  static constexpr int TAIL = HD % 64;                  // 0 or 32: the SW64 tail chunk
  static_assert(TAIL == 0 || TAIL == 32, "head dim must be a multiple of 64 or 64k + 32");
  static constexpr int CS = 4;                          // column splits (softmax warps per quarter)
  static constexpr int kThreads = 64 + 128 * CS;
  static constexpr int kTileBytes = 128 * 128;          // one [128 rows][64] bf16 chunk
  static constexpr int kTailBytes = TAIL ? 128 * 64 : 0;  // [128 rows][32] bf16, 64-byte rows
  static constexpr int kQBytes = NF * kTileBytes + kTailBytes;
  static constexpr int kKVBytes = NF * kTileBytes + kTailBytes;
  static constexpr int kStages = NC <= 2 ? 3 : 2;       // K ring and V ring depth
  // dynamic smem is declared __align__(1024) (checked at run time), so no alignment slack
  static constexpr int kSmem = kQBytes + 2 * kStages * kKVBytes + CS * 128 * 4 + 256;
  static_assert(kSmem <= 232448, "fa_fwd smem over the 227 KB opt-in limit");
  static constexpr int kTmemCols = 512;                 // S0 | S1 | O
};

template <int HD>
__global__ void __launch_bounds__(TcFwdCfg<HD>::kThreads, 1)
    fa_fwd_tc_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_tail,
                     __nv_bfloat16* __restrict__ out, float* __restrict__ lse, int s, int ht, float scale_log2) {
  using Cfg = TcFwdCfg<HD>;
  constexpr int NF = Cfg::NF, TAIL = Cfg::TAIL, ST = Cfg::kStages, CS = Cfg::CS;
  constexpr int CW = kBN / CS;  // score columns per softmax warp
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if ((ptx::smem_u32(smem_raw) & 1023u) != 0) __trap();  // 128B-swizzle atoms need 1 KB alignment
  uint8_t* smem = smem_raw;
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + Cfg::kQBytes;             // [ST][NC][128][64]
  uint8_t* sV = sK + ST * Cfg::kKVBytes;       // [ST][NC][128][64]
  float* xch = reinterpret_cast<float*>(sV + ST * Cfg::kKVBytes);  // [CS][128] row max / sum exchange
  uint64_t* bars = reinterpret_cast<uint64_t*>(xch + CS * 128);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;        // [ST]
  uint64_t* k_empty = k_full + ST;    // [ST]  released when S_j completes
  uint64_t* v_full = k_empty + ST;    // [ST]
  uint64_t* v_empty = v_full + ST;    // [ST]  released when PV_j completes
  uint64_t* s_full = v_empty + ST;    // [2]
  uint64_t* s_free = s_full + 2;      // [2]   released by the PV commit that consumed P_j
  uint64_t* p_full = s_free + 2;      // [2]
  uint64_t* pv_done = p_full + 2;     // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 2);

  // warp index via shfl: provably warp-uniform, so role branches are not treated as divergent
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x / 32), 0), lane = threadIdx.x % 32;
  const int qb = gridDim.x - 1 - blockIdx.x;  // heaviest causal blocks first
  const int b = blockIdx.y / ht, h = blockIdx.y % ht;
  const int dt = ht * HD;
  const int row0 = b * s;
  const int n_tiles = qb + 1;  // kBM == kBN: tile qb is the diagonal

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tm_qkv);
    if constexpr (TAIL != 0) ptx::tma_prefetch_desc(&tm_tail);
    ptx::mbar_init(q_full, 1);
    for (int i = 0; i < ST; ++i) {
      ptx::mbar_init(&k_full[i], 1);
      ptx::mbar_init(&k_empty[i], 1);
      ptx::mbar_init(&v_full[i], 1);
      ptx::mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&s_full[i], 1);
      ptx::mbar_init(&s_free[i], 1);
      ptx::mbar_init(&p_full[i], 4 * CS);
      ptx::mbar_init(&pv_done[i], 1);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);  // warp-uniform
  const uint32_t tO = tmem + 2 * kBN;
  pdl_trigger();  // prologue (smem / TMEM / barriers) done: see pdl.cuh
  pdl_wait();

  if (warp == 0) {
    if (lane == 0) {
      // a head's columns: NF SW128 chunks, then the SW64 tail chunk
      auto load_head = [&](uint8_t* dst, uint64_t* bar, int col0, int row) {
        for (int c = 0; c < NF; ++c) ptx::tma_load_2d(dst + c * Cfg::kTileBytes, &tm_qkv, bar, col0 + 64 * c, row);
        if constexpr (TAIL != 0) ptx::tma_load_2d(dst + NF * Cfg::kTileBytes, &tm_tail, bar, col0 + 64 * NF, row);
      };
      ptx::mbar_arrive_expect_tx(q_full, Cfg::kQBytes);
      load_head(sQ, q_full, h * HD, row0 + qb * kBM);
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j % ST, use = j / ST;
        WAIT(&k_empty[st], (use & 1) ^ 1, 1);
        ptx::mbar_arrive_expect_tx(&k_full[st], Cfg::kKVBytes);
        load_head(sK + st * Cfg::kKVBytes, &k_full[st], dt + h * HD, row0 + j * kBN);
        WAIT(&v_empty[st], (use & 1) ^ 1, 2);
        ptx::mbar_arrive_expect_tx(&v_full[st], Cfg::kKVBytes);
        load_head(sV + st * Cfg::kKVBytes, &v_full[st], 2 * dt + h * HD, row0 + j * kBN);
      }
    }
  } else if (warp == 1) {
    {  // all 32 lanes: uniform descriptors, one elected lane issues
      constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(kBM, kBN, false, false);
      constexpr uint32_t idesc_o = ptx::idesc_bf16_f32(kBM, 64 * NF, false, true);   // O columns of the SW128 chunks
      constexpr uint32_t idesc_t = ptx::idesc_bf16_f32(kBM, TAIL ? TAIL : 32, false, true);  // tail columns
      const uint32_t q_addr = ptx::smem_u32(sQ);
      WAIT(q_full, 0, 3);
      auto issue_pv = [&](int j) {
        const int st = j % ST, pb = j & 1;
        WAIT(&p_full[pb], (j >> 1) & 1, 4);
        WAIT(&v_full[st], (j / ST) & 1, 5);
        ptx::tc_fence_after();
        const uint32_t v_addr = ptx::smem_u32(sV + st * Cfg::kKVBytes);
#pragma unroll
        for (int kk = 0; kk < kBN / 16; ++kk) {  // P: 8 packed bf16x2 TMEM columns per K = 16 step
          const uint64_t bd = ptx::smem_desc_sw128(v_addr + kk * 2048, Cfg::kTileBytes, 1024);
          ptx::mma_bf16_ts_w(tO, tmem + pb * kBN + kk * 8, bd, idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
          if constexpr (TAIL != 0) {  // O[:, 64 NF ..) from the SW64 tail chunk of V (16 kv rows = 1 KB)
            const uint64_t bt = ptx::smem_desc_sw64(v_addr + NF * Cfg::kTileBytes + kk * 1024, 512, 512);
            ptx::mma_bf16_ts_w(tO + 64 * NF, tmem + pb * kBN + kk * 8, bt, idesc_t, (j > 0 || kk > 0) ? 1u : 0u);
          }
        }
        ptx::mma_commit_w(&pv_done[pb]);
        ptx::mma_commit_w(&v_empty[st]);
        ptx::mma_commit_w(&s_free[pb]);  // P (in S_j's columns) consumed
      };
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j % ST, buf = j & 1;
        WAIT(&k_full[st], (j / ST) & 1, 6);
        WAIT(&s_free[buf], ((j >> 1) & 1) ^ 1, 7);
        ptx::tc_fence_after();
        const uint32_t k_addr = ptx::smem_u32(sK + st * Cfg::kKVBytes);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          if (kk < 4 * NF) {
            const uint32_t off = (kk / 4) * Cfg::kTileBytes + (kk % 4) * 32;
            ptx::mma_bf16_ss_w(tmem + buf * kBN, ptx::smem_desc_sw128(q_addr + off, 16, 1024),
                               ptx::smem_desc_sw128(k_addr + off, 16, 1024), idesc_s, kk > 0 ? 1u : 0u);
          } else {  // tail chunk: 64-byte rows, 8-row atoms of 512 B
            const uint32_t off = NF * Cfg::kTileBytes + (kk - 4 * NF) * 32;
            ptx::mma_bf16_ss_w(tmem + buf * kBN, ptx::smem_desc_sw64(q_addr + off, 16, 512),
                               ptx::smem_desc_sw64(k_addr + off, 16, 512), idesc_s, 1u);
          }
        }
        ptx::mma_commit_w(&s_full[buf]);
        ptx::mma_commit_w(&k_empty[st]);
        if (j > 0) issue_pv(j - 1);
      }
      issue_pv(n_tiles - 1);
    }
  } else {
    // ------------------------------------------------------------ softmax / epilogue
    // CS warps per TMEM lane quarter: warp owns query rows 32q..32q+31 (its lanes) and CW score
    // columns; the CS column parts of a row exchange their max through smem once per tile (one
    // named barrier per quarter) and their row sums at the end.
    const int quarter = warp & 3;
    const int part = (warp - 2) >> 2;   // 0..CS-1
    const int r = quarter * 32 + lane;  // query row within the block == TMEM lane
    const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
    const int q_row = qb * kBM + r;
    constexpr int NCH = HD / 32;  // 32-column chunks of O, split over the CS parts
    const int oc0 = part * NCH / CS, oc1 = (part + 1) * NCH / CS;
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < n_tiles; ++j) {
      const int buf = j & 1;
      WAIT(&s_full[buf], (j >> 1) & 1, 8);
      ptx::tc_fence_after();
      // raw scores (scale_log2 > 0 is applied inside the exponent: max commutes with it)
      float x[CW];
      {
        uint32_t v[CW];
        if constexpr (CW == 32)
          ptx::tmem_ld_32x32b_x32(tmem + lane_base + buf * kBN + part * CW, v);
        else
          static_assert(CW == 32, "column split must give 32-column parts");
        ptx::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < CW; ++i) x[i] = __uint_as_float(v[i]);
      }
      if (j == qb) {  // diagonal tile: causal mask (the only tile that needs one)
#pragma unroll
        for (int i = 0; i < CW; ++i)
          if (part * CW + i > r) x[i] = -INFINITY;
      }
      float pm[8];  // 8 independent partial maxima (short dependency chains)
#pragma unroll
      for (int k = 0; k < 8; ++k) pm[k] = fmaxf(x[k], x[k + 8]);
#pragma unroll
      for (int i = 16; i < CW; i += 8)
#pragma unroll
        for (int k = 0; k < 8; ++k) pm[k] = fmaxf(pm[k], x[i + k]);
      float mt = fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])), fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7])));
      mt *= scale_log2;
      xch[part * 128 + r] = mt;
      named_sync(1 + quarter, 32 * CS);
#pragma unroll
      for (int o = 1; o < CS; ++o) mt = fmaxf(mt, xch[((part + o) % CS) * 128 + r]);
      named_sync(1 + quarter, 32 * CS);  // exchange slots are reused next tile
      // Lazy rescale (only when a row's max grows by > 2^8). tcgen05.ld/st are warp-collective,
      // so the decision is warp-uniform (and identical in every part of a row).
      if (__any_sync(0xffffffffu, mt > m_used + 8.f)) {
        const float m_new = fmaxf(m_used, mt);
        if (j > 0) {
          // O must hold all of PV_0..PV_{j-1} before it is rescaled
          WAIT(&pv_done[(j - 1) & 1], ((j - 1) >> 1) & 1, 9);
          const float f = exp2f(m_used - m_new);
          l *= f;
          ptx::tc_fence_after();
#pragma unroll 1
          for (int c = oc0; c < oc1; ++c) {
            uint32_t v[32];
            ptx::tmem_ld_32x32b_x32(tO + lane_base + c * 32, v);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * f);
            ptx::tmem_st_32x32b_x32(tO + lane_base + c * 32, v);
          }
          ptx::tmem_st_wait();
        }
        m_used = m_new;
      }
      // P = exp2(x - m_used) as bf16 pairs into this part's CW/2 columns of S_j (every part has read
      // its scores: the max exchange above is a barrier), the A operand of PV_j
      const float neg_m = -m_used;
      float ls[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // independent partial row sums
      uint32_t pk[CW / 2];
#pragma unroll
      for (int u = 0; u < CW / 8; ++u) {
        float pv[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          pv[e] = ex2(fmaf(x[u * 8 + e], scale_log2, neg_m));
          ls[e] += pv[e];
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) pk[u * 4 + e] = ptx::pack_bf16(pv[2 * e], pv[2 * e + 1]);
      }
      ptx::tmem_st_32x32b_x16(tmem + lane_base + buf * kBN + part * (CW / 2), pk);
      ptx::tmem_st_wait();
      l += ((ls[0] + ls[1]) + (ls[2] + ls[3])) + ((ls[4] + ls[5]) + (ls[6] + ls[7]));
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&p_full[buf]);
    }
    // combine the parts' row sums
    xch[part * 128 + r] = l;
    named_sync(1 + quarter, 32 * CS);
    float l_tot = l;
#pragma unroll
    for (int o = 1; o < CS; ++o) l_tot += xch[((part + o) % CS) * 128 + r];
    WAIT(&pv_done[(n_tiles - 1) & 1], ((n_tiles - 1) >> 1) & 1, 11);
    ptx::tc_fence_after();
    const float inv = 1.f / l_tot;
    __nv_bfloat16* orow = out + static_cast<size_t>(row0 + q_row) * dt + h * HD;
#pragma unroll 1
    for (int c = oc0; c < oc1; ++c) {
      uint32_t v[32];
      ptx::tmem_ld_32x32b_x32(tO + lane_base + c * 32, v);
      ptx::tmem_ld_wait();
      uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 pkk;
        pkk.x = ptx::pack_bf16(__uint_as_float(v[8 * q + 0]) * inv, __uint_as_float(v[8 * q + 1]) * inv);
        pkk.y = ptx::pack_bf16(__uint_as_float(v[8 * q + 2]) * inv, __uint_as_float(v[8 * q + 3]) * inv);
        pkk.z = ptx::pack_bf16(__uint_as_float(v[8 * q + 4]) * inv, __uint_as_float(v[8 * q + 5]) * inv);
        pkk.w = ptx::pack_bf16(__uint_as_float(v[8 * q + 6]) * inv, __uint_as_float(v[8 * q + 7]) * inv);
        dst[q] = pkk;
      }
    }
    if (part == 0) lse[(static_cast<size_t>(b) * ht + h) * s + q_row] = m_used + log2f(l_tot);
  }
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<Cfg::kTmemCols>(tmem);
  }
}

// Persistent variant (hd <= 128): one CTA per SM walks (q block, sequence-head) work items in
// heaviest-first order; the barrier rings run on a per-CTA global tile counter across items, the
// next item's Q loads as soon as the last S of the current one is issued, and the O accumulator
// alternates between two TMEM buffers so one item's epilogue overlaps the next item's MMAs.
// TMEM: S0 | S1 | O0 | O1.
template <int HD>
__global__ void __launch_bounds__(TcFwdCfg<HD>::kThreads, 1)
    fa_fwd_tc_persistent(const __grid_constant__ CUtensorMap tm_qkv, __nv_bfloat16* __restrict__ out,
                         float* __restrict__ lse, int s, int ht, int batch, float scale_log2) {
  using Cfg = TcFwdCfg<HD>;
  static_assert(2 * kBN + 2 * HD <= 512, "two O accumulators must fit in TMEM");
  constexpr int NC = Cfg::NC, ST = Cfg::kStages, CS = Cfg::CS;
  constexpr int CW = kBN / CS;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if ((ptx::smem_u32(smem_raw) & 1023u) != 0) __trap();
  uint8_t* sQ = smem_raw;
  uint8_t* sK = sQ + Cfg::kQBytes;
  uint8_t* sV = sK + ST * Cfg::kKVBytes;
  float* xch = reinterpret_cast<float*>(sV + ST * Cfg::kKVBytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(xch + CS * 128);
  uint64_t* q_full = bars;
  uint64_t* q_empty = bars + 1;       // all S MMAs of the item issued and complete
  uint64_t* k_full = bars + 2;        // [ST]
  uint64_t* k_empty = k_full + ST;    // [ST]
  uint64_t* v_full = k_empty + ST;    // [ST]
  uint64_t* v_empty = v_full + ST;    // [ST]
  uint64_t* s_full = v_empty + ST;    // [2]
  uint64_t* s_free = s_full + 2;      // [2]
  uint64_t* p_full = s_free + 2;      // [2]
  uint64_t* pv_done = p_full + 2;     // [2]
  uint64_t* o_free = pv_done + 2;     // [2] O buffer drained by the epilogue
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_free + 2);

  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x / 32), 0), lane = threadIdx.x % 32;
  const int dt = ht * HD;
  const int n_qb = s / kBM, BH = batch * ht;
  const int n_items = n_qb * BH;
  // items sorted heaviest first; round t hands them out forwards or backwards ("snake") so every
  // CTA gets a balanced mix of long and short causal blocks
  auto snake = [&](int t) {
    const int G = gridDim.x, c = blockIdx.x;
    return t * G + ((t & 1) ? G - 1 - c : c);
  };
  auto item = [&](int k, int& qb, int& b, int& h) {  // heaviest q blocks first
    qb = n_qb - 1 - k / BH;
    const int bh = k % BH;
    b = bh / ht;
    h = bh % ht;
  };

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tm_qkv);
    ptx::mbar_init(q_full, 1);
    ptx::mbar_init(q_empty, 1);
    for (int i = 0; i < ST; ++i) {
      ptx::mbar_init(&k_full[i], 1);
      ptx::mbar_init(&k_empty[i], 1);
      ptx::mbar_init(&v_full[i], 1);
      ptx::mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&s_full[i], 1);
      ptx::mbar_init(&s_free[i], 1);
      ptx::mbar_init(&p_full[i], 4 * CS);
      ptx::mbar_init(&pv_done[i], 1);
      ptx::mbar_init(&o_free[i], 4 * CS);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  pdl_trigger();  // prologue (smem / TMEM / barriers) done: see pdl.cuh
  pdl_wait();

  if (warp == 0) {
    if (lane == 0) {
      int gt = 0, t = 0;
      for (int k = snake(0); k < n_items; k = snake(t + 1), ++t) {
        int qb, b, h;
        item(k, qb, b, h);
        const int row0 = b * s;
        WAIT(q_empty, (t & 1) ^ 1, 12);
        ptx::mbar_arrive_expect_tx(q_full, Cfg::kQBytes);
        for (int c = 0; c < NC; ++c)
          ptx::tma_load_2d(sQ + c * Cfg::kTileBytes, &tm_qkv, q_full, h * HD + 64 * c, row0 + qb * kBM);
        for (int j = 0; j <= qb; ++j, ++gt) {
          const int st = gt % ST, use = gt / ST;
          WAIT(&k_empty[st], (use & 1) ^ 1, 1);
          ptx::mbar_arrive_expect_tx(&k_full[st], Cfg::kKVBytes);
          for (int c = 0; c < NC; ++c)
            ptx::tma_load_2d(sK + st * Cfg::kKVBytes + c * Cfg::kTileBytes, &tm_qkv, &k_full[st],
                             dt + h * HD + 64 * c, row0 + j * kBN);
          WAIT(&v_empty[st], (use & 1) ^ 1, 2);
          ptx::mbar_arrive_expect_tx(&v_full[st], Cfg::kKVBytes);
          for (int c = 0; c < NC; ++c)
            ptx::tma_load_2d(sV + st * Cfg::kKVBytes + c * Cfg::kTileBytes, &tm_qkv, &v_full[st],
                             2 * dt + h * HD + 64 * c, row0 + j * kBN);
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(kBM, kBN, false, false);
    constexpr uint32_t idesc_o = ptx::idesc_bf16_f32(kBM, HD, false, true);
    const uint32_t q_addr = ptx::smem_u32(sQ);
    int gt = 0, t = 0;
    for (int k = snake(0); k < n_items; k = snake(t + 1), ++t) {
      int qb, b, h;
      item(k, qb, b, h);
      const int n_tiles = qb + 1;
      const int ob = t & 1;
      const uint32_t tO = tmem + 2 * kBN + ob * HD;
      WAIT(q_full, t & 1, 3);
      auto issue_pv = [&](int g, bool first) {
        const int st = g % ST, pb = g & 1;
        if (first && t >= 2) WAIT(&o_free[ob], ((t >> 1) - 1) & 1, 13);  // O_ob drained (item t-2)
        WAIT(&p_full[pb], (g >> 1) & 1, 4);
        WAIT(&v_full[st], (g / ST) & 1, 5);
        ptx::tc_fence_after();
        const uint32_t v_addr = ptx::smem_u32(sV + st * Cfg::kKVBytes);
#pragma unroll
        for (int kk = 0; kk < kBN / 16; ++kk) {
          const uint64_t bd = ptx::smem_desc_sw128(v_addr + kk * 2048, Cfg::kTileBytes, 1024);
          ptx::mma_bf16_ts_w(tO, tmem + pb * kBN + kk * 8, bd, idesc_o, (!first || kk > 0) ? 1u : 0u);
        }
        ptx::mma_commit_w(&pv_done[pb]);
        ptx::mma_commit_w(&v_empty[st]);
        ptx::mma_commit_w(&s_free[pb]);
      };
      for (int j = 0; j < n_tiles; ++j) {
        const int g = gt + j, st = g % ST, buf = g & 1;
        WAIT(&k_full[st], (g / ST) & 1, 6);
        WAIT(&s_free[buf], ((g >> 1) & 1) ^ 1, 7);
        ptx::tc_fence_after();
        const uint32_t k_addr = ptx::smem_u32(sK + st * Cfg::kKVBytes);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = (kk / 4) * Cfg::kTileBytes + (kk % 4) * 32;
          ptx::mma_bf16_ss_w(tmem + buf * kBN, ptx::smem_desc_sw128(q_addr + off, 16, 1024),
                             ptx::smem_desc_sw128(k_addr + off, 16, 1024), idesc_s, kk > 0 ? 1u : 0u);
        }
        ptx::mma_commit_w(&s_full[buf]);
        ptx::mma_commit_w(&k_empty[st]);
        if (j == n_tiles - 1) ptx::mma_commit_w(q_empty);  // Q free for the next item
        if (j > 0) issue_pv(g - 1, j == 1);
      }
      issue_pv(gt + n_tiles - 1, n_tiles == 1);
      gt += n_tiles;
    }
  } else {
    const int quarter = warp & 3;
    const int part = (warp - 2) >> 2;
    const int r = quarter * 32 + lane;
    const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
    constexpr int NCH = HD / 32;
    const int oc0 = part * NCH / CS, oc1 = (part + 1) * NCH / CS;
    int gt = 0, t = 0;
    for (int k = snake(0); k < n_items; k = snake(t + 1), ++t) {
      int qb, b, h;
      item(k, qb, b, h);
      const int n_tiles = qb + 1;
      const uint32_t tO = tmem + 2 * kBN + (t & 1) * HD;
      const int q_row = qb * kBM + r;
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < n_tiles; ++j) {
        const int g = gt + j, buf = g & 1;
        WAIT(&s_full[buf], (g >> 1) & 1, 8);
        ptx::tc_fence_after();
        float x[CW];
        {
          uint32_t v[CW];
          ptx::tmem_ld_32x32b_x32(tmem + lane_base + buf * kBN + part * CW, v);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < CW; ++i) x[i] = __uint_as_float(v[i]);
        }
        if (j == qb) {
#pragma unroll
          for (int i = 0; i < CW; ++i)
            if (part * CW + i > r) x[i] = -INFINITY;
        }
        float pm[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) pm[q] = fmaxf(x[q], x[q + 8]);
#pragma unroll
        for (int i = 16; i < CW; i += 8)
#pragma unroll
          for (int q = 0; q < 8; ++q) pm[q] = fmaxf(pm[q], x[i + q]);
        float mt = fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])), fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7])));
        mt *= scale_log2;
        xch[part * 128 + r] = mt;
        named_sync(1 + quarter, 32 * CS);
#pragma unroll
        for (int o = 1; o < CS; ++o) mt = fmaxf(mt, xch[((part + o) % CS) * 128 + r]);
        named_sync(1 + quarter, 32 * CS);
        if (__any_sync(0xffffffffu, mt > m_used + 8.f)) {
          const float m_new = fmaxf(m_used, mt);
          if (j > 0) {
            WAIT(&pv_done[(g - 1) & 1], ((g - 1) >> 1) & 1, 9);
            const float f = exp2f(m_used - m_new);
            l *= f;
            ptx::tc_fence_after();
#pragma unroll 1
            for (int c = oc0; c < oc1; ++c) {
              uint32_t v[32];
              ptx::tmem_ld_32x32b_x32(tO + lane_base + c * 32, v);
              ptx::tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * f);
              ptx::tmem_st_32x32b_x32(tO + lane_base + c * 32, v);
            }
            ptx::tmem_st_wait();
          }
          m_used = m_new;
        }
        const float neg_m = -m_used;
        float ls[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        uint32_t pk[CW / 2];
#pragma unroll
        for (int u = 0; u < CW / 8; ++u) {
          float pv[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            pv[e] = ex2(fmaf(x[u * 8 + e], scale_log2, neg_m));
            ls[e] += pv[e];
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) pk[u * 4 + e] = ptx::pack_bf16(pv[2 * e], pv[2 * e + 1]);
        }
        ptx::tmem_st_32x32b_x16(tmem + lane_base + buf * kBN + part * (CW / 2), pk);
        ptx::tmem_st_wait();
        l += ((ls[0] + ls[1]) + (ls[2] + ls[3])) + ((ls[4] + ls[5]) + (ls[6] + ls[7]));
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&p_full[buf]);
      }
      // epilogue of this item: combine row sums, O / l -> bf16, lse; then release O for item t+2
      xch[part * 128 + r] = l;
      named_sync(1 + quarter, 32 * CS);
      float l_tot = l;
#pragma unroll
      for (int o = 1; o < CS; ++o) l_tot += xch[((part + o) % CS) * 128 + r];
      named_sync(1 + quarter, 32 * CS);  // exchange slots are reused by the next item
      const int g_last = gt + n_tiles - 1;
      WAIT(&pv_done[g_last & 1], (g_last >> 1) & 1, 11);
      ptx::tc_fence_after();
      const float inv = 1.f / l_tot;
      __nv_bfloat16* orow = out + static_cast<size_t>(b * s + q_row) * dt + h * HD;
#pragma unroll 1
      for (int c = oc0; c < oc1; ++c) {
        uint32_t v[32];
        ptx::tmem_ld_32x32b_x32(tO + lane_base + c * 32, v);
        ptx::tmem_ld_wait();
        uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 pkk;
          pkk.x = ptx::pack_bf16(__uint_as_float(v[8 * q + 0]) * inv, __uint_as_float(v[8 * q + 1]) * inv);
          pkk.y = ptx::pack_bf16(__uint_as_float(v[8 * q + 2]) * inv, __uint_as_float(v[8 * q + 3]) * inv);
          pkk.z = ptx::pack_bf16(__uint_as_float(v[8 * q + 4]) * inv, __uint_as_float(v[8 * q + 5]) * inv);
          pkk.w = ptx::pack_bf16(__uint_as_float(v[8 * q + 6]) * inv, __uint_as_float(v[8 * q + 7]) * inv);
          dst[q] = pkk;
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&o_free[t & 1]);
      if (part == 0) lse[(static_cast<size_t>(b) * ht + h) * s + q_row] = m_used + log2f(l_tot);
      gt += n_tiles;
    }
  }
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

// K5, two query tiles per CTA (hd 64 / 128). CTA = (256-row query block, sequence-head); heaviest
// blocks launch first. The tensor core always has the other tile's work while one tile's softmax
// runs:  per kv tile j the MMA warp issues  PV_0(j), S_0(j+1), PV_1(j), S_1(j+1), so softmax_0(j+1)
// overlaps PV_1(j) + S_1(j+1) and softmax_1(j+1) overlaps PV_0(j+1) + S_0(j+2) (every MMA is
// M128 x N128, at the tcgen05 issue floor; N = 64 halves of that measure 0.54 of it).
// TMEM: S_0 | S_1 (128 fp32 columns each; P_t overwrites S_t as packed bf16, the A operand of PV_t,
// and S_t(j+1) follows PV_t(j) in the same in-order MMA stream) | O_0 | O_1 (HD columns each).
// Warps: 0 TMA (Q_0 + Q_1 once, K / V rings), 1 MMA issuer, 2-3 idle, 4-7 softmax of tile 0, 8-11
// softmax of tile 1: thread = query row = TMEM lane, so the row max and sum are thread-local;
// O_t is rescaled lazily (running max grows by > 2^8) by the tile's own softmax warps.
// Paired fp32 (FFMA2 / FADD2) and 2^x on the FMA pipe for a pair: x = j + f with j = rint(x) (magic-number
// rounding), 2^f by a degree-3 minimax polynomial on [-0.5, 0.5] (relative error 7.5e-5, far below the
// bf16 rounding of P), 2^j added to the exponent field by one IMAD per element. Inputs <= 0 (scores
// minus the running max); clamped at -126 (2^j stays a normal exponent offset) so masked (-inf) scores
// give a denormal ~0.
__device__ __forceinline__ uint64_t fa_pack2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 fa_unpack2(uint64_t v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ uint64_t fa_fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fa_add2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float2 exp2_fma2(float a, float b) {
  constexpr float kMagic = 12582912.f;  // 1.5 * 2^23
  const uint64_t x = fa_pack2(fmaxf(a, -126.f), fmaxf(b, -126.f));
  const uint64_t t = fa_add2(x, fa_pack2(kMagic, kMagic));                  // low bits = rint(x)
  const uint64_t jf = fa_add2(t, fa_pack2(-kMagic, -kMagic));               // rint(x) as float
  const uint64_t f = fa_fma2(jf, fa_pack2(-1.f, -1.f), x);                   // x - rint(x)
  uint64_t p = fa_fma2(f, fa_pack2(0.05517163f, 0.05517163f), fa_pack2(0.24261117f, 0.24261117f));
  p = fa_fma2(p, f, fa_pack2(0.693261f, 0.693261f));
  p = fa_fma2(p, f, fa_pack2(0.99992807f, 0.99992807f));
  const float2 pv = fa_unpack2(p), tv = fa_unpack2(t);
  return make_float2(__int_as_float(__float_as_int(pv.x) + (__float_as_int(tv.x) << 23)),
                     __int_as_float(__float_as_int(pv.y) + (__float_as_int(tv.y) << 23)));
}

constexpr int kFwd2HeadGroup = 32;  // (sequence, head) pairs per L2-resident launch group of fa_fwd2

template <int HD, int CS>
struct TcFwd2Cfg {
  static constexpr int NC = HD / 64;
  static constexpr int kChunk = 128 * 128;              // [128 rows][64] bf16, SW128
  static constexpr int kTileBytes = NC * kChunk;        // [128 rows][HD]
  static constexpr int ST = 2;                          // K ring and V ring depth
  static constexpr int kThreads = 128 + 2 * CS * 128;   // WG0 + CS softmax warpgroups per query tile
  static constexpr int kSmem = 2 * kTileBytes + 2 * ST * kTileBytes + 2 * CS * 128 * 4 + 256;
  static_assert(kSmem <= 232448, "fa_fwd2 smem over the 227 KB opt-in limit");
  // register split (setmaxnreg): the launch allocates kRegBase per thread (65536 / threads, rounded
  // down to 8); WG0 drops to 56 and the softmax warpgroups may grow only by what it released —
  // asking for more blocks setmaxnreg.inc forever.
  static constexpr int kRegBase = (65536 / kThreads) / 8 * 8;
  static constexpr int kRegSoftmaxRaw = ((kThreads * kRegBase - 128 * 56) / (kThreads - 128)) / 8 * 8;
  static constexpr int kRegSoftmax = kRegSoftmaxRaw > 232 ? 232 : kRegSoftmaxRaw;
  static_assert(128 * 56 + (kThreads - 128) * kRegSoftmax <= kThreads * kRegBase, "setmaxnreg budget");
};

// EMU: pairs out of every 8 (16 scores) whose 2^x runs on the FMA pipe instead of the MUFU.
// CS: softmax warps per (query tile, TMEM lane quarter); each owns 128/CS score columns of its 32
// rows, the CS parts exchange their row max once per kv tile through shared memory.
template <int HD, int EMU, int CS>
__global__ void __launch_bounds__(TcFwd2Cfg<HD, CS>::kThreads, 1)
    fa_fwd2_kernel(const __grid_constant__ CUtensorMap tm_qkv, __nv_bfloat16* __restrict__ out,
                   float* __restrict__ lse, int s, int ht, float scale_log2) {
  using Cfg = TcFwd2Cfg<HD, CS>;
  constexpr int NC = Cfg::NC, ST = Cfg::ST, CH = Cfg::kChunk, TB = Cfg::kTileBytes;
  constexpr int CW = 128 / CS;  // score columns per softmax thread
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if ((ptx::smem_u32(smem_raw) & 1023u) != 0) __trap();  // 128B-swizzle atoms need 1 KB alignment
  uint8_t* sQ = smem_raw;                   // [2 tiles][NC][128][64]
  uint8_t* sK = sQ + 2 * TB;                // [ST][NC][128][64]
  uint8_t* sV = sK + ST * TB;               // [ST][NC][128][64]
  float* xch = reinterpret_cast<float*>(sV + ST * TB);  // [2 tiles][CS][128] row max / sum exchange
  uint64_t* bars = reinterpret_cast<uint64_t*>(xch + 2 * CS * 128);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;              // [ST]
  uint64_t* k_empty = k_full + ST;          // [ST]
  uint64_t* v_full = k_empty + ST;          // [ST]
  uint64_t* v_empty = v_full + ST;          // [ST]
  uint64_t* s_full = v_empty + ST;          // [2 tiles]
  uint64_t* p_full = s_full + 2;            // [2 tiles]
  uint64_t* pv_done = p_full + 2;           // [2 tiles]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 2);

  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x / 32), 0), lane = threadIdx.x % 32;
  // Launch order: groups of kFwd2HeadGroup (sequence, head) pairs, heaviest query blocks of the group
  // first. A group's K/V (1 MB per head at s 2048) stays in L2 while its blocks run, instead of every
  // head's K/V being re-read from HBM once per query block (heaviest-first over all heads).
  const int nqb = gridDim.y, BH = gridDim.x;
  const int t = blockIdx.y * BH + blockIdx.x;
  const int grp = t / (nqb * kFwd2HeadGroup), rem = t % (nqb * kFwd2HeadGroup);
  const int gsz = min(kFwd2HeadGroup, BH - grp * kFwd2HeadGroup);
  const int qb = nqb - 1 - rem / gsz;
  const int bh = grp * kFwd2HeadGroup + rem % gsz;
  const int b = bh / ht, h = bh % ht;
  const int dt = ht * HD;
  const int row0 = b * s;
  const int n = 2 * qb + 2;  // kv tiles of tile 1; tile 0 uses the first n - 1

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tm_qkv);
    ptx::mbar_init(q_full, 1);
    for (int i = 0; i < ST; ++i) {
      ptx::mbar_init(&k_full[i], 1);
      ptx::mbar_init(&k_empty[i], 1);
      ptx::mbar_init(&v_full[i], 1);
      ptx::mbar_init(&v_empty[i], 1);
    }
    for (int t = 0; t < 2; ++t) {
      ptx::mbar_init(&s_full[t], 1);
      ptx::mbar_init(&p_full[t], 4 * CS);
      ptx::mbar_init(&pv_done[t], 1);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);  // warp-uniform
  pdl_trigger();
  pdl_wait();
  const int wg = warp / 4;
  if (wg == 0) {
    ptx::setmaxnreg_dec<56>();
    if (warp == 0) {
      if (lane == 0) {
        ptx::mbar_arrive_expect_tx(q_full, 2 * TB);
        for (int t = 0; t < 2; ++t)
          for (int c = 0; c < NC; ++c)
            ptx::tma_load_2d(sQ + t * TB + c * CH, &tm_qkv, q_full, h * HD + 64 * c, row0 + qb * 256 + t * 128);
        for (int j = 0; j < n; ++j) {
          const int st = j % ST, use = j / ST;
          WAIT_SPIN(&k_empty[st], (use & 1) ^ 1, 60);
          ptx::mbar_arrive_expect_tx(&k_full[st], TB);
          for (int c = 0; c < NC; ++c)
            ptx::tma_load_2d(sK + st * TB + c * CH, &tm_qkv, &k_full[st], dt + h * HD + 64 * c, row0 + j * 128);
          WAIT_SPIN(&v_empty[st], (use & 1) ^ 1, 61);
          ptx::mbar_arrive_expect_tx(&v_full[st], TB);
          for (int c = 0; c < NC; ++c)
            ptx::tma_load_2d(sV + st * TB + c * CH, &tm_qkv, &v_full[st], 2 * dt + h * HD + 64 * c, row0 + j * 128);
        }
      }
    } else if (warp == 1) {
      constexpr uint32_t id_s = ptx::idesc_bf16_f32(128, 128, false, false);
      constexpr uint32_t id_o = ptx::idesc_bf16_f32(128, HD, false, true);
      const uint32_t aQ = ptx::smem_u32(sQ), aK0 = ptx::smem_u32(sK), aV0 = ptx::smem_u32(sV);
      auto issue_s = [&](int t, int j) {  // S_t = Q_t K_j^T
        const uint32_t aq = aQ + t * TB, ak = aK0 + (j % ST) * TB;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = (kk / 4) * CH + (kk % 4) * 32;
          ptx::mma_bf16_ss_w(tmem + t * 128, ptx::smem_desc_sw128(aq + off, 16, 1024),
                             ptx::smem_desc_sw128(ak + off, 16, 1024), id_s, kk > 0 ? 1u : 0u);
        }
        ptx::mma_commit_w(&s_full[t]);
      };
      auto issue_pv = [&](int t, int j) {  // O_t += P_t V_j (P_t from TMEM)
        const uint32_t av = aV0 + (j % ST) * TB;
#pragma unroll
        for (int kk = 0; kk < 128 / 16; ++kk)
          ptx::mma_bf16_ts_w(tmem + 256 + t * HD, tmem + t * 128 + kk * 8,
                             ptx::smem_desc_sw128(av + kk * 2048, CH, 1024), id_o, (j > 0 || kk > 0) ? 1u : 0u);
        ptx::mma_commit_w(&pv_done[t]);
      };
      WAIT_SPIN(q_full, 0, 62);
      WAIT_SPIN(&k_full[0], 0, 63);
      ptx::tc_fence_after();
      issue_s(0, 0);
      issue_s(1, 0);
      ptx::mma_commit_w(&k_empty[0]);
      for (int j = 0; j < n; ++j) {
        const int st = j % ST, st1 = (j + 1) % ST;
        const bool next = j + 1 < n;
        WAIT_SPIN(&v_full[st], (j / ST) & 1, 64);
        if (next) WAIT_SPIN(&k_full[st1], ((j + 1) / ST) & 1, 65);
        if (j < n - 1) {  // tile 0 (its last kv tile is n - 2)
          WAIT_SPIN(&p_full[0], j & 1, 66);
          ATTN_TRACE(0, j);
          ptx::tc_fence_after();
          issue_pv(0, j);
          if (j + 1 < n - 1) issue_s(0, j + 1);
          ATTN_TRACE(1, j);
        }
        WAIT_SPIN(&p_full[1], j & 1, 67);
        ATTN_TRACE(2, j);
        ptx::tc_fence_after();
        issue_pv(1, j);
        ptx::mma_commit_w(&v_empty[st]);
        if (next) {
          issue_s(1, j + 1);
          ptx::mma_commit_w(&k_empty[st1]);
        }
        ATTN_TRACE(3, j);
      }
    }
  } else {
    ptx::setmaxnreg_inc<Cfg::kRegSoftmax>();
    const int t = (wg - 1) / CS;           // query tile
    const int part = (wg - 1) % CS;        // which CW score columns of the row
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;     // query row within the tile == TMEM lane
    const uint32_t lb = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t tS = tmem + lb + t * 128, tO = tmem + lb + 256 + t * HD;
    const int nt = n - 1 + t;              // kv tiles of this query tile; the last is the diagonal
    float* xrow = xch + t * CS * 128;      // [CS][128]
    const int bar_id = 1 + t * 4 + quarter;  // named barrier of the CS warps sharing these rows
    const bool tw = quarter == 0 && part == 0;
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < nt; ++j) {
      if (tw) ATTN_TRACE(4 + 5 * t, j);
      WAIT_SPIN(&s_full[t], j & 1, 68);
      if (tw) ATTN_TRACE(5 + 5 * t, j);
      ptx::tc_fence_after();
      float x[CW];
      {
        uint32_t v[CW / 32][32];
#pragma unroll
        for (int c = 0; c < CW / 32; ++c) ptx::tmem_ld_32x32b_x32(tS + part * CW + c * 32, v[c]);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < CW / 32; ++c)
#pragma unroll
          for (int i = 0; i < 32; ++i) x[c * 32 + i] = __uint_as_float(v[c][i]);
      }
      if (j == nt - 1) {  // diagonal tile
#pragma unroll
        for (int i = 0; i < CW; ++i)
          if (part * CW + i > r) x[i] = -INFINITY;
      }
      float pm[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) pm[k] = fmaxf(x[k], x[k + 8]);
#pragma unroll
      for (int i = 16; i < CW; i += 8)
#pragma unroll
        for (int k = 0; k < 8; ++k) pm[k] = fmaxf(pm[k], x[i + k]);
      float mt =
          fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])), fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7]))) *
          scale_log2;
      if constexpr (CS > 1) {  // row max over the parts (also orders every part's S reads before any P write)
        xrow[part * 128 + r] = mt;
        named_sync(bar_id, 32 * CS);
#pragma unroll
        for (int o = 1; o < CS; ++o) mt = fmaxf(mt, xrow[((part + o) % CS) * 128 + r]);
        named_sync(bar_id, 32 * CS);  // exchange slots are reused next tile
      }
      if (tw) ATTN_TRACE(6 + 5 * t, j);
      if (__any_sync(0xffffffffu, mt > m_used + 8.f)) {
        const float m_new = fmaxf(m_used, mt);
        if (j > 0) {  // O_t holds PV_t(0..j-1) once pv_done completes phase j-1
          WAIT_SPIN(&pv_done[t], (j - 1) & 1, 69);
          const float f = exp2f(m_used - m_new);
          l *= f;
          ptx::tc_fence_after();
#pragma unroll 1
          for (int c = part * (HD / 32) / CS; c < (part + 1) * (HD / 32) / CS; ++c) {
            uint32_t v[32];
            ptx::tmem_ld_32x32b_x32(tO + c * 32, v);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * f);
            ptx::tmem_st_32x32b_x32(tO + c * 32, v);
          }
        }
        m_used = m_new;
      }
      const uint64_t sc2 = fa_pack2(scale_log2, scale_log2), nm2 = fa_pack2(-m_used, -m_used);
      uint64_t ls[4] = {0ull, 0ull, 0ull, 0ull};  // paired partial row sums
#pragma unroll
      for (int c = 0; c < CW / 32; ++c) {  // 32 scores -> 16 packed bf16x2 columns of P over S
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float2 sv = fa_unpack2(fa_fma2(fa_pack2(x[c * 32 + 2 * e], x[c * 32 + 2 * e + 1]), sc2, nm2));
          float2 pv;
          if ((e & 7) >= 8 - EMU) {
            pv = exp2_fma2(sv.x, sv.y);
          } else {
            pv.x = ex2(sv.x);
            pv.y = ex2(sv.y);
          }
          ls[e & 3] = fa_add2(ls[e & 3], fa_pack2(pv.x, pv.y));
          pk[e] = ptx::pack_bf16(pv.x, pv.y);
        }
        ptx::tmem_st_32x32b_x16(tS + part * (CW / 2) + c * 16, pk);
      }
      {
        const float2 a0 = fa_unpack2(fa_add2(ls[0], ls[1])), a1 = fa_unpack2(fa_add2(ls[2], ls[3]));
        l += (a0.x + a0.y) + (a1.x + a1.y);
      }
      if (tw) ATTN_TRACE(7 + 5 * t, j);
      ptx::tmem_st_wait();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&p_full[t]);
      if (tw) ATTN_TRACE(8 + 5 * t, j);
    }
    float l_tot = l;
    if constexpr (CS > 1) {
      xrow[part * 128 + r] = l;
      named_sync(bar_id, 32 * CS);
#pragma unroll
      for (int o = 1; o < CS; ++o) l_tot += xrow[((part + o) % CS) * 128 + r];
    }
    WAIT_SPIN(&pv_done[t], (nt - 1) & 1, 70);
    ptx::tc_fence_after();
    const int q_row = qb * 256 + t * 128 + r;
    const float inv = 1.f / l_tot;
    __nv_bfloat16* orow = out + static_cast<size_t>(row0 + q_row) * dt + h * HD;
#pragma unroll 1
    for (int c = part * (HD / 32) / CS; c < (part + 1) * (HD / 32) / CS; ++c) {
      uint32_t v[32];
      ptx::tmem_ld_32x32b_x32(tO + c * 32, v);
      ptx::tmem_ld_wait();
      uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 pkk;
        pkk.x = ptx::pack_bf16(__uint_as_float(v[8 * q + 0]) * inv, __uint_as_float(v[8 * q + 1]) * inv);
        pkk.y = ptx::pack_bf16(__uint_as_float(v[8 * q + 2]) * inv, __uint_as_float(v[8 * q + 3]) * inv);
        pkk.z = ptx::pack_bf16(__uint_as_float(v[8 * q + 4]) * inv, __uint_as_float(v[8 * q + 5]) * inv);
        pkk.w = ptx::pack_bf16(__uint_as_float(v[8 * q + 6]) * inv, __uint_as_float(v[8 * q + 7]) * inv);
        dst[q] = pkk;
      }
    }
    if (part == 0) lse[(static_cast<size_t>(b) * ht + h) * s + q_row] = m_used + log2f(l_tot);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

// ----------------------------------------------------------------------------- backward
// K6 on tcgen05. CTA = one (sequence, head, 128-row KV block); loops over the 128-row query tiles
// at and after the diagonal. Per tile:  S^T = K Q^T and dP^T = V dO^T (TMEM), one thread per KV
// row builds P^T = exp2(S^T*scale - lse) and dS^T = P^T (dP^T - D) in 128B-swizzled smem, then
// dV += P^T dO and dK += dS^T Q accumulate in TMEM for the whole loop while dQ_tile = dS K
// (dS^T re-read as an MN-major operand) lands in the S^T columns and is flushed with vector
// fp32 reductions into dq_acc. TMEM: S^T|dQ (128) + dP^T (128) + dV (hd) + dK (hd) <= 512.
template <int HD>
struct TcBwdCfg {
  static constexpr int NC = HD / 64;
  static constexpr int kTileBytes = 128 * 128;
  static constexpr int kOpBytes = NC * kTileBytes;  // one [128][HD] operand
  static constexpr int kSmem = 4 * kOpBytes + 2 * 2 * kTileBytes + 4 * 128 * 4 + 1024 + 256;
};

__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}



template <int HD>
__global__ void __launch_bounds__(320, 1)
    fa_bwd_tc_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                     const float* __restrict__ lse, const float* __restrict__ Dg, float* __restrict__ dq_acc,
                     __nv_bfloat16* __restrict__ dqkv, int s, int ht, float scale_log2, float scale) {
  using Cfg = TcBwdCfg<HD>;
  constexpr int NC = Cfg::NC, TB = Cfg::kTileBytes;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = ptx::smem_align1024(smem_raw);
  uint8_t* sK = smem;
  uint8_t* sV = sK + Cfg::kOpBytes;
  uint8_t* sQ = sV + Cfg::kOpBytes;
  uint8_t* sdO = sQ + Cfg::kOpBytes;
  uint8_t* sPT = sdO + Cfg::kOpBytes;  // [2 q-chunks][128 kv][64]
  uint8_t* sdST = sPT + 2 * TB;        // [2 q-chunks][128 kv][64]
  float* sL = reinterpret_cast<float*>(sdST + 2 * TB);  // [2][128]
  float* sD = sL + 2 * 128;                              // [2][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sD + 2 * 128);
  uint64_t* kv_full = bars;
  uint64_t* qdo_full = bars + 1;
  uint64_t* qdo_empty = bars + 2;
  uint64_t* sdp_full = bars + 3;
  uint64_t* sdp_free = bars + 4;
  uint64_t* pds_full = bars + 5;
  uint64_t* pds_free = bars + 6;
  uint64_t* dq_full = bars + 7;
  uint64_t* dq_free = bars + 8;
  uint64_t* kdv_full = bars + 9;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 10);

  // warp index via shfl: provably warp-uniform, so role branches are not treated as divergent
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x / 32), 0), lane = threadIdx.x % 32;
  const int kvb = blockIdx.x;
  const int b = blockIdx.y / ht, h = blockIdx.y % ht;
  const int dt = ht * HD;
  const int row0 = b * s;
  const int kv0 = kvb * 128;
  const int qt_first = kvb, qt_end = s / 128;
  const int n_it = qt_end - qt_first;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tm_qkv);
    ptx::tma_prefetch_desc(&tm_do);
    ptx::mbar_init(kv_full, 1);
    ptx::mbar_init(qdo_full, 1);
    ptx::mbar_init(qdo_empty, 1);
    ptx::mbar_init(sdp_full, 1);
    ptx::mbar_init(sdp_free, 8);
    ptx::mbar_init(pds_full, 8);
    ptx::mbar_init(pds_free, 1);
    ptx::mbar_init(dq_full, 1);
    ptx::mbar_init(dq_free, 8);
    ptx::mbar_init(kdv_full, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);  // warp-uniform
  const uint32_t tS = tmem, tdP = tmem + 128, tdV = tmem + 256, tdK = tmem + 256 + HD;

  if (warp == 0) {
    if (lane == 0) {
      ptx::mbar_arrive_expect_tx(kv_full, 2 * Cfg::kOpBytes);
      for (int c = 0; c < NC; ++c) {
        ptx::tma_load_2d(sK + c * TB, &tm_qkv, kv_full, dt + h * HD + 64 * c, row0 + kv0);
        ptx::tma_load_2d(sV + c * TB, &tm_qkv, kv_full, 2 * dt + h * HD + 64 * c, row0 + kv0);
      }
      for (int it = 0; it < n_it; ++it) {
        const int q0 = (qt_first + it) * 128;
        WAIT(qdo_empty, (it & 1) ^ 1, 20);
        ptx::mbar_arrive_expect_tx(qdo_full, 2 * Cfg::kOpBytes);
        for (int c = 0; c < NC; ++c) {
          ptx::tma_load_2d(sQ + c * TB, &tm_qkv, qdo_full, h * HD + 64 * c, row0 + q0);
          ptx::tma_load_2d(sdO + c * TB, &tm_do, qdo_full, h * HD + 64 * c, row0 + q0);
        }
      }
    }
  } else if (warp == 1) {
    {  // all 32 lanes: uniform descriptors, one elected lane issues
      constexpr uint32_t id_sq = ptx::idesc_bf16_f32(128, 128, false, false);  // S^T, dP^T
      constexpr uint32_t id_acc = ptx::idesc_bf16_f32(128, HD, false, true);   // dV, dK
      constexpr uint32_t id_dq = ptx::idesc_bf16_f32(128, HD, true, true);     // dQ
      const uint32_t aK = ptx::smem_u32(sK), aV = ptx::smem_u32(sV), aQ = ptx::smem_u32(sQ),
                     adO = ptx::smem_u32(sdO), aPT = ptx::smem_u32(sPT), adST = ptx::smem_u32(sdST);
      WAIT(kv_full, 0, 21);
      for (int it = 0; it < n_it; ++it) {
        WAIT(qdo_full, it & 1, 22);
        WAIT(dq_free, (it & 1) ^ 1, 23);
        WAIT(sdp_free, (it & 1) ^ 1, 24);
        ptx::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = (kk / 4) * TB + (kk % 4) * 32;
          ptx::mma_bf16_ss_w(tS, ptx::smem_desc_sw128(aK + off, 16, 1024), ptx::smem_desc_sw128(aQ + off, 16, 1024),
                           id_sq, kk > 0 ? 1u : 0u);
          ptx::mma_bf16_ss_w(tdP, ptx::smem_desc_sw128(aV + off, 16, 1024), ptx::smem_desc_sw128(adO + off, 16, 1024),
                           id_sq, kk > 0 ? 1u : 0u);
        }
        ptx::mma_commit_w(sdp_full);
        WAIT(pds_full, it & 1, 25);
        ptx::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 128 / 16; ++kk) {  // K = 128 query rows
          const uint32_t aoff = (kk / 4) * TB + (kk % 4) * 32;
          const uint64_t bdo = ptx::smem_desc_sw128(adO + kk * 2048, TB, 1024);
          const uint64_t bq = ptx::smem_desc_sw128(aQ + kk * 2048, TB, 1024);
          const uint32_t acc = (it > 0 || kk > 0) ? 1u : 0u;
          ptx::mma_bf16_ss_w(tdV, ptx::smem_desc_sw128(aPT + aoff, 16, 1024), bdo, id_acc, acc);
          ptx::mma_bf16_ss_w(tdK, ptx::smem_desc_sw128(adST + aoff, 16, 1024), bq, id_acc, acc);
        }
#pragma unroll
        for (int kk = 0; kk < 128 / 16; ++kk) {  // K = 128 kv rows
          ptx::mma_bf16_ss_w(tS, ptx::smem_desc_sw128(adST + kk * 2048, TB, 1024),
                           ptx::smem_desc_sw128(aK + kk * 2048, TB, 1024), id_dq, kk > 0 ? 1u : 0u);
        }
        ptx::mma_commit_w(dq_full);
        ptx::mma_commit_w(qdo_empty);
        ptx::mma_commit_w(pds_free);
      }
      ptx::mma_commit_w(kdv_full);
    }
  } else {
    // 8 compute warps: warp w owns TMEM lane quarter (w & 3) and one half of the 128 query
    // columns (P^T / dS^T) or of the head dim (dQ, dK, dV readout).
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    const int r = quarter * 32 + lane;  // TMEM lane: kv row for S^T/dP^T/dK/dV, q row for dQ
    const uint32_t lb = static_cast<uint32_t>(quarter * 32) << 16;
    const int tid = threadIdx.x - 64;   // 0..255
    const float* gL = lse + (static_cast<size_t>(b) * ht + h) * s;
    const float* gD = Dg + (static_cast<size_t>(b) * ht + h) * s;
    constexpr int NCH = HD / 32;
    const int hc0 = half ? NCH / 2 : 0, hc1 = half ? NCH : NCH / 2;
    for (int it = 0; it < n_it; ++it) {
      const int q0 = (qt_first + it) * 128;
      const int lb2 = (it & 1) * 128;
      if (tid < 128) sL[lb2 + tid] = gL[q0 + tid];
      else sD[lb2 + tid - 128] = gD[q0 + tid - 128];
      named_sync(1, 256);
      WAIT(sdp_full, it & 1, 26);
      ptx::tc_fence_after();
      WAIT(pds_free, (it & 1) ^ 1, 27);
      uint8_t* prow = sPT + half * TB + r * 128;
      uint8_t* drow = sdST + half * TB + r * 128;
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {  // 32 query columns at a time: half*64 + c*32 ..
        const int qc = half * 64 + c * 32;
        uint32_t sv[32], dv[32];
        ptx::tmem_ld_32x32b_x32(tS + lb + qc, sv);
        ptx::tmem_ld_32x32b_x32(tdP + lb + qc, dv);
        ptx::tmem_ld_wait();
        const float4* L4 = reinterpret_cast<const float4*>(sL + lb2 + qc);
        const float4* D4 = reinterpret_cast<const float4*>(sD + lb2 + qc);
        uint32_t pk[16], dk[16];
#pragma unroll
        for (int e4 = 0; e4 < 8; ++e4) {
          const float4 l4 = L4[e4], d4 = D4[e4];
          const float lv[4] = {l4.x, l4.y, l4.z, l4.w}, dvv[4] = {d4.x, d4.y, d4.z, d4.w};
          float p[4], ds[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            p[k] = ex2(fmaf(__uint_as_float(sv[4 * e4 + k]), scale_log2, -lv[k]));
            ds[k] = p[k] * (__uint_as_float(dv[4 * e4 + k]) - dvv[k]);
          }
          pk[2 * e4] = ptx::pack_bf16(p[0], p[1]);
          pk[2 * e4 + 1] = ptx::pack_bf16(p[2], p[3]);
          dk[2 * e4] = ptx::pack_bf16(ds[0], ds[1]);
          dk[2 * e4 + 1] = ptx::pack_bf16(ds[2], ds[3]);
        }
        if (it == 0 && qc < r + 1) {  // diagonal tile: queries before this kv row see nothing
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (qc + e < r) {
              pk[e / 2] &= (e & 1) ? 0x0000FFFFu : 0xFFFF0000u;
              dk[e / 2] &= (e & 1) ? 0x0000FFFFu : 0xFFFF0000u;
            }
        }
        // columns qc..qc+31 = 16B units u0..u0+3 (u0 = c*4) of this half's swizzle chunk
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int off = ((c * 4 + u) ^ (r & 7)) * 16;
          *reinterpret_cast<uint4*>(prow + off) = make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
          *reinterpret_cast<uint4*>(drow + off) = make_uint4(dk[4 * u], dk[4 * u + 1], dk[4 * u + 2], dk[4 * u + 3]);
        }
      }
      ptx::fence_proxy_async();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        ptx::mbar_arrive(sdp_free);
        ptx::mbar_arrive(pds_full);
      }
      // dQ tile (thread = query row q0 + r, this half's head-dim columns) -> fp32 reductions
      WAIT(dq_full, it & 1, 28);
      ptx::tc_fence_after();
      float* dqrow = dq_acc + static_cast<size_t>(row0 + q0 + r) * dt + h * HD;
#pragma unroll 1
      for (int c = hc0; c < hc1; ++c) {
        uint32_t v[32];
        ptx::tmem_ld_32x32b_x32(tS + lb + c * 32, v);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; e += 4)
          red_add_v4(dqrow + c * 32 + e, __uint_as_float(v[e]), __uint_as_float(v[e + 1]), __uint_as_float(v[e + 2]),
                     __uint_as_float(v[e + 3]));
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(dq_free);
    }
    // dK (scaled) and dV rows of this KV block (this half's head-dim columns)
    WAIT(kdv_full, 0, 29);
    ptx::tc_fence_after();
    __nv_bfloat16* krow = dqkv + static_cast<size_t>(row0 + kv0 + r) * 3 * dt + dt + h * HD;
    __nv_bfloat16* vrow = krow + dt;
#pragma unroll 1
    for (int c = hc0; c < hc1; ++c) {
      uint32_t kv[32], vv[32];
      ptx::tmem_ld_32x32b_x32(tdK + lb + c * 32, kv);
      ptx::tmem_ld_32x32b_x32(tdV + lb + c * 32, vv);
      ptx::tmem_ld_wait();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 a, bb;
        a.x = ptx::pack_bf16(__uint_as_float(kv[8 * q]) * scale, __uint_as_float(kv[8 * q + 1]) * scale);
        a.y = ptx::pack_bf16(__uint_as_float(kv[8 * q + 2]) * scale, __uint_as_float(kv[8 * q + 3]) * scale);
        a.z = ptx::pack_bf16(__uint_as_float(kv[8 * q + 4]) * scale, __uint_as_float(kv[8 * q + 5]) * scale);
        a.w = ptx::pack_bf16(__uint_as_float(kv[8 * q + 6]) * scale, __uint_as_float(kv[8 * q + 7]) * scale);
        bb.x = ptx::pack_bf16(__uint_as_float(vv[8 * q]), __uint_as_float(vv[8 * q + 1]));
        bb.y = ptx::pack_bf16(__uint_as_float(vv[8 * q + 2]), __uint_as_float(vv[8 * q + 3]));
        bb.z = ptx::pack_bf16(__uint_as_float(vv[8 * q + 4]), __uint_as_float(vv[8 * q + 5]));
        bb.w = ptx::pack_bf16(__uint_as_float(vv[8 * q + 6]), __uint_as_float(vv[8 * q + 7]));
        reinterpret_cast<uint4*>(krow + c * 32)[q] = a;
        reinterpret_cast<uint4*>(vrow + c * 32)[q] = bb;
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

// K6 (hd 128), pipelined: 64-row query tiles so Q/dO and P^T/dS^T double-buffer in smem and
// S^T/dP^T double-buffer in TMEM. Per tile j the MMA warp issues stage 1 (S^T_j = K Q_j^T,
// dP^T_j = V dO_j^T) and then stage 2 of tile j-1 (dV += P^T dO, dK += dS^T Q, and
// dQ^T = K^T dS^T into the S^T buffer the compute warps have just drained), so the compute warps'
// exp/dS work on tile j overlaps the tensor core on tile j-1. TMEM: S^T|dQ^T (2x64) + dP^T
// (2x64) + dV (128) + dK (128) = 512 columns. dQ^T rows are head-dim lanes: the flush into
// dq_acc is one coalesced fp32 reduction per (query, 32 head dims) per warp.
// 16 warps, register-rebalanced per warpgroup (setmaxnreg): WG0 = TMA producer (warp 0) + MMA
// issuer (warp 1); WG1-2 = P/dS compute (TMEM lane quarter x 32-query half); WG3 = dQ flush, one
// warp per 32 head dims, each staging its own [64 q][32 hd] box and issuing its own TMA
// reduce-add, so the flush of tile j-1 runs concurrently with the P/dS math of tile j.
// Column sums over a warp's 32 rows (lane = row) of 32 columns (x[e] = column e of this lane's row):
// a butterfly in which every level halves the columns a lane carries; lane l ends with column l.
// 31 shuffles for 32 columns. Used to fold the qkv bias gradient into the backward's dK / dV epilogue.
__device__ __forceinline__ float warp_colsum32(float (&x)[32], int lane) {
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) {
    const bool up = (lane & w) != 0;
#pragma unroll
    for (int i = 0; i < w; ++i) {
      const float send = up ? x[i] : x[i + w];
      const float keep = up ? x[i + w] : x[i];
      x[i] = keep + __shfl_xor_sync(0xffffffffu, send, w);
    }
  }
  return x[0];
}

template <int HD>
struct TcBwd2Cfg {
  static constexpr int NC = HD / 64;
  static constexpr int kTileBytes = 128 * 128;         // [128 rows][64] bf16
  static constexpr int kKVBytes = NC * kTileBytes;     // [128 kv][HD]
  static constexpr int kQBytes = NC * 64 * 128;        // [64 q][HD]
  static constexpr int kPBytes = 128 * 128;            // [128 kv][64 q]
  static constexpr int QST = 3;                        // Q/dO (+ LSE/D) ring depth
  static constexpr int kSmem = 2 * kKVBytes + 2 * QST * kQBytes + 4 * kPBytes + QST * 2 * 64 * 4 + 1024 + 256;
  static_assert(kSmem <= 232448, "smem over the 227 KB opt-in limit");
};

// TP (P^T / dS^T in TMEM): the compute warps write P^T and dS^T as packed bf16 over the S^T
// columns they have just read (each half of the tile into its own 32 columns: P^T 16, dS^T 16), and
// dV += P^T dO, dK += dS^T Q read their A operand from TMEM; only dS^T goes to shared memory (the B
// operand of dQ^T). S^T_{j+2} overwrites those columns after stage 2 of tile j in the same in-order
// MMA stream.
template <int HD, bool TP>
__global__ void __launch_bounds__(512, 1)
    fa_bwd_tc2_kernel(const __grid_constant__ CUtensorMap tm_kv, const __grid_constant__ CUtensorMap tm_q,
                      const __grid_constant__ CUtensorMap tm_do, const float* __restrict__ lse,
                      const float* __restrict__ Dg, float* __restrict__ dq_acc, __nv_bfloat16* __restrict__ dqkv,
                      float* __restrict__ dbqkv, int s, int ht, float scale_log2, float scale) {
  using Cfg = TcBwd2Cfg<HD>;
  constexpr int NC = Cfg::NC, TB = Cfg::kTileBytes;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = ptx::smem_align1024(smem_raw);
  uint8_t* sK = smem;
  uint8_t* sV = sK + Cfg::kKVBytes;
  constexpr int QST = Cfg::QST;
  uint8_t* sQ = sV + Cfg::kKVBytes;          // [QST][NC][64][64]
  uint8_t* sdO = sQ + QST * Cfg::kQBytes;    // [QST][NC][64][64]
  uint8_t* sPT = sdO + QST * Cfg::kQBytes;   // [2][128 kv][64 q]
  uint8_t* sdST = sPT + 2 * Cfg::kPBytes;    // [2][128 kv][64 q]
  float* sL = reinterpret_cast<float*>(sdST + 2 * Cfg::kPBytes);  // [QST][64]
  float* sD = sL + QST * 64;                                      // [QST][64]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sD + QST * 64);
  uint64_t* kv_full = bars;
  uint64_t* qdo_full = bars + 1;            // [QST]
  uint64_t* qdo_empty = qdo_full + QST;     // [QST]
  uint64_t* s_full = qdo_empty + QST;       // [2]
  uint64_t* pds_full = s_full + 2;          // [2]
  uint64_t* pds_free = pds_full + 2;        // [2]
  uint64_t* st_free = pds_free + 2;         // [2]  S^T_j / dP^T_j read out by the compute warps
  uint64_t* dq_full = st_free + 2;          // dQ^T in its own TMEM columns
  uint64_t* dq_free = dq_full + 1;
  uint64_t* kdv_full = dq_free + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(kdv_full + 1);

  // warp index via shfl: provably warp-uniform, so role branches are not treated as divergent
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x / 32), 0), lane = threadIdx.x % 32;
  const int kvb = blockIdx.x;
  const int b = blockIdx.y / ht, h = blockIdx.y % ht;
  const int dt = ht * HD;
  const int row0 = b * s;
  const int kv0 = kvb * 128;
  const int qt_first = kv0 / 64;          // 64-row query tiles at and after the diagonal
  const int n_it = s / 64 - qt_first;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tm_kv);
    ptx::tma_prefetch_desc(&tm_q);
    ptx::tma_prefetch_desc(&tm_do);
    ptx::mbar_init(kv_full, 1);
    for (int i = 0; i < QST; ++i) {
      ptx::mbar_init(&qdo_full[i], 1);
      ptx::mbar_init(&qdo_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&s_full[i], 1);
      ptx::mbar_init(&pds_full[i], 8);
      ptx::mbar_init(&pds_free[i], 1);
      ptx::mbar_init(&st_free[i], 8);
    }
    ptx::mbar_init(dq_full, 1);
    ptx::mbar_init(dq_free, 4);
    ptx::mbar_init(kdv_full, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);  // warp-uniform
  pdl_trigger();  // prologue (smem / TMEM / barriers) done: see pdl.cuh
  pdl_wait();
  // TMEM: S^T [2][64] | dP^T [64] (released as soon as it is loaded) | dQ^T [64] | dV | dK
  const uint32_t tS = tmem, tdP = tmem + 128, tDQ = tmem + 192, tdV = tmem + 256, tdK = tmem + 256 + HD;
  const int wg = warp / 4;
  if (wg == 0) ptx::setmaxnreg_dec<64>();

  if (warp == 0) {
    if (lane == 0) {
      const float* gLq = lse + (static_cast<size_t>(b) * ht + h) * s;
      const float* gDq = Dg + (static_cast<size_t>(b) * ht + h) * s;
      ptx::mbar_arrive_expect_tx(kv_full, 2 * Cfg::kKVBytes);
      for (int c = 0; c < NC; ++c) {
        ptx::tma_load_2d(sK + c * TB, &tm_kv, kv_full, dt + h * HD + 64 * c, row0 + kv0);
        ptx::tma_load_2d(sV + c * TB, &tm_kv, kv_full, 2 * dt + h * HD + 64 * c, row0 + kv0);
      }
      for (int j = 0; j < n_it; ++j) {
        const int sq = j % QST;
        const int q0 = (qt_first + j) * 64;
        WAIT(&qdo_empty[sq], ((j / QST) & 1) ^ 1, 40);
        ptx::mbar_arrive_expect_tx(&qdo_full[sq], 2 * Cfg::kQBytes + 2 * 64 * 4);
        for (int c = 0; c < NC; ++c) {
          ptx::tma_load_2d(sQ + sq * Cfg::kQBytes + c * 8192, &tm_q, &qdo_full[sq], h * HD + 64 * c, row0 + q0);
          ptx::tma_load_2d(sdO + sq * Cfg::kQBytes + c * 8192, &tm_do, &qdo_full[sq], h * HD + 64 * c, row0 + q0);
        }
        // the tile's LSE and D rows ride on the same transaction
        ptx::bulk_load(sL + sq * 64, gLq + q0, 64 * 4, &qdo_full[sq]);
        ptx::bulk_load(sD + sq * 64, gDq + q0, 64 * 4, &qdo_full[sq]);
      }
    }
  } else if (warp == 1) {
    {  // all 32 lanes: uniform descriptors, one elected lane issues
      constexpr uint32_t id_s = ptx::idesc_bf16_f32(128, 64, false, false);   // S^T, dP^T
      constexpr uint32_t id_acc = ptx::idesc_bf16_f32(128, HD, false, true);  // dV, dK
      constexpr uint32_t id_dq = ptx::idesc_bf16_f32(HD, 64, true, true);     // dQ^T
      // Shared-window addresses from the symbol (provably warp-uniform, so descriptors stay in
      // uniform registers): same layout as the generic pointers above.
      const uint32_t u0 = (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) + 1023u) & ~1023u;
      const uint32_t aK = u0, aV = u0 + Cfg::kKVBytes;
      const uint32_t aQ0 = u0 + 2 * Cfg::kKVBytes, adO0 = aQ0 + QST * Cfg::kQBytes;
      const uint32_t aP0 = adO0 + QST * Cfg::kQBytes, adS0 = aP0 + 2 * Cfg::kPBytes;
      WAIT(kv_full, 0, 41);
      auto stage2 = [&](int i) {
        const int bb = i & 1, sq = i % QST;
        ATTN_TRACE(3, i);
        WAIT(&pds_full[bb], (i >> 1) & 1, 42);
        ATTN_TRACE(4, i);
        ptx::tc_fence_after();
        const uint32_t aQ = aQ0 + sq * Cfg::kQBytes, adO = adO0 + sq * Cfg::kQBytes;
        const uint32_t aP = aP0 + bb * Cfg::kPBytes, adS = adS0 + bb * Cfg::kPBytes;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {  // K = 64 query rows
          const uint32_t acc = (i > 0 || kk > 0) ? 1u : 0u;
          if constexpr (TP) {  // 16 query rows = 8 packed columns; half h of the tile at column 32 h
            const uint32_t ta = tS + bb * 64 + (kk >> 1) * 32 + (kk & 1) * 8;
            ptx::mma_bf16_ts_w(tdV, ta, ptx::smem_desc_sw128(adO + kk * 2048, 8192, 1024), id_acc, acc);
            ptx::mma_bf16_ts_w(tdK, ta + 16, ptx::smem_desc_sw128(aQ + kk * 2048, 8192, 1024), id_acc, acc);
          } else {
            ptx::mma_bf16_ss_w(tdV, ptx::smem_desc_sw128(aP + kk * 32, 16, 1024),
                               ptx::smem_desc_sw128(adO + kk * 2048, 8192, 1024), id_acc, acc);
            ptx::mma_bf16_ss_w(tdK, ptx::smem_desc_sw128(adS + kk * 32, 16, 1024),
                               ptx::smem_desc_sw128(aQ + kk * 2048, 8192, 1024), id_acc, acc);
          }
        }
        if (i > 0) WAIT(dq_free, (i - 1) & 1, 44);  // dQ^T_{i-1} read out of its TMEM columns
        ATTN_TRACE(5, i);
        ptx::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)  // K = 128 kv rows
          ptx::mma_bf16_ss_w(tDQ, ptx::smem_desc_sw128(aK + kk * 2048, TB, 1024),
                             ptx::smem_desc_sw128(adS + kk * 2048, TB, 1024), id_dq, kk > 0 ? 1u : 0u);
        ptx::mma_commit_w(dq_full);
        ptx::mma_commit_w(&qdo_empty[sq]);
        ptx::mma_commit_w(&pds_free[bb]);
        ATTN_TRACE(6, i);
      };
      for (int j = 0; j < n_it; ++j) {
        const int bb = j & 1, sq = j % QST;
        ATTN_TRACE(0, j);
        WAIT(&qdo_full[sq], (j / QST) & 1, 43);
        // S^T_{j-1} and dP^T_{j-1} loaded by the compute warps: dP^T is free, and so is S^T[bb]
        // (its previous tile j-2 was loaded before j-1)
        if (j >= 1) WAIT(&st_free[(j - 1) & 1], ((j - 1) >> 1) & 1, 50);
        ATTN_TRACE(1, j);
        ptx::tc_fence_after();
        const uint32_t aQ = aQ0 + sq * Cfg::kQBytes, adO = adO0 + sq * Cfg::kQBytes;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t ak = (kk / 4) * TB + (kk % 4) * 32, aq = (kk / 4) * 8192 + (kk % 4) * 32;
          ptx::mma_bf16_ss_w(tS + bb * 64, ptx::smem_desc_sw128(aK + ak, 16, 1024),
                           ptx::smem_desc_sw128(aQ + aq, 16, 1024), id_s, kk > 0 ? 1u : 0u);
          ptx::mma_bf16_ss_w(tdP, ptx::smem_desc_sw128(aV + ak, 16, 1024),
                           ptx::smem_desc_sw128(adO + aq, 16, 1024), id_s, kk > 0 ? 1u : 0u);
        }
        ptx::mma_commit_w(&s_full[bb]);
        ATTN_TRACE(2, j);
        if (j > 0) stage2(j - 1);
      }
      stage2(n_it - 1);
      ptx::mma_commit_w(kdv_full);
    }
  } else if (wg == 3) {
    ptx::setmaxnreg_dec<64>();
    // dQ_i flush: TMEM (lane = head dim, column = query) -> fp32 reductions into dq_acc; per
    // query one warp instruction covers 32 consecutive head dims (one 128-byte L2 request).
    const int quarter = warp & 3;
    const uint32_t lb = static_cast<uint32_t>(quarter * 32) << 16;
    for (int i = 0; i < n_it; ++i) {
      const int q0 = (qt_first + i) * 64;
      float* dst = dq_acc + static_cast<size_t>(row0 + q0) * dt + h * HD + quarter * 32;
      WAIT(dq_full, i & 1, 45);
      if (quarter == 0) ATTN_TRACE(14, i);
      ptx::tc_fence_after();
#pragma unroll
      for (int hq = 0; hq < 2; ++hq) {
        uint32_t v[32];
        ptx::tmem_ld_32x32b_x32(tDQ + lb + hq * 32, v);
        ptx::tmem_ld_wait();
        if (hq == 1) {
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(dq_free);
        }
#pragma unroll
        for (int e = 0; e < 32; ++e) atomicAdd(dst + static_cast<size_t>(hq * 32 + e) * dt + lane, __uint_as_float(v[e]));
      }
      if (quarter == 0) ATTN_TRACE(15, i);
    }
  } else if (wg == 1 || wg == 2) {
    ptx::setmaxnreg_inc<192>();
    const int quarter = warp & 3;
    const int half = wg - 1;            // which 32 query columns of the 64-row tile
    const int r = quarter * 32 + lane;  // TMEM lane: kv row (S^T, dP^T, dK, dV)
    const uint32_t lb = static_cast<uint32_t>(quarter * 32) << 16;
    for (int j = 0; j < n_it; ++j) {
      const int bb = j & 1, sq = j % QST;
      const int q0 = (qt_first + j) * 64;
      const bool tw = warp == 4;  // traced compute warp (half 0, quarter 0)
      if (tw) ATTN_TRACE(8, j);
      WAIT(&s_full[bb], (j >> 1) & 1, 46);
      if (tw) ATTN_TRACE(9, j);
      WAIT(&qdo_full[sq], (j / QST) & 1, 49);  // LSE / D rows of this tile (already complete)
      ptx::tc_fence_after();
      const int qc = half * 32;
      uint32_t sv[32], dv[32];
      ptx::tmem_ld_32x32b_x32(tS + lb + bb * 64 + qc, sv);
      ptx::tmem_ld_32x32b_x32(tdP + lb + qc, dv);
      ptx::tmem_ld_wait();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&st_free[bb]);  // S^T / dP^T of this tile consumed
      if (tw) ATTN_TRACE(10, j);
      const float4* L4 = reinterpret_cast<const float4*>(sL + sq * 64 + qc);
      const float4* D4 = reinterpret_cast<const float4*>(sD + sq * 64 + qc);
      uint32_t pk[16], dk[16];
#pragma unroll
      for (int e4 = 0; e4 < 8; ++e4) {
        const float4 l4 = L4[e4], d4 = D4[e4];
        const float lv[4] = {l4.x, l4.y, l4.z, l4.w}, dvv[4] = {d4.x, d4.y, d4.z, d4.w};
        float pp[4], ds[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          pp[k] = ex2(fmaf(__uint_as_float(sv[4 * e4 + k]), scale_log2, -lv[k]));
          ds[k] = pp[k] * (__uint_as_float(dv[4 * e4 + k]) - dvv[k]);
        }
        pk[2 * e4] = ptx::pack_bf16(pp[0], pp[1]);
        pk[2 * e4 + 1] = ptx::pack_bf16(pp[2], pp[3]);
        dk[2 * e4] = ptx::pack_bf16(ds[0], ds[1]);
        dk[2 * e4 + 1] = ptx::pack_bf16(ds[2], ds[3]);
      }
      if (q0 + qc < kv0 + r) {  // near the diagonal: queries before this kv row see nothing
#pragma unroll
        for (int e = 0; e < 32; ++e)
          if (q0 + qc + e < kv0 + r) {
            pk[e / 2] &= (e & 1) ? 0x0000FFFFu : 0xFFFF0000u;
            dk[e / 2] &= (e & 1) ? 0x0000FFFFu : 0xFFFF0000u;
          }
      }
      if (tw) ATTN_TRACE(11, j);
      if constexpr (TP) {  // over this half's own (already read) S^T columns
        ptx::tmem_st_32x32b_x16(tS + lb + bb * 64 + qc, pk);
        ptx::tmem_st_32x32b_x16(tS + lb + bb * 64 + qc + 16, dk);
      }
      WAIT(&pds_free[bb], ((j >> 1) & 1) ^ 1, 47);  // stage 2 of tile j-2 is done with buffer bb
      if (tw) ATTN_TRACE(12, j);
      uint8_t* prow = sPT + bb * Cfg::kPBytes + r * 128;
      uint8_t* drow = sdST + bb * Cfg::kPBytes + r * 128;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int off = ((half * 4 + u) ^ (r & 7)) * 16;
        if constexpr (!TP)
          *reinterpret_cast<uint4*>(prow + off) = make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
        *reinterpret_cast<uint4*>(drow + off) = make_uint4(dk[4 * u], dk[4 * u + 1], dk[4 * u + 2], dk[4 * u + 3]);
      }
      if (tw) ATTN_TRACE(16, j);
      ptx::fence_proxy_async();
      if (tw) ATTN_TRACE(17, j);
      if constexpr (TP) ptx::tmem_st_wait();
      if (tw) ATTN_TRACE(18, j);
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&pds_full[bb]);
      if (tw) ATTN_TRACE(13, j);
    }
    // dK (scaled) and dV rows of this KV block
    WAIT(kdv_full, 0, 48);
    ptx::tc_fence_after();
    __nv_bfloat16* krow = dqkv + static_cast<size_t>(row0 + kv0 + r) * 3 * dt + dt + h * HD;
    __nv_bfloat16* vrow = krow + dt;
    constexpr int NCH = HD / 32;
#pragma unroll 1
    for (int c = half * (NCH / 2); c < (half + 1) * (NCH / 2); ++c) {
      uint32_t kv[32], vv[32];
      ptx::tmem_ld_32x32b_x32(tdK + lb + c * 32, kv);
      ptx::tmem_ld_32x32b_x32(tdV + lb + c * 32, vv);
      ptx::tmem_ld_wait();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 a, bb2;
        a.x = ptx::pack_bf16(__uint_as_float(kv[8 * q]) * scale, __uint_as_float(kv[8 * q + 1]) * scale);
        a.y = ptx::pack_bf16(__uint_as_float(kv[8 * q + 2]) * scale, __uint_as_float(kv[8 * q + 3]) * scale);
        a.z = ptx::pack_bf16(__uint_as_float(kv[8 * q + 4]) * scale, __uint_as_float(kv[8 * q + 5]) * scale);
        a.w = ptx::pack_bf16(__uint_as_float(kv[8 * q + 6]) * scale, __uint_as_float(kv[8 * q + 7]) * scale);
        bb2.x = ptx::pack_bf16(__uint_as_float(vv[8 * q]), __uint_as_float(vv[8 * q + 1]));
        bb2.y = ptx::pack_bf16(__uint_as_float(vv[8 * q + 2]), __uint_as_float(vv[8 * q + 3]));
        bb2.z = ptx::pack_bf16(__uint_as_float(vv[8 * q + 4]), __uint_as_float(vv[8 * q + 5]));
        bb2.w = ptx::pack_bf16(__uint_as_float(vv[8 * q + 6]), __uint_as_float(vv[8 * q + 7]));
        reinterpret_cast<uint4*>(krow + c * 32)[q] = a;
        reinterpret_cast<uint4*>(vrow + c * 32)[q] = bb2;
      }
      if (dbqkv) {  // qkv bias gradient, k and v parts: this warp's 32 kv rows of columns c*32..+31
        float x[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) x[e] = __uint_as_float(kv[e]) * scale;
        atomicAdd(dbqkv + dt + h * HD + c * 32 + lane, warp_colsum32(x, lane));
#pragma unroll
        for (int e = 0; e < 32; ++e) x[e] = __uint_as_float(vv[e]);
        atomicAdd(dbqkv + 2 * dt + h * HD + c * 32 + lane, warp_colsum32(x, lane));
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

template <int HD>
__global__ void __launch_bounds__(512, 1)
    fa_bwd_tc2_persistent(const __grid_constant__ CUtensorMap tm_kv, const __grid_constant__ CUtensorMap tm_q,
                      const __grid_constant__ CUtensorMap tm_do, const float* __restrict__ lse,
                      const float* __restrict__ Dg, float* __restrict__ dq_acc, __nv_bfloat16* __restrict__ dqkv,
                      float* __restrict__ dbqkv, int s, int ht, int batch, float scale_log2, float scale) {
  using Cfg = TcBwd2Cfg<HD>;
  constexpr int NC = Cfg::NC, TB = Cfg::kTileBytes;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = ptx::smem_align1024(smem_raw);
  uint8_t* sK = smem;
  uint8_t* sV = sK + Cfg::kKVBytes;
  constexpr int QST = Cfg::QST;
  uint8_t* sQ = sV + Cfg::kKVBytes;          // [QST][NC][64][64]
  uint8_t* sdO = sQ + QST * Cfg::kQBytes;    // [QST][NC][64][64]
  uint8_t* sPT = sdO + QST * Cfg::kQBytes;   // [2][128 kv][64 q]
  uint8_t* sdST = sPT + 2 * Cfg::kPBytes;    // [2][128 kv][64 q]
  float* sL = reinterpret_cast<float*>(sdST + 2 * Cfg::kPBytes);  // [QST][64]
  float* sD = sL + QST * 64;                                      // [QST][64]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sD + QST * 64);
  uint64_t* kv_full = bars;
  uint64_t* qdo_full = bars + 1;            // [QST]
  uint64_t* qdo_empty = qdo_full + QST;     // [QST]
  uint64_t* s_full = qdo_empty + QST;       // [2]
  uint64_t* pds_full = s_full + 2;          // [2]
  uint64_t* pds_free = pds_full + 2;        // [2]
  uint64_t* st_free = pds_free + 2;         // [2]  S^T_j / dP^T_j read out by the compute warps
  uint64_t* dq_full = st_free + 2;          // dQ^T in its own TMEM columns
  uint64_t* dq_free = dq_full + 1;
  uint64_t* kdv_full = dq_free + 1;
  uint64_t* kv_empty = kdv_full + 1;  // every MMA reading this item's K / V complete
  uint64_t* kdv_free = kv_empty + 1;  // dK / dV drained from TMEM by the epilogue
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(kdv_free + 1);

  // warp index via shfl: provably warp-uniform, so role branches are not treated as divergent
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x / 32), 0), lane = threadIdx.x % 32;
  const int dt = ht * HD;
  const int n_kvb = s / 128, BH = batch * ht;
  const int n_items = n_kvb * BH;
  // work items (kv block, sequence-head), heaviest (kv block 0) first, handed out in snake order
  auto snake = [&](int t) {
    const int G = gridDim.x, c = blockIdx.x;
    return t * G + ((t & 1) ? G - 1 - c : c);
  };
  struct Item {
    int b, h, row0, kv0, qt_first, n_it;
  };
  auto item = [&](int kidx) {
    Item it;
    const int kvb = kidx / BH, bh = kidx % BH;
    it.b = bh / ht;
    it.h = bh % ht;
    it.row0 = it.b * s;
    it.kv0 = kvb * 128;
    it.qt_first = it.kv0 / 64;
    it.n_it = s / 64 - it.qt_first;
    return it;
  };

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tm_kv);
    ptx::tma_prefetch_desc(&tm_q);
    ptx::tma_prefetch_desc(&tm_do);
    ptx::mbar_init(kv_full, 1);
    for (int i = 0; i < QST; ++i) {
      ptx::mbar_init(&qdo_full[i], 1);
      ptx::mbar_init(&qdo_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&s_full[i], 1);
      ptx::mbar_init(&pds_full[i], 8);
      ptx::mbar_init(&pds_free[i], 1);
      ptx::mbar_init(&st_free[i], 8);
    }
    ptx::mbar_init(dq_full, 1);
    ptx::mbar_init(dq_free, 4);
    ptx::mbar_init(kdv_full, 1);
    ptx::mbar_init(kv_empty, 1);
    ptx::mbar_init(kdv_free, 8);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);  // warp-uniform
  pdl_trigger();  // prologue (smem / TMEM / barriers) done: see pdl.cuh
  pdl_wait();
  // TMEM: S^T [2][64] | dP^T [64] (released as soon as it is loaded) | dQ^T [64] | dV | dK
  const uint32_t tS = tmem, tdP = tmem + 128, tDQ = tmem + 192, tdV = tmem + 256, tdK = tmem + 256 + HD;
  const int wg = warp / 4;
  if (wg == 0) ptx::setmaxnreg_dec<64>();

  if (warp == 0) {
    if (lane == 0) {
      int gt = 0, t = 0;
      for (int kidx = snake(0); kidx < n_items; kidx = snake(t + 1), ++t) {
        const Item it = item(kidx);
        const float* gLq = lse + (static_cast<size_t>(it.b) * ht + it.h) * s;
        const float* gDq = Dg + (static_cast<size_t>(it.b) * ht + it.h) * s;
        WAIT(kv_empty, (t & 1) ^ 1, 39);  // previous item's MMAs are done with K / V
        ptx::mbar_arrive_expect_tx(kv_full, 2 * Cfg::kKVBytes);
        for (int c = 0; c < NC; ++c) {
          ptx::tma_load_2d(sK + c * TB, &tm_kv, kv_full, dt + it.h * HD + 64 * c, it.row0 + it.kv0);
          ptx::tma_load_2d(sV + c * TB, &tm_kv, kv_full, 2 * dt + it.h * HD + 64 * c, it.row0 + it.kv0);
        }
        for (int j = 0; j < it.n_it; ++j, ++gt) {
          const int sq = gt % QST;
          const int q0 = (it.qt_first + j) * 64;
          WAIT(&qdo_empty[sq], ((gt / QST) & 1) ^ 1, 40);
          ptx::mbar_arrive_expect_tx(&qdo_full[sq], 2 * Cfg::kQBytes + 2 * 64 * 4);
          for (int c = 0; c < NC; ++c) {
            ptx::tma_load_2d(sQ + sq * Cfg::kQBytes + c * 8192, &tm_q, &qdo_full[sq], it.h * HD + 64 * c, it.row0 + q0);
            ptx::tma_load_2d(sdO + sq * Cfg::kQBytes + c * 8192, &tm_do, &qdo_full[sq], it.h * HD + 64 * c,
                             it.row0 + q0);
          }
          ptx::bulk_load(sL + sq * 64, gLq + q0, 64 * 4, &qdo_full[sq]);
          ptx::bulk_load(sD + sq * 64, gDq + q0, 64 * 4, &qdo_full[sq]);
        }
      }
    }
  } else if (warp == 1) {
    {  // all 32 lanes: uniform descriptors, one elected lane issues
      constexpr uint32_t id_s = ptx::idesc_bf16_f32(128, 64, false, false);   // S^T, dP^T
      constexpr uint32_t id_acc = ptx::idesc_bf16_f32(128, HD, false, true);  // dV, dK
      constexpr uint32_t id_dq = ptx::idesc_bf16_f32(HD, 64, true, true);     // dQ^T
      // Shared-window addresses from the symbol (provably warp-uniform, so descriptors stay in
      // uniform registers): same layout as the generic pointers above.
      const uint32_t u0 = (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) + 1023u) & ~1023u;
      const uint32_t aK = u0, aV = u0 + Cfg::kKVBytes;
      const uint32_t aQ0 = u0 + 2 * Cfg::kKVBytes, adO0 = aQ0 + QST * Cfg::kQBytes;
      const uint32_t aP0 = adO0 + QST * Cfg::kQBytes, adS0 = aP0 + 2 * Cfg::kPBytes;
      int gt = 0, t = 0;
      for (int kidx = snake(0); kidx < n_items; kidx = snake(t + 1), ++t) {
        const int n_it = item(kidx).n_it;
        WAIT(kv_full, t & 1, 41);
        auto stage2 = [&](int i, int g) {  // i: tile within the item, g: global tile
          const int bb = g & 1, sq = g % QST;
          if (i == 0 && t > 0) WAIT(kdv_free, (t - 1) & 1, 51);  // previous item's dK / dV drained
          WAIT(&pds_full[bb], (g >> 1) & 1, 42);
          ptx::tc_fence_after();
          const uint32_t aQ = aQ0 + sq * Cfg::kQBytes, adO = adO0 + sq * Cfg::kQBytes;
          const uint32_t aP = aP0 + bb * Cfg::kPBytes, adS = adS0 + bb * Cfg::kPBytes;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {  // K = 64 query rows
            const uint32_t acc = (i > 0 || kk > 0) ? 1u : 0u;
            ptx::mma_bf16_ss_w(tdV, ptx::smem_desc_sw128(aP + kk * 32, 16, 1024),
                               ptx::smem_desc_sw128(adO + kk * 2048, 8192, 1024), id_acc, acc);
            ptx::mma_bf16_ss_w(tdK, ptx::smem_desc_sw128(adS + kk * 32, 16, 1024),
                               ptx::smem_desc_sw128(aQ + kk * 2048, 8192, 1024), id_acc, acc);
          }
          if (g > 0) WAIT(dq_free, (g - 1) & 1, 44);  // dQ^T_{g-1} read out of its TMEM columns
          ptx::tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)  // K = 128 kv rows
            ptx::mma_bf16_ss_w(tDQ, ptx::smem_desc_sw128(aK + kk * 2048, TB, 1024),
                               ptx::smem_desc_sw128(adS + kk * 2048, TB, 1024), id_dq, kk > 0 ? 1u : 0u);
          ptx::mma_commit_w(dq_full);
          ptx::mma_commit_w(&qdo_empty[sq]);
          ptx::mma_commit_w(&pds_free[bb]);
        };
        for (int j = 0; j < n_it; ++j) {
          const int g = gt + j, bb = g & 1, sq = g % QST;
          WAIT(&qdo_full[sq], (g / QST) & 1, 43);
          if (g >= 1) WAIT(&st_free[(g - 1) & 1], ((g - 1) >> 1) & 1, 50);
          ptx::tc_fence_after();
          const uint32_t aQ = aQ0 + sq * Cfg::kQBytes, adO = adO0 + sq * Cfg::kQBytes;
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {
            const uint32_t ak = (kk / 4) * TB + (kk % 4) * 32, aq = (kk / 4) * 8192 + (kk % 4) * 32;
            ptx::mma_bf16_ss_w(tS + bb * 64, ptx::smem_desc_sw128(aK + ak, 16, 1024),
                               ptx::smem_desc_sw128(aQ + aq, 16, 1024), id_s, kk > 0 ? 1u : 0u);
            ptx::mma_bf16_ss_w(tdP, ptx::smem_desc_sw128(aV + ak, 16, 1024),
                               ptx::smem_desc_sw128(adO + aq, 16, 1024), id_s, kk > 0 ? 1u : 0u);
          }
          ptx::mma_commit_w(&s_full[bb]);
          if (j > 0) stage2(j - 1, g - 1);
        }
        stage2(n_it - 1, gt + n_it - 1);
        ptx::mma_commit_w(kdv_full);
        ptx::mma_commit_w(kv_empty);
        gt += n_it;
      }
    }
  } else if (wg == 3) {
    ptx::setmaxnreg_dec<64>();
    // dQ_i flush: TMEM (lane = head dim, column = query) -> fp32 reductions into dq_acc; per
    // query one warp instruction covers 32 consecutive head dims (one 128-byte L2 request).
    const int quarter = warp & 3;
    const uint32_t lb = static_cast<uint32_t>(quarter * 32) << 16;
    int gt = 0, t = 0;
    for (int kidx = snake(0); kidx < n_items; kidx = snake(t + 1), ++t) {
      const Item it = item(kidx);
      for (int i = 0; i < it.n_it; ++i, ++gt) {
        const int q0 = (it.qt_first + i) * 64;
        float* dst = dq_acc + static_cast<size_t>(it.row0 + q0) * dt + it.h * HD + quarter * 32;
        WAIT(dq_full, gt & 1, 45);
        ptx::tc_fence_after();
#pragma unroll
        for (int hq = 0; hq < 2; ++hq) {
          uint32_t v[32];
          ptx::tmem_ld_32x32b_x32(tDQ + lb + hq * 32, v);
          ptx::tmem_ld_wait();
          if (hq == 1) {
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(dq_free);
          }
#pragma unroll
          for (int e = 0; e < 32; ++e) atomicAdd(dst + static_cast<size_t>(hq * 32 + e) * dt + lane, __uint_as_float(v[e]));
        }
      }
    }
  } else if (wg == 1 || wg == 2) {
    ptx::setmaxnreg_inc<192>();
    const int quarter = warp & 3;
    const int half = wg - 1;            // which 32 query columns of the 64-row tile
    const int r = quarter * 32 + lane;  // TMEM lane: kv row (S^T, dP^T, dK, dV)
    const uint32_t lb = static_cast<uint32_t>(quarter * 32) << 16;
    int gt = 0, t = 0;
    for (int kidx = snake(0); kidx < n_items; kidx = snake(t + 1), ++t) {
    const Item it = item(kidx);
    const int kv0 = it.kv0, row0 = it.row0, h = it.h;
    for (int j = 0; j < it.n_it; ++j) {
      const int g = gt + j, bb = g & 1, sq = g % QST;
      const int q0 = (it.qt_first + j) * 64;
      WAIT(&s_full[bb], (g >> 1) & 1, 46);
      WAIT(&qdo_full[sq], (g / QST) & 1, 49);  // LSE / D rows of this tile (already complete)
      ptx::tc_fence_after();
      const int qc = half * 32;
      uint32_t sv[32], dv[32];
      ptx::tmem_ld_32x32b_x32(tS + lb + bb * 64 + qc, sv);
      ptx::tmem_ld_32x32b_x32(tdP + lb + qc, dv);
      ptx::tmem_ld_wait();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&st_free[bb]);  // S^T / dP^T of this tile consumed
      const float4* L4 = reinterpret_cast<const float4*>(sL + sq * 64 + qc);
      const float4* D4 = reinterpret_cast<const float4*>(sD + sq * 64 + qc);
      uint32_t pk[16], dk[16];
#pragma unroll
      for (int e4 = 0; e4 < 8; ++e4) {
        const float4 l4 = L4[e4], d4 = D4[e4];
        const float lv[4] = {l4.x, l4.y, l4.z, l4.w}, dvv[4] = {d4.x, d4.y, d4.z, d4.w};
        float pp[4], ds[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          pp[k] = ex2(fmaf(__uint_as_float(sv[4 * e4 + k]), scale_log2, -lv[k]));
          ds[k] = pp[k] * (__uint_as_float(dv[4 * e4 + k]) - dvv[k]);
        }
        pk[2 * e4] = ptx::pack_bf16(pp[0], pp[1]);
        pk[2 * e4 + 1] = ptx::pack_bf16(pp[2], pp[3]);
        dk[2 * e4] = ptx::pack_bf16(ds[0], ds[1]);
        dk[2 * e4 + 1] = ptx::pack_bf16(ds[2], ds[3]);
      }
      if (q0 + qc < kv0 + r) {  // near the diagonal: queries before this kv row see nothing
#pragma unroll
        for (int e = 0; e < 32; ++e)
          if (q0 + qc + e < kv0 + r) {
            pk[e / 2] &= (e & 1) ? 0x0000FFFFu : 0xFFFF0000u;
            dk[e / 2] &= (e & 1) ? 0x0000FFFFu : 0xFFFF0000u;
          }
      }
      WAIT(&pds_free[bb], ((g >> 1) & 1) ^ 1, 47);  // stage 2 of tile j-2 is done with buffer bb
      uint8_t* prow = sPT + bb * Cfg::kPBytes + r * 128;
      uint8_t* drow = sdST + bb * Cfg::kPBytes + r * 128;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int off = ((half * 4 + u) ^ (r & 7)) * 16;
        *reinterpret_cast<uint4*>(prow + off) = make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
        *reinterpret_cast<uint4*>(drow + off) = make_uint4(dk[4 * u], dk[4 * u + 1], dk[4 * u + 2], dk[4 * u + 3]);
      }
      ptx::fence_proxy_async();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&pds_full[bb]);
    }
    // dK (scaled) and dV rows of this KV block
    WAIT(kdv_full, t & 1, 48);
    ptx::tc_fence_after();
    __nv_bfloat16* krow = dqkv + static_cast<size_t>(row0 + kv0 + r) * 3 * dt + dt + h * HD;
    __nv_bfloat16* vrow = krow + dt;
    constexpr int NCH = HD / 32;
#pragma unroll 1
    for (int c = half * (NCH / 2); c < (half + 1) * (NCH / 2); ++c) {
      uint32_t kv[32], vv[32];
      ptx::tmem_ld_32x32b_x32(tdK + lb + c * 32, kv);
      ptx::tmem_ld_32x32b_x32(tdV + lb + c * 32, vv);
      ptx::tmem_ld_wait();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 a, bb2;
        a.x = ptx::pack_bf16(__uint_as_float(kv[8 * q]) * scale, __uint_as_float(kv[8 * q + 1]) * scale);
        a.y = ptx::pack_bf16(__uint_as_float(kv[8 * q + 2]) * scale, __uint_as_float(kv[8 * q + 3]) * scale);
        a.z = ptx::pack_bf16(__uint_as_float(kv[8 * q + 4]) * scale, __uint_as_float(kv[8 * q + 5]) * scale);
        a.w = ptx::pack_bf16(__uint_as_float(kv[8 * q + 6]) * scale, __uint_as_float(kv[8 * q + 7]) * scale);
        bb2.x = ptx::pack_bf16(__uint_as_float(vv[8 * q]), __uint_as_float(vv[8 * q + 1]));
        bb2.y = ptx::pack_bf16(__uint_as_float(vv[8 * q + 2]), __uint_as_float(vv[8 * q + 3]));
        bb2.z = ptx::pack_bf16(__uint_as_float(vv[8 * q + 4]), __uint_as_float(vv[8 * q + 5]));
        bb2.w = ptx::pack_bf16(__uint_as_float(vv[8 * q + 6]), __uint_as_float(vv[8 * q + 7]));
        reinterpret_cast<uint4*>(krow + c * 32)[q] = a;
        reinterpret_cast<uint4*>(vrow + c * 32)[q] = bb2;
      }
      if (dbqkv) {  // qkv bias gradient, k and v parts: this warp's 32 kv rows of columns c*32..+31
        float x[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) x[e] = __uint_as_float(kv[e]) * scale;
        atomicAdd(dbqkv + dt + h * HD + c * 32 + lane, warp_colsum32(x, lane));
#pragma unroll
        for (int e = 0; e < 32; ++e) x[e] = __uint_as_float(vv[e]);
        atomicAdd(dbqkv + 2 * dt + h * HD + c * 32 + lane, warp_colsum32(x, lane));
      }
    }
    ptx::tc_fence_before();
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(kdv_free);  // dK / dV TMEM reusable by the next item
    gt += it.n_it;
    }
  }
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

// K6 for head dim 160 (the 1T shape) on tcgen05. At 64-query tiles TMEM cannot hold S^T, dP^T
// and dQ^T next to the 2 x 160 accumulator columns of dV and dK, so the query tile is 32 rows and
// every transient buffer is double-buffered:
//   dV (0..159) | S^T x2 | dQ^T hd 0-127 || dK (256..415) | dP^T x2 | dQ^T hd 128-159
// = 512 columns. dQ^T = K^T dS^T has M = 160 rows: two M = 128 MMAs, the second over head dims
// 128..255 of the K tile — rows 160..255 read the next 96 columns of shared memory (the rest of
// the K tile's third swizzle chunk, then the V tile: finite data) and are never loaded from TMEM.
// P^T / dS^T tiles are [128 kv][32 q] with 64-byte rows (SWIZZLE_64B), so one buffer serves as the
// K-major A operand of dV / dK and as the MN-major B operand of dQ^T.
// Warps: WG0 = TMA producer (warp 0) + MMA issuer (warp 1); WG1 / WG2 = P/dS compute of the even /
// odd query tiles (each owns one S^T/dP^T TMEM pair and one P^T/dS^T smem pair); WG3 = dQ flush
// (coalesced fp32 reductions, one per 32 head dims and query). Per tile j the MMA warp issues
// stage 1 (S^T_j, dP^T_j) and then stage 2 of tile j-1 (dV, dK, dQ^T), so the exp / dS math of one
// tile overlaps the tensor core on the other.
template <int HD>
struct TcBwd3Cfg {
  static constexpr int NC = (HD + 63) / 64;        // 64-column SW128 chunks of a head (3)
  static constexpr int QT = 32;                     // query rows per tile
  static constexpr int kTileBytes = 128 * 128;      // [128 rows][64] bf16 chunk
  static constexpr int kKVBytes = NC * kTileBytes;  // [128 kv][NC x 64]
  static constexpr int kQChunk = QT * 128;          // [32 q][64]
  static constexpr int kQBytes = NC * kQChunk;
  static constexpr int kPBytes = 128 * QT * 2;      // [128 kv][32 q], 64-byte rows
  static constexpr int QST = 3;                     // Q / dO / LSE / D ring depth
  static constexpr int kSmem = 2 * kKVBytes + 2 * QST * kQBytes + 4 * kPBytes + QST * 2 * QT * 4 + 1024 + 256;
  static_assert(HD > 128 && HD <= 160 && HD % 32 == 0, "two M = 128 dQ^T MMAs cover head dims 0..255; TMEM map");
  static_assert(kSmem <= 232448, "smem over the 227 KB opt-in limit");
};

template <int HD>
__global__ void __launch_bounds__(512, 1)
    fa_bwd_tc3_kernel(const __grid_constant__ CUtensorMap tm_kv, const __grid_constant__ CUtensorMap tm_q,
                      const __grid_constant__ CUtensorMap tm_do, const float* __restrict__ lse,
                      const float* __restrict__ Dg, float* __restrict__ dq_acc, __nv_bfloat16* __restrict__ dqkv,
                      int s, int ht, float scale_log2, float scale) {
  using Cfg = TcBwd3Cfg<HD>;
  constexpr int NC = Cfg::NC, TB = Cfg::kTileBytes, QT = Cfg::QT, QST = Cfg::QST;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = ptx::smem_align1024(smem_raw);
  uint8_t* sK = smem;
  uint8_t* sV = sK + Cfg::kKVBytes;  // directly after K: the second dQ^T MMA reads past the K tile
  uint8_t* sQ = sV + Cfg::kKVBytes;         // [QST][NC][32][64]
  uint8_t* sdO = sQ + QST * Cfg::kQBytes;   // [QST][NC][32][64]
  uint8_t* sPT = sdO + QST * Cfg::kQBytes;  // [2][128 kv][32 q]
  uint8_t* sdST = sPT + 2 * Cfg::kPBytes;   // [2][128 kv][32 q]
  float* sL = reinterpret_cast<float*>(sdST + 2 * Cfg::kPBytes);  // [QST][32]
  float* sD = sL + QST * QT;                                      // [QST][32]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sD + QST * QT);
  uint64_t* kv_full = bars;
  uint64_t* qdo_full = bars + 1;         // [QST]
  uint64_t* qdo_empty = qdo_full + QST;  // [QST]
  uint64_t* s_full = qdo_empty + QST;    // [2] S^T / dP^T of buffer b computed
  uint64_t* st_free = s_full + 2;        // [2] ... and read out by its compute warpgroup
  uint64_t* pds_full = st_free + 2;      // [2] P^T / dS^T of buffer b written to smem
  uint64_t* pds_free = pds_full + 2;     // [2] ... and consumed by stage 2
  uint64_t* dq_full = pds_free + 2;
  uint64_t* dq_free = dq_full + 1;
  uint64_t* kdv_full = dq_free + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(kdv_full + 1);

  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x / 32), 0), lane = threadIdx.x % 32;
  const int kvb = blockIdx.x;
  const int b = blockIdx.y / ht, h = blockIdx.y % ht;
  const int dt = ht * HD;
  const int row0 = b * s;
  const int kv0 = kvb * 128;
  const int qt_first = kv0 / QT;  // query tiles at and after the diagonal
  const int n_it = s / QT - qt_first;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tm_kv);
    ptx::tma_prefetch_desc(&tm_q);
    ptx::tma_prefetch_desc(&tm_do);
    ptx::mbar_init(kv_full, 1);
    for (int i = 0; i < QST; ++i) {
      ptx::mbar_init(&qdo_full[i], 1);
      ptx::mbar_init(&qdo_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&s_full[i], 1);
      ptx::mbar_init(&st_free[i], 4);
      ptx::mbar_init(&pds_full[i], 4);
      ptx::mbar_init(&pds_free[i], 1);
    }
    ptx::mbar_init(dq_full, 1);
    ptx::mbar_init(dq_free, 4);
    ptx::mbar_init(kdv_full, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  pdl_trigger();
  pdl_wait();
  // accumulators on 256-column boundaries, the 32-column transients in the gaps
  const uint32_t tdV = tmem, tdK = tmem + 256, tS = tmem + HD, tDQa = tmem + HD + 2 * QT, tdP = tmem + 256 + HD,
                 tDQb = tmem + 256 + HD + 2 * QT;
  const int wg = warp / 4;

  if (warp == 0) {
    if (lane == 0) {
      const float* gLq = lse + (static_cast<size_t>(b) * ht + h) * s;
      const float* gDq = Dg + (static_cast<size_t>(b) * ht + h) * s;
      ptx::mbar_arrive_expect_tx(kv_full, 2 * Cfg::kKVBytes);
      for (int c = 0; c < NC; ++c) {
        ptx::tma_load_2d(sK + c * TB, &tm_kv, kv_full, dt + h * HD + 64 * c, row0 + kv0);
        ptx::tma_load_2d(sV + c * TB, &tm_kv, kv_full, 2 * dt + h * HD + 64 * c, row0 + kv0);
      }
      for (int j = 0; j < n_it; ++j) {
        const int sq = j % QST;
        const int q0 = (qt_first + j) * QT;
        WAIT(&qdo_empty[sq], ((j / QST) & 1) ^ 1, 60);
        ptx::mbar_arrive_expect_tx(&qdo_full[sq], 2 * Cfg::kQBytes + 2 * QT * 4);
        for (int c = 0; c < NC; ++c) {
          ptx::tma_load_2d(sQ + sq * Cfg::kQBytes + c * Cfg::kQChunk, &tm_q, &qdo_full[sq], h * HD + 64 * c, row0 + q0);
          ptx::tma_load_2d(sdO + sq * Cfg::kQBytes + c * Cfg::kQChunk, &tm_do, &qdo_full[sq], h * HD + 64 * c,
                           row0 + q0);
        }
        ptx::bulk_load(sL + sq * QT, gLq + q0, QT * 4, &qdo_full[sq]);
        ptx::bulk_load(sD + sq * QT, gDq + q0, QT * 4, &qdo_full[sq]);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t id_s = ptx::idesc_bf16_f32(128, QT, false, false);   // S^T, dP^T
    constexpr uint32_t id_acc = ptx::idesc_bf16_f32(128, HD, false, true);  // dV, dK
    constexpr uint32_t id_dq = ptx::idesc_bf16_f32(128, QT, true, true);    // dQ^T halves
    const uint32_t u0 = (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) + 1023u) & ~1023u;
    const uint32_t aK = u0, aV = u0 + Cfg::kKVBytes;
    const uint32_t aQ0 = u0 + 2 * Cfg::kKVBytes, adO0 = aQ0 + QST * Cfg::kQBytes;
    const uint32_t aP0 = adO0 + QST * Cfg::kQBytes, adS0 = aP0 + 2 * Cfg::kPBytes;
    WAIT(kv_full, 0, 61);
    auto stage2 = [&](int i) {
      const int bb = i & 1, sq = i % QST;
      WAIT(&pds_full[bb], (i >> 1) & 1, 62);
      ptx::tc_fence_after();
      const uint32_t aQ = aQ0 + sq * Cfg::kQBytes, adO = adO0 + sq * Cfg::kQBytes;
      const uint32_t aP = aP0 + bb * Cfg::kPBytes, adS = adS0 + bb * Cfg::kPBytes;
#pragma unroll
      for (int kk = 0; kk < QT / 16; ++kk) {  // K = 32 query rows
        const uint32_t acc = (i > 0 || kk > 0) ? 1u : 0u;
        ptx::mma_bf16_ss_w(tdV, ptx::smem_desc_sw64(aP + kk * 32, 16, 512),
                           ptx::smem_desc_sw128(adO + kk * 2048, Cfg::kQChunk, 1024), id_acc, acc);
        ptx::mma_bf16_ss_w(tdK, ptx::smem_desc_sw64(adS + kk * 32, 16, 512),
                           ptx::smem_desc_sw128(aQ + kk * 2048, Cfg::kQChunk, 1024), id_acc, acc);
      }
      if (i > 0) WAIT(dq_free, (i - 1) & 1, 63);  // dQ^T_{i-1} read out of TMEM
      ptx::tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {  // K = 128 kv rows
        const uint64_t bdesc = ptx::smem_desc_sw64(adS + kk * 1024, 512, 512);
        ptx::mma_bf16_ss_w(tDQa, ptx::smem_desc_sw128(aK + kk * 2048, TB, 1024), bdesc, id_dq, kk > 0 ? 1u : 0u);
        ptx::mma_bf16_ss_w(tDQb, ptx::smem_desc_sw128(aK + 2 * TB + kk * 2048, TB, 1024), bdesc, id_dq,
                           kk > 0 ? 1u : 0u);
      }
      ptx::mma_commit_w(dq_full);
      ptx::mma_commit_w(&qdo_empty[sq]);
      ptx::mma_commit_w(&pds_free[bb]);
    };
    for (int j = 0; j < n_it; ++j) {
      const int bb = j & 1, sq = j % QST;
      WAIT(&qdo_full[sq], (j / QST) & 1, 64);
      if (j >= 2) WAIT(&st_free[bb], ((j - 2) >> 1) & 1, 65);  // tile j-2 read buffer bb out
      ptx::tc_fence_after();
      const uint32_t aQ = aQ0 + sq * Cfg::kQBytes, adO = adO0 + sq * Cfg::kQBytes;
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        const uint32_t ak = (kk / 4) * TB + (kk % 4) * 32, aq = (kk / 4) * Cfg::kQChunk + (kk % 4) * 32;
        ptx::mma_bf16_ss_w(tS + bb * QT, ptx::smem_desc_sw128(aK + ak, 16, 1024),
                           ptx::smem_desc_sw128(aQ + aq, 16, 1024), id_s, kk > 0 ? 1u : 0u);
        ptx::mma_bf16_ss_w(tdP + bb * QT, ptx::smem_desc_sw128(aV + ak, 16, 1024),
                           ptx::smem_desc_sw128(adO + aq, 16, 1024), id_s, kk > 0 ? 1u : 0u);
      }
      ptx::mma_commit_w(&s_full[bb]);
      if (j > 0) stage2(j - 1);
    }
    stage2(n_it - 1);
    ptx::mma_commit_w(kdv_full);
  } else if (wg == 3) {
    // dQ^T (lane = head dim, column = query) -> fp32 reductions into dq_acc (one coalesced
    // 128-byte request per query and 32 head dims); head dims 128..159 by the quarter-0 warp.
    const int quarter = warp & 3;
    const uint32_t lb = static_cast<uint32_t>(quarter * 32) << 16;
    for (int i = 0; i < n_it; ++i) {
      const int q0 = (qt_first + i) * QT;
      float* dst = dq_acc + static_cast<size_t>(row0 + q0) * dt + h * HD + quarter * 32;
      WAIT(dq_full, i & 1, 66);
      ptx::tc_fence_after();
      uint32_t va[32], vb[32];
      ptx::tmem_ld_32x32b_x32(tDQa + lb, va);
      if (quarter == 0) ptx::tmem_ld_32x32b_x32(tDQb, vb);
      ptx::tmem_ld_wait();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(dq_free);
#pragma unroll
      for (int e = 0; e < QT; ++e) atomicAdd(dst + static_cast<size_t>(e) * dt + lane, __uint_as_float(va[e]));
      if (quarter == 0) {
#pragma unroll
        for (int e = 0; e < QT; ++e) atomicAdd(dst + static_cast<size_t>(e) * dt + 128 + lane, __uint_as_float(vb[e]));
      }
    }

  } else if (wg == 1 || wg == 2) {  // P^T, dS^T of the even / odd query tiles (warps 2-3 idle)
    const int bb = wg - 1;
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;  // TMEM lane = kv row of this KV block
    const uint32_t lb = static_cast<uint32_t>(quarter * 32) << 16;
    const int sw = (r >> 1) & 3;        // SWIZZLE_64B: 16-byte unit u of row r sits at u ^ ((r >> 1) & 3)
    for (int j = bb; j < n_it; j += 2) {
      const int sq = j % QST;
      const int q0 = (qt_first + j) * QT;
      WAIT(&s_full[bb], (j >> 1) & 1, 67);
      WAIT(&qdo_full[sq], (j / QST) & 1, 68);  // LSE / D rows of this tile
      ptx::tc_fence_after();
      uint32_t sv[32], dv[32];
      ptx::tmem_ld_32x32b_x32(tS + lb + bb * QT, sv);
      ptx::tmem_ld_32x32b_x32(tdP + lb + bb * QT, dv);
      ptx::tmem_ld_wait();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&st_free[bb]);
      const float4* L4 = reinterpret_cast<const float4*>(sL + sq * QT);
      const float4* D4 = reinterpret_cast<const float4*>(sD + sq * QT);
      uint32_t pk[16], dk[16];
#pragma unroll
      for (int e4 = 0; e4 < 8; ++e4) {
        const float4 l4 = L4[e4], d4 = D4[e4];
        const float lv[4] = {l4.x, l4.y, l4.z, l4.w}, dvv[4] = {d4.x, d4.y, d4.z, d4.w};
        float pp[4], ds[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          pp[k] = ex2(fmaf(__uint_as_float(sv[4 * e4 + k]), scale_log2, -lv[k]));
          ds[k] = pp[k] * (__uint_as_float(dv[4 * e4 + k]) - dvv[k]);
        }
        pk[2 * e4] = ptx::pack_bf16(pp[0], pp[1]);
        pk[2 * e4 + 1] = ptx::pack_bf16(pp[2], pp[3]);
        dk[2 * e4] = ptx::pack_bf16(ds[0], ds[1]);
        dk[2 * e4 + 1] = ptx::pack_bf16(ds[2], ds[3]);
      }
      if (q0 < kv0 + r) {  // near the diagonal: queries before this kv row see nothing
#pragma unroll
        for (int e = 0; e < QT; ++e)
          if (q0 + e < kv0 + r) {
            pk[e / 2] &= (e & 1) ? 0x0000FFFFu : 0xFFFF0000u;
            dk[e / 2] &= (e & 1) ? 0x0000FFFFu : 0xFFFF0000u;
          }
      }
      WAIT(&pds_free[bb], ((j >> 1) & 1) ^ 1, 69);  // stage 2 of tile j-2 done with this buffer
      uint8_t* prow = sPT + bb * Cfg::kPBytes + r * 64;
      uint8_t* drow = sdST + bb * Cfg::kPBytes + r * 64;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int off = (u ^ sw) * 16;
        *reinterpret_cast<uint4*>(prow + off) = make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
        *reinterpret_cast<uint4*>(drow + off) = make_uint4(dk[4 * u], dk[4 * u + 1], dk[4 * u + 2], dk[4 * u + 3]);
      }
      ptx::fence_proxy_async();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&pds_full[bb]);
    }
    // dK (scaled) and dV rows of this KV block: WG1 columns [0, 96), WG2 [96, 160)
    WAIT(kdv_full, 0, 70);
    ptx::tc_fence_after();
    __nv_bfloat16* krow = dqkv + static_cast<size_t>(row0 + kv0 + r) * 3 * dt + dt + h * HD;
    __nv_bfloat16* vrow = krow + dt;
    constexpr int NCH = HD / 32, SPLIT = (NCH + 1) / 2;
#pragma unroll 1
    for (int c = bb == 0 ? 0 : SPLIT; c < (bb == 0 ? SPLIT : NCH); ++c) {
      uint32_t kv[32], vv[32];
      ptx::tmem_ld_32x32b_x32(tdK + lb + c * 32, kv);
      ptx::tmem_ld_32x32b_x32(tdV + lb + c * 32, vv);
      ptx::tmem_ld_wait();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 a, bb2;
        a.x = ptx::pack_bf16(__uint_as_float(kv[8 * q]) * scale, __uint_as_float(kv[8 * q + 1]) * scale);
        a.y = ptx::pack_bf16(__uint_as_float(kv[8 * q + 2]) * scale, __uint_as_float(kv[8 * q + 3]) * scale);
        a.z = ptx::pack_bf16(__uint_as_float(kv[8 * q + 4]) * scale, __uint_as_float(kv[8 * q + 5]) * scale);
        a.w = ptx::pack_bf16(__uint_as_float(kv[8 * q + 6]) * scale, __uint_as_float(kv[8 * q + 7]) * scale);
        bb2.x = ptx::pack_bf16(__uint_as_float(vv[8 * q]), __uint_as_float(vv[8 * q + 1]));
        bb2.y = ptx::pack_bf16(__uint_as_float(vv[8 * q + 2]), __uint_as_float(vv[8 * q + 3]));
        bb2.z = ptx::pack_bf16(__uint_as_float(vv[8 * q + 4]), __uint_as_float(vv[8 * q + 5]));
        bb2.w = ptx::pack_bf16(__uint_as_float(vv[8 * q + 6]), __uint_as_float(vv[8 * q + 7]));
        reinterpret_cast<uint4*>(krow + c * 32)[q] = a;
        reinterpret_cast<uint4*>(vrow + c * 32)[q] = bb2;
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

template <int HD>
int bwd_tc3(const AttnShape& a, const __nv_bfloat16* qkv, const __nv_bfloat16* dout, const float* lse, const float* D,
            float* dq_acc, __nv_bfloat16* dqkv, cudaStream_t st) {
  using Cfg = TcBwd3Cfg<HD>;
  if (ensure_dynamic_smem(reinterpret_cast<const void*>(fa_bwd_tc3_kernel<HD>), Cfg::kSmem) != 0) return 3;
  count_variant(KV_ATTN_BWD_HD160);
  const int dt = a.heads * HD;
  const uint64_t M = static_cast<uint64_t>(a.batch) * a.seq;
  CUtensorMap tkv, tq, tdo;
  if (!make_tmap_bf16(&tkv, qkv, 3 * static_cast<uint64_t>(dt), M, 3 * dt, 64, 128)) return 3;
  if (!make_tmap_bf16(&tq, qkv, 3 * static_cast<uint64_t>(dt), M, 3 * dt, 64, Cfg::QT)) return 3;
  if (!make_tmap_bf16(&tdo, dout, static_cast<uint64_t>(dt), M, dt, 64, Cfg::QT)) return 3;
  dim3 grid(a.seq / 128, a.batch * a.heads);
  const float scale = 1.f / sqrtf(static_cast<float>(HD));
  const cudaError_t e = launch_pdl(fa_bwd_tc3_kernel<HD>, grid, dim3(512), Cfg::kSmem, st, tkv, tq, tdo, lse, D,
                                   dq_acc, dqkv, a.seq, a.heads, scale * kLog2e, scale);
  if (e != cudaSuccess) std::fprintf(stderr, "fa_bwd_tc3 launch: %s\n", cudaGetErrorString(e));
  return e == cudaSuccess && cudaGetLastError() == cudaSuccess ? 0 : 3;
}

// Backward preprocessing when D was not produced by the W_o dgrad epilogue: D[b,h,q] =
// sum_c dO[q,c] * O[q,c] (one warp per (row, head)) and the fp32 dQ accumulator zeroed.
template <int HD>
__global__ void attn_bwd_pre_kernel(const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dout,
                                    float* __restrict__ D, float* __restrict__ dq_acc, int s, int ht, int M) {
  const int wg = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  const int dt = ht * HD;
  if (wg >= M * ht) return;
  const int row = wg / ht, h = wg % ht;
  const __nv_bfloat16* op = o + static_cast<size_t>(row) * dt + h * HD;
  const __nv_bfloat16* dp = dout + static_cast<size_t>(row) * dt + h * HD;
  float acc = 0.f;
  for (int c = lane * 2; c < HD; c += 64) {
    const float2 x = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(op + c));
    const float2 y = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(dp + c));
    acc = fmaf(x.x, y.x, fmaf(x.y, y.y, acc));
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) D[(static_cast<size_t>(row / s) * ht + h) * s + row % s] = acc;
  float* dqa = dq_acc + static_cast<size_t>(row) * dt + h * HD;
  for (int c = lane; c < HD; c += 32) dqa[c] = 0.f;
}

// dQ = scale * dq_acc (fp32) -> bf16 into the q section of dqkv.
__global__ void attn_dq_convert_kernel(const float* __restrict__ dq_acc, __nv_bfloat16* __restrict__ dqkv, int M,
                                       int dt, float scale) {
  const size_t n = static_cast<size_t>(M) * dt / 4;
  const int ldq = 3 * dt;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t e = i * 4, row = e / dt, col = e % dt;
    const float4 v = reinterpret_cast<const float4*>(dq_acc)[i];
    uint2 pk;
    pk.x = ptx::pack_bf16(v.x * scale, v.y * scale);
    pk.y = ptx::pack_bf16(v.z * scale, v.w * scale);
    *reinterpret_cast<uint2*>(dqkv + row * ldq + col) = pk;
  }
}

// dQ = scale * dq_acc -> bf16 (as attn_dq_convert_kernel) plus the q part of the qkv bias gradient:
// a block covers 64 rows x 128 columns (8 warps x 8 rows, a lane 4 columns) and adds its column sums
// into dbq with one fp32 reduction per column.
__global__ void __launch_bounds__(256) attn_dq_convert_colsum_kernel(const float* __restrict__ dq_acc,
                                                                     __nv_bfloat16* __restrict__ dqkv, int dt,
                                                                     float scale, float* __restrict__ dbq) {
  __shared__ float4 part[8][32];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int col = blockIdx.x * 128 + lane * 4;
  const size_t r0 = static_cast<size_t>(blockIdx.y) * 64 + warp * 8;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const size_t row = r0 + i;
    float4 v = reinterpret_cast<const float4*>(dq_acc + row * dt + col)[0];
    v.x *= scale, v.y *= scale, v.z *= scale, v.w *= scale;
    acc.x += v.x, acc.y += v.y, acc.z += v.z, acc.w += v.w;
    uint2 pk;
    pk.x = ptx::pack_bf16(v.x, v.y);
    pk.y = ptx::pack_bf16(v.z, v.w);
    *reinterpret_cast<uint2*>(dqkv + row * 3 * dt + col) = pk;
  }
  part[warp][lane] = acc;
  __syncthreads();
  if (warp == 0) {
    float4 t = part[0][lane];
#pragma unroll
    for (int w = 1; w < 8; ++w) {
      const float4 u = part[w][lane];
      t.x += u.x, t.y += u.y, t.z += u.z, t.w += u.w;
    }
    atomicAdd(dbq + col, t.x);
    atomicAdd(dbq + col + 1, t.y);
    atomicAdd(dbq + col + 2, t.z);
    atomicAdd(dbq + col + 3, t.w);
  }
}

template <int HD>
int bwd_tc2(const AttnShape& a, const __nv_bfloat16* qkv, const __nv_bfloat16* dout, const float* lse, const float* D,
            float* dq_acc, __nv_bfloat16* dqkv, float* dbqkv, cudaStream_t st) {
  using Cfg = TcBwd2Cfg<HD>;
  static const bool tp = std::getenv("GPTB200_ATTN_BWD_SMEM_P") == nullptr;  // A/B: P^T/dS^T in smem
  const auto kern = tp ? fa_bwd_tc2_kernel<HD, true> : fa_bwd_tc2_kernel<HD, false>;
  if (ensure_dynamic_smem(reinterpret_cast<const void*>(kern), Cfg::kSmem) != 0) return 3;
  count_variant(KV_ATTN_BWD_PER_BLOCK);
  const int dt = a.heads * HD;
  const uint64_t M = static_cast<uint64_t>(a.batch) * a.seq;
  CUtensorMap tkv, tq, tdo;
  if (!make_tmap_bf16(&tkv, qkv, 3 * static_cast<uint64_t>(dt), M, 3 * dt, 64, 128)) return 3;
  if (!make_tmap_bf16(&tq, qkv, 3 * static_cast<uint64_t>(dt), M, 3 * dt, 64, 64)) return 3;
  if (!make_tmap_bf16(&tdo, dout, static_cast<uint64_t>(dt), M, dt, 64, 64)) return 3;
  dim3 grid(a.seq / 128, a.batch * a.heads);
  const float scale = 1.f / sqrtf(static_cast<float>(HD));
#ifdef GPTB200_ATTN_TRACE
  unsigned long long* tbuf = nullptr;
  const char* tpath = std::getenv("GPTB200_ATTN_TRACE");
  if (tpath) {
    cudaMalloc(&tbuf, kTraceTiles * kTraceEv * 8);
    cudaMemset(tbuf, 0, kTraceTiles * kTraceEv * 8);
    cudaMemcpyToSymbol(g_attn_trace, &tbuf, sizeof(tbuf));
  }
#endif
  launch_pdl(kern, grid, dim3(512), Cfg::kSmem, st, tkv, tq, tdo, lse, D, dq_acc, dqkv, dbqkv, a.seq,
             a.heads, scale * kLog2e, scale);
#ifdef GPTB200_ATTN_TRACE
  if (tbuf) {
    cudaStreamSynchronize(st);
    std::vector<unsigned long long> h(kTraceTiles * kTraceEv);
    cudaMemcpy(h.data(), tbuf, h.size() * 8, cudaMemcpyDeviceToHost);
    if (FILE* f = std::fopen(tpath, "w")) {
      for (int t = 0; t < kTraceTiles; ++t) {
        for (int e = 0; e < kTraceEv; ++e) std::fprintf(f, "%llu%c", h[t * kTraceEv + e], e + 1 < kTraceEv ? ',' : '\n');
      }
      std::fclose(f);
    }
    unsigned long long* null = nullptr;
    cudaMemcpyToSymbol(g_attn_trace, &null, sizeof(null));
    cudaFree(tbuf);
  }
#endif
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

template <int HD>
int bwd_tc2_persistent(const AttnShape& a, const __nv_bfloat16* qkv, const __nv_bfloat16* dout, const float* lse,
                       const float* D, float* dq_acc, __nv_bfloat16* dqkv, float* dbqkv, cudaStream_t st) {
  using Cfg = TcBwd2Cfg<HD>;
  if (ensure_dynamic_smem(reinterpret_cast<const void*>(fa_bwd_tc2_persistent<HD>), Cfg::kSmem) != 0) return 3;
  count_variant(KV_ATTN_BWD_PERSISTENT);
  const int dt = a.heads * HD;
  const uint64_t M = static_cast<uint64_t>(a.batch) * a.seq;
  CUtensorMap tkv, tq, tdo;
  if (!make_tmap_bf16(&tkv, qkv, 3 * static_cast<uint64_t>(dt), M, 3 * dt, 64, 128)) return 3;
  if (!make_tmap_bf16(&tq, qkv, 3 * static_cast<uint64_t>(dt), M, 3 * dt, 64, 64)) return 3;
  if (!make_tmap_bf16(&tdo, dout, static_cast<uint64_t>(dt), M, dt, 64, 64)) return 3;
  const int items = (a.seq / 128) * a.batch * a.heads;
  const int grid = items < device_sm_count() ? items : device_sm_count();
  const float scale = 1.f / sqrtf(static_cast<float>(HD));
  launch_pdl(fa_bwd_tc2_persistent<HD>, dim3(grid), dim3(512), Cfg::kSmem, st, tkv, tq, tdo, lse, D, dq_acc, dqkv,
             dbqkv, a.seq, a.heads, a.batch, scale * kLog2e, scale);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

template <int HD>
int bwd_tc(const AttnShape& a, const __nv_bfloat16* qkv, const __nv_bfloat16* dout, const float* lse, const float* D,
           float* dq_acc, __nv_bfloat16* dqkv, cudaStream_t st) {
  using Cfg = TcBwdCfg<HD>;
  if (ensure_dynamic_smem(reinterpret_cast<const void*>(fa_bwd_tc_kernel<HD>), Cfg::kSmem) != 0) return 3;
  count_variant(KV_ATTN_BWD_HD64);
  const int dt = a.heads * HD;
  const uint64_t M = static_cast<uint64_t>(a.batch) * a.seq;
  CUtensorMap tq, tdo;
  if (!make_tmap_bf16(&tq, qkv, 3 * static_cast<uint64_t>(dt), M, 3 * dt, 64, 128)) return 3;
  if (!make_tmap_bf16(&tdo, dout, static_cast<uint64_t>(dt), M, dt, 64, 128)) return 3;
  dim3 grid(a.seq / 128, a.batch * a.heads);
  const float scale = 1.f / sqrtf(static_cast<float>(HD));
  fa_bwd_tc_kernel<HD><<<grid, 320, Cfg::kSmem, st>>>(tq, tdo, lse, D, dq_acc, dqkv, a.seq, a.heads, scale * kLog2e,
                                                       scale);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

template <int HD>
int fwd_tc_persistent(const AttnShape& a, const __nv_bfloat16* qkv, __nv_bfloat16* out, float* lse, cudaStream_t st) {
  using Cfg = TcFwdCfg<HD>;
  if (ensure_dynamic_smem(reinterpret_cast<const void*>(fa_fwd_tc_persistent<HD>), Cfg::kSmem) != 0) return 3;
  count_variant(KV_ATTN_FWD_PERSISTENT);
  const int dt = a.heads * HD;
  CUtensorMap tm;
  if (!make_tmap_bf16(&tm, qkv, 3 * static_cast<uint64_t>(dt), static_cast<uint64_t>(a.batch) * a.seq, 3 * dt, 64, 128))
    return 3;
  const int items = (a.seq / kBM) * a.batch * a.heads;
  const int grid = items < device_sm_count() ? items : device_sm_count();
  launch_pdl(fa_fwd_tc_persistent<HD>, dim3(grid), dim3(Cfg::kThreads), Cfg::kSmem, st, tm, out, lse, a.seq, a.heads,
             a.batch, kLog2e / sqrtf(static_cast<float>(HD)));
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

// Debug builds (-DGPTB200_ATTN_TRACE): per-tile clock64 stamps of one CTA -> $GPTB200_ATTN_TRACE.
struct TraceDump {
#ifdef GPTB200_ATTN_TRACE
  unsigned long long* buf = nullptr;
  const char* path = std::getenv("GPTB200_ATTN_TRACE");
  TraceDump() {
    if (!path) return;
    cudaMalloc(&buf, kTraceTiles * kTraceEv * 8);
    cudaMemset(buf, 0, kTraceTiles * kTraceEv * 8);
    cudaMemcpyToSymbol(g_attn_trace, &buf, sizeof(buf));
  }
  void dump(cudaStream_t st) {
    if (!buf) return;
    cudaStreamSynchronize(st);
    std::vector<unsigned long long> h(kTraceTiles * kTraceEv);
    cudaMemcpy(h.data(), buf, h.size() * 8, cudaMemcpyDeviceToHost);
    if (FILE* f = std::fopen(path, "w")) {
      for (int t = 0; t < kTraceTiles; ++t)
        for (int e = 0; e < kTraceEv; ++e) std::fprintf(f, "%llu%c", h[t * kTraceEv + e], e + 1 < kTraceEv ? ',' : '\n');
      std::fclose(f);
    }
    unsigned long long* null = nullptr;
    cudaMemcpyToSymbol(g_attn_trace, &null, sizeof(null));
    cudaFree(buf);
    buf = nullptr;
  }
#else
  void dump(cudaStream_t) {}
#endif
};

template <int HD, int CS>
int fwd_tc2q_cs(const AttnShape& a, const __nv_bfloat16* qkv, __nv_bfloat16* out, float* lse, cudaStream_t st, int emu) {
  using Cfg = TcFwd2Cfg<HD, CS>;
  // EMU 2 (2 of every 8 exponent pairs on the FMA pipe) is the measured best of 0..4; 0 (all on the
  // MUFU) stays instantiated as the A/B reference
  const auto kern = emu == 0 ? fa_fwd2_kernel<HD, 0, CS> : fa_fwd2_kernel<HD, 2, CS>;
  if (ensure_dynamic_smem(reinterpret_cast<const void*>(kern), Cfg::kSmem) != 0) return 3;
  count_variant(KV_ATTN_FWD_TWO_Q);
  const int dt = a.heads * HD;
  CUtensorMap tm;
  if (!make_tmap_bf16(&tm, qkv, 3 * static_cast<uint64_t>(dt), static_cast<uint64_t>(a.batch) * a.seq, 3 * dt, 64, 128))
    return 3;
  dim3 grid(a.batch * a.heads, a.seq / 256);
  TraceDump trace;
  launch_pdl(kern, grid, dim3(Cfg::kThreads), Cfg::kSmem, st, tm, out, lse, a.seq, a.heads,
             kLog2e / sqrtf(static_cast<float>(HD)));
  trace.dump(st);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

template <int HD>
int fwd_tc2q(const AttnShape& a, const __nv_bfloat16* qkv, __nv_bfloat16* out, float* lse, cudaStream_t st) {
  static const int emu = [] {
    const char* e = std::getenv("GPTB200_ATTN_FWD_EMU");
    return e ? std::atoi(e) : 2;  // measured best of 0..4 (1.4B shapes: 865 / 901 TF/s; 0: 855 / 883)
  }();
  // one softmax warp per 32 rows (CS = 1): 2 warps per row measured 3 % slower (more row-max exchange
  // than gain); the CS template parameter keeps that variant available for experiments
  return fwd_tc2q_cs<HD, 1>(a, qkv, out, lse, st, emu);
}

template <int HD>
int fwd_tc(const AttnShape& a, const __nv_bfloat16* qkv, __nv_bfloat16* out, float* lse, cudaStream_t st) {
  using Cfg = TcFwdCfg<HD>;
  if (ensure_dynamic_smem(reinterpret_cast<const void*>(fa_fwd_tc_kernel<HD>), Cfg::kSmem) != 0) return 3;
  count_variant(KV_ATTN_FWD_PER_BLOCK);
  const int dt = a.heads * HD;
  CUtensorMap tm, tt;
  const uint64_t M = static_cast<uint64_t>(a.batch) * a.seq;
  if (!make_tmap_bf16(&tm, qkv, 3 * static_cast<uint64_t>(dt), M, 3 * dt, 64, 128)) return 3;
  if (Cfg::TAIL ? !make_tmap_bf16_sw64(&tt, qkv, 3 * static_cast<uint64_t>(dt), M, 3 * dt, Cfg::TAIL, 128) : (tt = tm, false))
    return 3;
  dim3 grid(a.seq / kBM, a.batch * a.heads);
  launch_pdl(fa_fwd_tc_kernel<HD>, grid, dim3(Cfg::kThreads), Cfg::kSmem, st, tm, tt, out, lse, a.seq, a.heads,
             kLog2e / sqrtf(static_cast<float>(HD)));
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

}  // namespace

int flash_attn_bwd_tc_main(const AttnShape& a, const __nv_bfloat16* qkv, const __nv_bfloat16* dout, const float* lse,
                           const float* D, float* dq_acc, __nv_bfloat16* dqkv, cudaStream_t st, float* dbqkv) {
  if (a.seq % 128 != 0) return 1;
  switch (a.head_dim) {
    case 64: return bwd_tc<64>(a, qkv, dout, lse, D, dq_acc, dqkv, st);
    case 128: {
      // persistent CTAs win when there are few (kv block, head) items per SM (the per-item K/V
      // reload and dK/dV drain are cheaper than CTA turnover); with many items the per-block grid
      // keeps more work in flight (measured: 6 heads x 4 seqs 0.132 -> 0.113 ms, 16 x 8 0.540 -> 0.607)
      static const char* forced = std::getenv("GPTB200_ATTN_BWD_PER_BLOCK");  // A/B switch: 1 / 0
      const int items = (a.seq / 128) * a.batch * a.heads;
      const bool per_block = forced ? forced[0] == '1' : items > 6 * device_sm_count();
      return per_block ? bwd_tc2<128>(a, qkv, dout, lse, D, dq_acc, dqkv, dbqkv, st)
                       : bwd_tc2_persistent<128>(a, qkv, dout, lse, D, dq_acc, dqkv, dbqkv, st);
    }
    case 160: return bwd_tc3<160>(a, qkv, dout, lse, D, dq_acc, dqkv, st);
    default: return 1;
  }
}

int flash_attn_fwd(const AttnShape& a, const __nv_bfloat16* qkv, __nv_bfloat16* out, float* lse, cudaStream_t st) {
  return flash_attn_fwd_tc(a, qkv, out, lse, st);
}

int flash_attn_bwd(const AttnShape& a, const __nv_bfloat16* qkv, const __nv_bfloat16* out, const __nv_bfloat16* dout,
                   const float* lse, float* D, float* dq_acc, __nv_bfloat16* dqkv, cudaStream_t st, bool d_ready,
                   float* dbqkv) {
  if (a.seq % 128 != 0) return 1;
  const int hd = a.head_dim;
  if (hd != 64 && hd != 128 && hd != 160) return 1;
  const int M = a.batch * a.seq, dt = a.heads * hd;
  if (d_ready && hd == 128) {
    cudaMemsetAsync(dq_acc, 0, static_cast<size_t>(M) * dt * sizeof(float), st);
  } else {
    const int warps = M * a.heads, grid = (warps + 7) / 8;
    if (hd == 64) attn_bwd_pre_kernel<64><<<grid, 256, 0, st>>>(out, dout, D, dq_acc, a.seq, a.heads, M);
    if (hd == 128) attn_bwd_pre_kernel<128><<<grid, 256, 0, st>>>(out, dout, D, dq_acc, a.seq, a.heads, M);
    if (hd == 160) attn_bwd_pre_kernel<160><<<grid, 256, 0, st>>>(out, dout, D, dq_acc, a.seq, a.heads, M);
  }
  static const bool dbg = std::getenv("GPTB200_ATTN_SYNC_DEBUG") != nullptr;  // locate a faulting launch
  if (dbg && cudaStreamSynchronize(st) != cudaSuccess) {
    std::fprintf(stderr, "attention bwd: preprocessing failed: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 3;
  }
  // qkv bias gradient folded in (hd 128): k / v column sums in the main kernel's dK / dV epilogue,
  // q column sums in the dQ conversion; other head dims leave dbqkv to the caller
  float* dbias = hd == 128 ? dbqkv : nullptr;
  const int r = flash_attn_bwd_tc_main(a, qkv, dout, lse, D, dq_acc, dqkv, st, dbias);
  if (r != 0) return r;
  if (dbg && cudaStreamSynchronize(st) != cudaSuccess) {
    std::fprintf(stderr, "attention bwd: main kernel failed: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 3;
  }
  if (dbias)
    attn_dq_convert_colsum_kernel<<<dim3(dt / 128, M / 64), 256, 0, st>>>(dq_acc, dqkv, dt,
                                                                          1.f / sqrtf(static_cast<float>(hd)), dbias);
  else
    attn_dq_convert_kernel<<<8 * device_sm_count(), 256, 0, st>>>(dq_acc, dqkv, M, dt,
                                                                  1.f / sqrtf(static_cast<float>(hd)));
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

int flash_attn_fwd_tc(const AttnShape& a, const __nv_bfloat16* qkv, __nv_bfloat16* out, float* lse, cudaStream_t st) {
  if (a.seq % kBM != 0) return 1;
  // persistent CTAs for hd <= 128. In isolation the per-block grid wins at many items (1.4B MBS 32:
  // 766 vs 670 TF/s) but inside the step it loses (530 vs 610 TF/s, same build and box class: the
  // persistent CTAs' prologue overlap matters more behind the QKV GEMM), so it stays an A/B switch.
  static const bool per_block = std::getenv("GPTB200_ATTN_FWD_PER_BLOCK") != nullptr;
  // two query tiles per CTA (fa_fwd2_kernel) when its grid of 256-row blocks fills the GPU at least
  // once: 1.4B MBS 32 / 8: 865 / 901 vs 703 / 766 TF/s; tensor-parallel shapes with 192 blocks (24 heads
  // x 8 or 2 x 12 x 8): 758 / 751 vs 672 / 659; with fewer blocks (12 heads x 8) the persistent one-tile
  // kernel keeps every SM busy (555 vs 386 TF/s). `profiles/r02_attn_fwd_tp_shapes.txt`.
  static const char* two_q_env = std::getenv("GPTB200_ATTN_FWD_2Q");  // A/B: 1 always, 0 never
  const int blocks256 = a.batch * a.heads * (a.seq / 256);
  const bool two_q = two_q_env ? two_q_env[0] == '1' : blocks256 >= device_sm_count();
  if (two_q && a.seq % 256 == 0 && (a.head_dim == 64 || a.head_dim == 128) && !per_block)
    return a.head_dim == 64 ? fwd_tc2q<64>(a, qkv, out, lse, st) : fwd_tc2q<128>(a, qkv, out, lse, st);
  switch (a.head_dim) {
    case 64: return per_block ? fwd_tc<64>(a, qkv, out, lse, st) : fwd_tc_persistent<64>(a, qkv, out, lse, st);
    case 128: return per_block ? fwd_tc<128>(a, qkv, out, lse, st) : fwd_tc_persistent<128>(a, qkv, out, lse, st);
    case 160: return fwd_tc<160>(a, qkv, out, lse, st);
    default: return 1;
  }
}

}  // namespace gptb200
