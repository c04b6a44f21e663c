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
#include "sm100_ptx.cuh"
#include "tma_host.h"

#include <cstdio>

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
#else
#define WAIT(bar, par, id) ptx::mbar_wait(bar, par)
#endif
constexpr float kLog2e = 1.4426950408889634f;

template <int HD>
struct TcFwdCfg {
  static constexpr int NC = (HD + 63) / 64;             // 64-wide swizzle chunks of the head dim
  static constexpr int kStages = NC <= 2 ? 2 : 1;       // K ring and V ring depth
  static constexpr int kPBufs = NC <= 2 ? 2 : 1;        // P double buffer when smem allows
  static constexpr int kTileBytes = 128 * 128;          // one [128 rows][64] bf16 chunk
  static constexpr int kQBytes = NC * kTileBytes;
  static constexpr int kKVBytes = NC * kTileBytes;
  static constexpr int kPBytes = 2 * kTileBytes;        // P [128][128] = 2 chunks
  static constexpr int kSmem = kQBytes + 2 * kStages * kKVBytes + kPBufs * kPBytes + 1024 + 256;
  static constexpr int kTmemCols = 512;                 // S0 | S1 | O
};

template <int HD>
__global__ void __launch_bounds__(192, 1)
    fa_fwd_tc_kernel(const __grid_constant__ CUtensorMap tm_qkv, __nv_bfloat16* __restrict__ out,
                     float* __restrict__ lse, int s, int ht, float scale_log2) {
  using Cfg = TcFwdCfg<HD>;
  constexpr int NC = Cfg::NC, ST = Cfg::kStages, PB = Cfg::kPBufs;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + Cfg::kQBytes;             // [ST][NC][128][64]
  uint8_t* sV = sK + ST * Cfg::kKVBytes;       // [ST][NC][128][64]
  uint8_t* sP = sV + ST * Cfg::kKVBytes;       // [PB][2][128][64]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + PB * Cfg::kPBytes);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;        // [ST]
  uint64_t* k_empty = k_full + ST;    // [ST]  released when S_j completes
  uint64_t* v_full = k_empty + ST;    // [ST]
  uint64_t* v_empty = v_full + ST;    // [ST]  released when PV_j completes
  uint64_t* s_full = v_empty + ST;    // [2]
  uint64_t* s_free = s_full + 2;      // [2]
  uint64_t* p_full = s_free + 2;      // [PB]
  uint64_t* pv_done = p_full + PB;    // [PB]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + PB);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int qb = gridDim.x - 1 - blockIdx.x;  // heaviest causal blocks first
  const int b = blockIdx.y / ht, h = blockIdx.y % ht;
  const int dt = ht * HD;
  const int row0 = b * s;
  const int n_tiles = qb + 1;  // kBM == kBN: tile qb is the diagonal

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tm_qkv);
    ptx::mbar_init(q_full, 1);
    for (int i = 0; i < ST; ++i) {
      ptx::mbar_init(&k_full[i], 1);
      ptx::mbar_init(&k_empty[i], 1);
      ptx::mbar_init(&v_full[i], 1);
      ptx::mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&s_full[i], 1);
      ptx::mbar_init(&s_free[i], 4);
    }
    for (int i = 0; i < PB; ++i) {
      ptx::mbar_init(&p_full[i], 4);
      ptx::mbar_init(&pv_done[i], 1);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tO = tmem + 2 * kBN;

  if (warp == 0) {
    if (lane == 0) {
      ptx::mbar_arrive_expect_tx(q_full, Cfg::kQBytes);
      for (int c = 0; c < NC; ++c)
        ptx::tma_load_2d(sQ + c * Cfg::kTileBytes, &tm_qkv, q_full, h * HD + 64 * c, row0 + qb * kBM);
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j % ST, use = j / ST;
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
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(kBM, kBN, false, false);
      constexpr uint32_t idesc_o = ptx::idesc_bf16_f32(kBM, HD, false, true);
      const uint32_t q_addr = ptx::smem_u32(sQ), p_addr = ptx::smem_u32(sP);
      WAIT(q_full, 0, 3);
      auto issue_pv = [&](int j) {
        const int st = j % ST, pb = j % PB;
        WAIT(&p_full[pb], (j / PB) & 1, 4);
        WAIT(&v_full[st], (j / ST) & 1, 5);
        ptx::tc_fence_after();
        const uint32_t v_addr = ptx::smem_u32(sV + st * Cfg::kKVBytes);
        const uint32_t pa = p_addr + pb * Cfg::kPBytes;
#pragma unroll
        for (int kk = 0; kk < kBN / 16; ++kk) {
          const uint64_t a = ptx::smem_desc_sw128(pa + (kk / 4) * Cfg::kTileBytes + (kk % 4) * 32, 16, 1024);
          const uint64_t bd = ptx::smem_desc_sw128(v_addr + kk * 2048, Cfg::kTileBytes, 1024);
          ptx::mma_bf16_ss(tO, a, bd, idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
        }
        ptx::mma_commit(&pv_done[pb]);
        ptx::mma_commit(&v_empty[st]);
      };
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j % ST, buf = j & 1;
        WAIT(&k_full[st], (j / ST) & 1, 6);
        WAIT(&s_free[buf], ((j >> 1) & 1) ^ 1, 7);
        ptx::tc_fence_after();
        const uint32_t k_addr = ptx::smem_u32(sK + st * Cfg::kKVBytes);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = (kk / 4) * Cfg::kTileBytes + (kk % 4) * 32;
          ptx::mma_bf16_ss(tmem + buf * kBN, ptx::smem_desc_sw128(q_addr + off, 16, 1024),
                           ptx::smem_desc_sw128(k_addr + off, 16, 1024), idesc_s, kk > 0 ? 1u : 0u);
        }
        ptx::mma_commit(&s_full[buf]);
        ptx::mma_commit(&k_empty[st]);
        if (j > 0) issue_pv(j - 1);
      }
      issue_pv(n_tiles - 1);
    }
  } else {
    // ------------------------------------------------------------ softmax / epilogue
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;  // query row within the block == TMEM lane
    const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
    const int q_row = qb * kBM + r;
    float m_used = -INFINITY, l = 0.f;
    uint8_t* p_row0 = sP + r * 128;
    for (int j = 0; j < n_tiles; ++j) {
      const int buf = j & 1;
      WAIT(&s_full[buf], (j >> 1) & 1, 8);
      ptx::tc_fence_after();
      float x[kBN];
#pragma unroll
      for (int c = 0; c < kBN / 32; ++c) {
        uint32_t v[32];
        ptx::tmem_ld_32x32b_x32(tmem + lane_base + buf * kBN + c * 32, v);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) x[c * 32 + i] = __uint_as_float(v[i]) * scale_log2;
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&s_free[buf]);
      const bool diag = (j == qb);
      float mt = -INFINITY;
#pragma unroll
      for (int i = 0; i < kBN; ++i) {
        if (diag && i > r) x[i] = -INFINITY;
        mt = fmaxf(mt, x[i]);
      }
      // Lazy rescale (only when a row's max grows by > 2^8). tcgen05.ld/st are warp-collective,
      // so the decision is warp-uniform: every lane of the warp rescales (factor 1 if unchanged).
      if (__any_sync(0xffffffffu, mt > m_used + 8.f)) {
        const float m_new = fmaxf(m_used, mt);
        if (j > 0) {
          // O must hold all of PV_0..PV_{j-1} before it is rescaled
          WAIT(&pv_done[(j - 1) % PB], ((j - 1) / PB) & 1, 9);
          const float f = exp2f(m_used - m_new);
          l *= f;
          ptx::tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < (HD + 31) / 32; ++c) {
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
      // the P buffer of tile j must be free of PV_{j-PB}
      if (j >= PB) WAIT(&pv_done[j % PB], ((j / PB) - 1) & 1, 10);
      uint8_t* p_row = p_row0 + (j % PB) * Cfg::kPBytes;
      // P = exp2(x - m_used) -> bf16, 128B-swizzled K-major rows: chunk c2 (64 cols), 16B unit u
#pragma unroll
      for (int c2 = 0; c2 < 2; ++c2) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          float p[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            p[e] = exp2f(x[c2 * 64 + u * 8 + e] - m_used);
            l += p[e];
          }
          uint4 pk;
          pk.x = ptx::pack_bf16(p[0], p[1]);
          pk.y = ptx::pack_bf16(p[2], p[3]);
          pk.z = ptx::pack_bf16(p[4], p[5]);
          pk.w = ptx::pack_bf16(p[6], p[7]);
          *reinterpret_cast<uint4*>(p_row + c2 * Cfg::kTileBytes + ((u ^ (r & 7)) * 16)) = pk;
        }
      }
      ptx::fence_proxy_async();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&p_full[j % PB]);
    }
    WAIT(&pv_done[(n_tiles - 1) % PB], ((n_tiles - 1) / PB) & 1, 11);
    ptx::tc_fence_after();
    const float inv = 1.f / l;
    __nv_bfloat16* orow = out + static_cast<size_t>(row0 + q_row) * dt + h * HD;
#pragma unroll 1
    for (int c = 0; c < (HD + 31) / 32; ++c) {
      uint32_t v[32];
      ptx::tmem_ld_32x32b_x32(tO + lane_base + c * 32, v);
      ptx::tmem_ld_wait();
      const int ncol = (HD - c * 32) < 32 ? (HD - c * 32) : 32;
      if (ncol == 32) {
        uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 pk;
          pk.x = ptx::pack_bf16(__uint_as_float(v[8 * q + 0]) * inv, __uint_as_float(v[8 * q + 1]) * inv);
          pk.y = ptx::pack_bf16(__uint_as_float(v[8 * q + 2]) * inv, __uint_as_float(v[8 * q + 3]) * inv);
          pk.z = ptx::pack_bf16(__uint_as_float(v[8 * q + 4]) * inv, __uint_as_float(v[8 * q + 5]) * inv);
          pk.w = ptx::pack_bf16(__uint_as_float(v[8 * q + 6]) * inv, __uint_as_float(v[8 * q + 7]) * inv);
          dst[q] = pk;
        }
      }
    }
    lse[(static_cast<size_t>(b) * ht + h) * s + q_row] = m_used + log2f(l);
  }
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<Cfg::kTmemCols>(tmem);
  }
}

template <int HD>
int fwd_tc(const AttnShape& a, const __nv_bfloat16* qkv, __nv_bfloat16* out, float* lse, cudaStream_t st) {
  using Cfg = TcFwdCfg<HD>;
  static bool init = false;
  if (!init) {
    if (cudaFuncSetAttribute(fa_fwd_tc_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem) !=
        cudaSuccess)
      return 3;
    init = true;
  }
  const int dt = a.heads * HD;
  CUtensorMap tm;
  if (!make_tmap_bf16(&tm, qkv, 3 * static_cast<uint64_t>(dt), static_cast<uint64_t>(a.batch) * a.seq, 3 * dt, 64, 128))
    return 3;
  dim3 grid(a.seq / kBM, a.batch * a.heads);
  fa_fwd_tc_kernel<HD><<<grid, 192, Cfg::kSmem, st>>>(tm, out, lse, a.seq, a.heads,
                                                       kLog2e / sqrtf(static_cast<float>(HD)));
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

}  // namespace

int flash_attn_fwd_tc(const AttnShape& a, const __nv_bfloat16* qkv, __nv_bfloat16* out, float* lse, cudaStream_t st) {
  if (a.seq % kBM != 0) return 1;
  switch (a.head_dim) {
    case 64: return fwd_tc<64>(a, qkv, out, lse, st);
    case 128: return fwd_tc<128>(a, qkv, out, lse, st);
    case 160: return fwd_tc<160>(a, qkv, out, lse, st);
    default: return 1;
  }
}

}  // namespace gptb200
