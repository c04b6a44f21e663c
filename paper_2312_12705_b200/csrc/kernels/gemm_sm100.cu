// K1-K4: Megatron column/row-parallel GEMMs (forward, dgrad, wgrad) on sm_100a.
//
// One persistent, warp-specialised kernel computes C[m,n] = sum_k A(m,k) * B(n,k) with
//   A(m,k) = A[m*lda + k]  (K-major)  or  A[k*lda + m]  (MN-major)
//   B(n,k) = B[n*ldb + k]  (K-major)  or  B[k*ldb + n]  (MN-major)
// which covers every GEMM of the GPT block (row-major tensors throughout):
//   forward  Y  = X  . W^T   A=X  K-major, B=W  K-major
//   dgrad    dX = dY . W     A=dY K-major, B=W  MN-major
//   wgrad    dW = dY^T . X   A=dY MN-major, B=X MN-major  (fp32 accumulate into main grad)
//
// Roles per CTA (192 threads): warp 0 = TMA producer, warp 1 = TMEM owner + tcgen05.mma
// issuer, warps 2..5 = epilogue (TMEM -> registers -> fused epilogue -> HBM). Operand tiles
// land in 128B-swizzled shared memory through TMA; the fp32 accumulator lives in TMEM and
// is double-buffered so the epilogue of tile i overlaps the MMAs of tile i+1.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "gemm.h"
#include "pdl.cuh"
#include "sm100_ptx.cuh"
#include "tma_host.h"

namespace gptb200 {

namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;
constexpr int kThreads = 320;  // warp 0 TMA, warp 1 MMA, warps 2..9 epilogue (2 per TMEM lane quarter)

// CG = 1: one CTA computes a 128 x BN tile.  CG = 2: a CTA pair (cluster of 2) computes a
// 256 x BN tile with tcgen05.mma.cta_group::2 — each CTA stages 128 rows of A and BN/2 rows of B,
// halving the per-SM operand traffic through shared memory.
template <int BN, int CG>
struct GemmCfg {
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = (BN / CG) * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = (kStageBytes <= 32768) ? 6 : 4;
  // BN = 512 (CTA pair 256 x 512): two N = 256 MMAs per k-step share A; the fp32 accumulator then
  // fills TMEM, so it is single-buffered (the epilogue is not overlapped with the next mainloop).
  static constexpr int kNsub = BN > 256 ? BN / 256 : 1;
  static constexpr int kMmaN = BN / kNsub;
  static constexpr int kAccBufs = 2 * BN <= 512 ? 2 : 1;
  static constexpr int kTmemCols = kAccBufs * BN;
  static constexpr int kStageOutBytes = 8 * 4096;  // per epilogue warp: one [32 rows][128 B] swizzled box
  static constexpr int kSmemBytes = kStages * kStageBytes + kStageOutBytes + 1024 + 256;
};

__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float gelu_tanh(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  const float t = tanh_fast(k0 * (x + k1 * x * x * x));
  return 0.5f * x * (1.f + t);
}

__device__ __forceinline__ float gelu_tanh_grad(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  const float t = tanh_fast(k0 * (x + k1 * x * x * x));
  return 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * k0 * (1.f + 3.f * k1 * x * x);
}

// Tile order: groups of kGroup M-blocks sweep all N-blocks so concurrently running CTAs share
// both operand panels in L2.
__device__ __forceinline__ void tile_coords(int tile, int num_m, int num_n, int kGroup, int& mb, int& nb) {
  if (kGroup <= 0) kGroup = 8;
  int group = tile / (kGroup * num_n);
  int first_m = group * kGroup;
  int gsize = min(kGroup, num_m - first_m);
  int in_group = tile - group * kGroup * num_n;
  mb = first_m + in_group % gsize;
  nb = in_group / gsize;
}

// Output path: bf16 tiles of >= 128 columns and every fp32 tile leave through TMA (swizzled smem
// box per epilogue warp -> full-line bulk tensor store, or bulk reduce-add for fp32 accumulation
// and K slices); the 64-column bf16 configuration keeps direct vector stores.
template <int BN, int EPI>
constexpr bool kTmaOut = EPI == EPI_F32 || BN >= 128;

template <int BN, int CG, bool A_MN, bool B_MN, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_sm100_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmC2,
                      const GemmParams p) {
  using Cfg = GemmCfg<BN, CG>;
  constexpr int kStages = Cfg::kStages;
  constexpr int kTileM = kBM * CG;   // rows of C per tile (per CTA pair)
  constexpr int kBN_cta = BN / CG;   // rows of B staged by each CTA
  constexpr int kNsub = Cfg::kNsub, kAccBufs = Cfg::kAccBufs;
  constexpr int kNsubRows = kBN_cta / kNsub;  // B rows per CTA per N sub-tile
  constexpr uint32_t kBSubOff = B_MN ? (kNsubRows / 64) * kBK * 128 : kNsubRows * 128;  // smem bytes
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = ptx::smem_align1024(smem_raw);
  uint8_t* stage_out = smem + kStages * Cfg::kStageBytes;  // 1024-aligned (stage sizes are 1 KB multiples)
  uint64_t* full = reinterpret_cast<uint64_t*>(stage_out + Cfg::kStageOutBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x / 32), 0);  // provably warp-uniform
  const int lane = threadIdx.x % 32;
  const uint32_t rank = CG == 2 ? ptx::cluster_ctarank() : 0;
  const bool leader = rank == 0;
  const int cluster_id = blockIdx.x / CG;
  const int num_clusters = gridDim.x / CG;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tmA);
    ptx::tma_prefetch_desc(&tmB);
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 8 * CG);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) {
    if constexpr (CG == 2)
      ptx::tmem_alloc_cg2<Cfg::kTmemCols>(tmem_slot);
    else
      ptx::tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  }
  ptx::tc_fence_before();
  if constexpr (CG == 2)
    ptx::cluster_sync();
  else
    __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_slot, 0);  // warp-uniform
  // prologue done (smem / TMEM / barriers only): let the next kernel in the stream be scheduled,
  // then wait for the previous one before the first global-memory access
  pdl_trigger();
  pdl_wait();

  const int num_m = p.M / kTileM;
  const int num_n = p.N / BN;
  const int num_tiles = num_m * num_n;
  const int S = p.split_k > 1 ? p.split_k : 1;  // K slices per tile (work unit = tile x slice)
  const int kblocks_total = p.K / kBK;
  const int num_units = num_tiles * S;
  // k-block range of slice ks (slices may differ by one block)
  auto slice_begin = [&](int ks) { return ks * kblocks_total / S; };

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int unit = cluster_id; unit < num_units; unit += num_clusters) {
        const int tile = unit % num_tiles, kslice = unit / num_tiles;
        const int kb0 = slice_begin(kslice), kblocks = slice_begin(kslice + 1) - kb0;
        int mb, nb;
        tile_coords(tile, num_m, num_n, p.group_m, mb, nb);
        const int m0 = mb * kTileM + rank * kBM;
        auto n0_of = [&](int ns) { return nb * BN + ns * (BN / kNsub) + rank * kNsubRows; };
        for (int kb = 0; kb < kblocks; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * Cfg::kStageBytes;
          uint8_t* sb = sa + Cfg::kABytes;
          if (leader) ptx::mbar_arrive_expect_tx(&full[stage], CG * Cfg::kStageBytes);
          const int k0 = (kb0 + kb) * kBK;
          auto load = [&](void* dst, const CUtensorMap* tm, int c0, int c1) {
            if constexpr (CG == 2)
              ptx::tma_load_2d_cg2(dst, tm, &full[stage], c0, c1);
            else
              ptx::tma_load_2d(dst, tm, &full[stage], c0, c1);
          };
          if constexpr (A_MN) {
#pragma unroll
            for (int c = 0; c < kBM / 64; ++c) load(sa + c * kBK * 128, &tmA, m0 + 64 * c, k0);
          } else {
            load(sa, &tmA, k0, m0);
          }
          if constexpr (B_MN) {
#pragma unroll
            for (int c = 0; c < kBN_cta / 64; ++c)
              load(sb + c * kBK * 128, &tmB, n0_of(c / (kNsubRows / 64)) + 64 * (c % (kNsubRows / 64)), k0);
          } else {
#pragma unroll
            for (int ns = 0; ns < kNsub; ++ns) load(sb + ns * kBSubOff, &tmB, k0, n0_of(ns));
          }
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader CTA only)
    if (leader) {  // all 32 lanes: uniform descriptors, one elected lane issues
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(kTileM, Cfg::kMmaN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int unit = cluster_id; unit < num_units; unit += num_clusters, ++it) {
        const int kslice = unit / num_tiles;
        const int kblocks = slice_begin(kslice + 1) - slice_begin(kslice);
        const int acc = kAccBufs == 2 ? (it & 1) : 0;
        const int use = kAccBufs == 2 ? (it >> 1) : it;
        ptx::mbar_wait(&tempty[acc], (use & 1) ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < kblocks; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint32_t sa = ptx::smem_u32(smem + stage * Cfg::kStageBytes);
          const uint32_t sb = sa + Cfg::kABytes;
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            uint64_t adesc, bdesc;
            if constexpr (A_MN)
              adesc = ptx::smem_desc_sw128(sa + k * 2048, kBK * 128, 1024);
            else
              adesc = ptx::smem_desc_sw128(sa + k * 32, 16, 1024);
            if constexpr (B_MN)
              bdesc = ptx::smem_desc_sw128(sb + k * 2048, kBK * 128, 1024);
            else
              bdesc = ptx::smem_desc_sw128(sb + k * 32, 16, 1024);
#pragma unroll
            for (int ns = 0; ns < kNsub; ++ns) {
              if constexpr (CG == 2)
                ptx::mma_bf16_ss_cg2_w(d_tmem + ns * Cfg::kMmaN, adesc, bdesc + ((ns * kBSubOff) >> 4), idesc,
                                       (kb | k) != 0 ? 1u : 0u);
              else
                ptx::mma_bf16_ss_w(d_tmem + ns * Cfg::kMmaN, adesc, bdesc + ((ns * kBSubOff) >> 4), idesc,
                                   (kb | k) != 0 ? 1u : 0u);
            }
          }
          if constexpr (CG == 2)
            ptx::mma_commit_cg2_w(&empty[stage]);
          else
            ptx::mma_commit_w(&empty[stage]);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if constexpr (CG == 2)
          ptx::mma_commit_cg2_w(&tfull[acc]);
        else
          ptx::mma_commit_w(&tfull[acc]);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int ehalf = (warp - 2) >> 2;  // which half of the tile's columns this warp converts
    int it = 0;
    for (int unit = cluster_id; unit < num_units; unit += num_clusters, ++it) {
      const int tile = unit % num_tiles;
      int mb, nb;
      tile_coords(tile, num_m, num_n, p.group_m, mb, nb);
      const int acc = kAccBufs == 2 ? (it & 1) : 0;
      ptx::mbar_wait(&tfull[acc], ((kAccBufs == 2 ? (it >> 1) : it)) & 1);
      ptx::tc_fence_after();
      const int row_base = mb * kTileM + rank * kBM + 32 * q;
      const int row = row_base + lane;
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(32 * q) << 16) + acc * BN;
      if constexpr (kTmaOut<BN, EPI>) {
        // this warp's [32 rows][128 B] box; 16-byte unit u of row `lane` at the 128B-swizzled slot
        uint8_t* box = stage_out + (warp - 2) * 4096;
        uint8_t* box_row = box + lane * 128;
        auto put = [&](int u, uint4 val) { *reinterpret_cast<uint4*>(box_row + ((u ^ (lane & 7)) << 4)) = val; };
        auto box_free = [&]() {  // the previous bulk op of this warp has finished reading the box
          if (lane == 0) ptx::bulk_wait_read0();
          __syncwarp();
        };
        auto flush = [&](const CUtensorMap* tm, int col, bool reduce) {
          ptx::fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            if (reduce)
              ptx::tma_reduce_add_2d(tm, box, col, row_base);
            else
              ptx::tma_store_2d(tm, box, col, row_base);
            ptx::bulk_commit();
          }
        };
        if constexpr (EPI == EPI_F32) {
          const bool reduce = p.accumulate || S > 1;
#pragma unroll 1
          for (int c = ehalf * (BN / 64); c < (ehalf + 1) * (BN / 64); ++c) {
            uint32_t r[32];
            ptx::tmem_ld_32x32b_x32(t_row + c * 32, r);
            ptx::tmem_ld_wait();
            box_free();
#pragma unroll
            for (int u = 0; u < 8; ++u) put(u, make_uint4(r[4 * u], r[4 * u + 1], r[4 * u + 2], r[4 * u + 3]));
            flush(&tmC, nb * BN + c * 32, reduce);
          }
        } else {
#pragma unroll 1
          for (int c2 = ehalf * (BN / 128); c2 < (ehalf + 1) * (BN / 128); ++c2) {  // 64-column units
            uint32_t g[2][16];
            float rowdot = 0.f;
            float rs_m = -INFINITY, rs_s = 0.f;  // online (max, sum exp) of this row's 64 stored values
            // dGeLU: this row's 64 pre-activation values are loaded before the TMEM reads so the
            // two latencies overlap (the epilogue bounds the dgrad GEMM's tensor-pipe activity)
            uint4 auxv[2][4];
            if constexpr (EPI == EPI_DGELU) {
              const uint4* h4 = reinterpret_cast<const uint4*>(p.aux + static_cast<size_t>(row) * p.ldaux + nb * BN +
                                                               c2 * 64);
#pragma unroll
              for (int j = 0; j < 8; ++j) auxv[j / 4][j % 4] = h4[j];
            }
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              const int c = 2 * c2 + hh;
              uint32_t r[32];
              ptx::tmem_ld_32x32b_x32(t_row + c * 32, r);
              ptx::tmem_ld_wait();
              const int n = nb * BN + c * 32;
              float v[32];
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
              if constexpr (EPI == EPI_BF16 || EPI == EPI_BIAS_GELU) {
                if (p.bias != nullptr) {
                  const uint4* b4 = reinterpret_cast<const uint4*>(p.bias + n);
#pragma unroll
                  for (int j = 0; j < 4; ++j) {
                    uint4 bb = b4[j];
                    uint32_t w[4] = {bb.x, bb.y, bb.z, bb.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                      float2 f = ptx::unpack_bf16(w[e]);
                      v[8 * j + 2 * e] += f.x;
                      v[8 * j + 2 * e + 1] += f.y;
                    }
                  }
                }
              }
              if constexpr (EPI == EPI_DGELU) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const uint4 hv = auxv[hh][j];
                  uint32_t w[4] = {hv.x, hv.y, hv.z, hv.w};
#pragma unroll
                  for (int e = 0; e < 4; ++e) {
                    float2 f = ptx::unpack_bf16(w[e]);
                    v[8 * j + 2 * e] *= gelu_tanh_grad(f.x);
                    v[8 * j + 2 * e + 1] *= gelu_tanh_grad(f.y);
                  }
                }
              }
              uint32_t packed[16];
#pragma unroll
              for (int j = 0; j < 16; ++j) packed[j] = ptx::pack_bf16(v[2 * j], v[2 * j + 1]);
              if constexpr (EPI == EPI_BF16) {
                if (p.rowdot_out != nullptr) {  // D partial over these 32 columns (of the stored bf16)
                  const uint4* o4 = reinterpret_cast<const uint4*>(p.rowdot_b + static_cast<size_t>(row) * p.ldc + n);
#pragma unroll
                  for (int j = 0; j < 4; ++j) {
                    const uint4 ov = o4[j];
                    const uint32_t ow[4] = {ov.x, ov.y, ov.z, ov.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                      const float2 a = ptx::unpack_bf16(packed[4 * j + e]), b = ptx::unpack_bf16(ow[e]);
                      rowdot = fmaf(a.x, b.x, fmaf(a.y, b.y, rowdot));
                    }
                  }
                }
              }
              if constexpr (EPI == EPI_BIAS_GELU) {
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                  float2 f = ptx::unpack_bf16(packed[j]);
                  g[hh][j] = ptx::pack_bf16(gelu_tanh(f.x), gelu_tanh(f.y));
                }
              }
              if constexpr (EPI == EPI_BF16) {
                if (p.rowstat_part != nullptr) {
                  constexpr float kL2e = 1.4426950408889634f;
                  float mx = rs_m;
#pragma unroll
                  for (int j = 0; j < 16; ++j) {
                    const float2 f = ptx::unpack_bf16(packed[j]);
                    mx = fmaxf(mx, fmaxf(f.x, f.y));
                  }
                  float acc = rs_s * exp2f((rs_m - mx) * kL2e);
#pragma unroll
                  for (int j = 0; j < 16; ++j) {
                    const float2 f = ptx::unpack_bf16(packed[j]);
                    acc += exp2f((f.x - mx) * kL2e) + exp2f((f.y - mx) * kL2e);
                  }
                  rs_m = mx;
                  rs_s = acc;
                }
              }
              if (hh == 0) box_free();
#pragma unroll
              for (int j = 0; j < 4; ++j)
                put(4 * hh + j, make_uint4(packed[4 * j], packed[4 * j + 1], packed[4 * j + 2], packed[4 * j + 3]));
            }
            flush(&tmC, nb * BN + c2 * 64, false);
            if constexpr (EPI == EPI_BF16) {
              if (p.rowstat_part != nullptr)
                p.rowstat_part[static_cast<size_t>(row) * (p.N / 64) + (nb * BN + c2 * 64) / 64] = make_float2(rs_m, rs_s);
            }
            if constexpr (EPI == EPI_BF16 || EPI == EPI_DGELU) {
              if (p.colsum_part != nullptr) {  // this warp's 32 rows x 64 columns, from the staged box
                float s0 = 0.f, s1 = 0.f;
#pragma unroll 8
                for (int r = 0; r < 32; ++r) {
                  const uint8_t* brow = box + r * 128;
                  s0 += __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(
                      brow + (((lane >> 3) ^ (r & 7)) << 4) + (lane & 7) * 2));
                  s1 += __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(
                      brow + ((((lane >> 3) + 4) ^ (r & 7)) << 4) + (lane & 7) * 2));
                }
                float* dst = p.colsum_part + static_cast<size_t>(row_base / 32) * p.N + nb * BN + c2 * 64;
                dst[lane] = s0;
                dst[lane + 32] = s1;
              }
            }
            if constexpr (EPI == EPI_BF16) {
              if (p.rowdot_out != nullptr) {  // <= 2 partials per (row, head) onto zero: order-free
                const int n0 = nb * BN + c2 * 64;
                const int bq = row / p.rowdot_seq, q = row % p.rowdot_seq;
                atomicAdd(p.rowdot_out + (static_cast<size_t>(bq) * p.rowdot_heads + n0 / 128) * p.rowdot_seq + q, rowdot);
              }
            }
            if constexpr (EPI == EPI_BIAS_GELU) {
              box_free();
#pragma unroll
              for (int hh = 0; hh < 2; ++hh)
#pragma unroll
                for (int j = 0; j < 4; ++j)
                  put(4 * hh + j, make_uint4(g[hh][4 * j], g[hh][4 * j + 1], g[hh][4 * j + 2], g[hh][4 * j + 3]));
              flush(&tmC2, nb * BN + c2 * 64, false);
            }
          }
        }
      } else {
#pragma unroll 1
      for (int c = ehalf * (BN / 64); c < (ehalf + 1) * (BN / 64); ++c) {
        uint32_t r[32];
        ptx::tmem_ld_32x32b_x32(t_row + c * 32, r);
        ptx::tmem_ld_wait();
        const int n = nb * BN + c * 32;
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        if constexpr (EPI == EPI_F32) {
          float* dst = reinterpret_cast<float*>(p.C) + static_cast<size_t>(row) * p.ldc + n;
          float4* d4 = reinterpret_cast<float4*>(dst);
          if (S > 1) {  // K-sliced: the slices meet in C through fp32 reductions
#pragma unroll
            for (int j = 0; j < 8; ++j) ptx::red_add_f32x4(dst + 4 * j, v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          } else
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float4 o = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            if (p.accumulate) {
              float4 old = d4[j];
              o.x += old.x;
              o.y += old.y;
              o.z += old.z;
              o.w += old.w;
            }
            d4[j] = o;
          }
        } else {
          if constexpr (EPI == EPI_BF16 || EPI == EPI_BIAS_GELU) {
            if (p.bias != nullptr) {
              const uint4* b4 = reinterpret_cast<const uint4*>(p.bias + n);
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                uint4 bb = b4[j];
                uint32_t w[4] = {bb.x, bb.y, bb.z, bb.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  float2 f = ptx::unpack_bf16(w[e]);
                  v[8 * j + 2 * e] += f.x;
                  v[8 * j + 2 * e + 1] += f.y;
                }
              }
            }
          }
          if constexpr (EPI == EPI_DGELU) {
            const uint4* h4 = reinterpret_cast<const uint4*>(
                p.aux + static_cast<size_t>(row) * p.ldaux + n);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              uint4 hh = h4[j];
              uint32_t w[4] = {hh.x, hh.y, hh.z, hh.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                float2 f = ptx::unpack_bf16(w[e]);
                v[8 * j + 2 * e] *= gelu_tanh_grad(f.x);
                v[8 * j + 2 * e + 1] *= gelu_tanh_grad(f.y);
              }
            }
          }
          uint32_t packed[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) packed[j] = ptx::pack_bf16(v[2 * j], v[2 * j + 1]);
          uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.C) +
                                                static_cast<size_t>(row) * p.ldc + n);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            dst[j] = make_uint4(packed[4 * j], packed[4 * j + 1], packed[4 * j + 2],
                                packed[4 * j + 3]);
          if constexpr (EPI == EPI_BIAS_GELU) {
            uint32_t g[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              float2 f = ptx::unpack_bf16(packed[j]);
              g[j] = ptx::pack_bf16(gelu_tanh(f.x), gelu_tanh(f.y));
            }
            uint4* dst2 = reinterpret_cast<uint4*>(p.C2 + static_cast<size_t>(row) * p.ldc + n);
#pragma unroll
            for (int j = 0; j < 4; ++j)
              dst2[j] = make_uint4(g[4 * j], g[4 * j + 1], g[4 * j + 2], g[4 * j + 3]);
          }
        }
      }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 2)
          ptx::mbar_arrive_cluster(&tempty[acc], 0);  // the leader's MMA thread waits on it
        else
          ptx::mbar_arrive(&tempty[acc]);
      }
    }
  }

  if (warp >= 2 && lane == 0) ptx::bulk_wait0();  // output bulk stores / reductions complete
  if constexpr (CG == 2)
    ptx::cluster_sync();
  else
    __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    if constexpr (CG == 2)
      ptx::tmem_dealloc_cg2<Cfg::kTmemCols>(tmem_base);
    else
      ptx::tmem_dealloc<Cfg::kTmemCols>(tmem_base);
  }
}

// ---------------------------------------------------------------- host side
bool make_tmap(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld, uint32_t box_outer) {
  return make_tmap_bf16(m, ptr, inner, outer, ld, 64, box_outer);
}

int num_sms() { return device_sm_count(); }

template <int BN, int CG, bool A_MN, bool B_MN, int EPI>
int launch(const GemmParams& p, cudaStream_t stream) {
  using Cfg = GemmCfg<BN, CG>;
  auto kern = gemm_sm100_kernel<BN, CG, A_MN, B_MN, EPI>;
  if (ensure_dynamic_smem(reinterpret_cast<const void*>(kern), Cfg::kSmemBytes) != 0) return kGemmErrCuda;
  count_variant(CG == 1 ? KV_GEMM_SINGLE : (BN == 512 ? KV_GEMM_PAIR_512 : KV_GEMM_PAIR_256));
  if (p.split_k > 1) count_variant(KV_GEMM_KSPLIT);
  CUtensorMap ta, tb;
  bool ok = A_MN ? make_tmap(&ta, p.A, p.M, p.K, p.lda, 64)
                 : make_tmap(&ta, p.A, p.K, p.M, p.lda, kBM);
  ok = ok && (B_MN ? make_tmap(&tb, p.B, p.N, p.K, p.ldb, 64)
                   : make_tmap(&tb, p.B, p.K, p.N, p.ldb, BN / CG / GemmCfg<BN, CG>::kNsub));
  CUtensorMap tc, tc2;
  if constexpr (EPI == EPI_F32) {
    ok = ok && make_tmap_f32(&tc, p.C, p.N, p.M, p.ldc, 32, 32, true);
    tc2 = tc;
  } else {
    ok = ok && make_tmap_bf16(&tc, p.C, p.N, p.M, p.ldc, 64, 32);
    ok = ok && (EPI == EPI_BIAS_GELU ? make_tmap_bf16(&tc2, p.C2, p.N, p.M, p.ldc, 64, 32) : (tc2 = tc, true));
  }
  if (!ok) return kGemmErrTmap;
  const int tiles = (p.M / (kBM * CG)) * (p.N / BN) * (p.split_k > 1 ? p.split_k : 1);
  const int max_clusters = num_sms() / CG;
  const int grid = CG * (tiles < max_clusters ? tiles : max_clusters);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = Cfg::kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // see pdl.cuh
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  if (cudaLaunchKernelEx(&cfg, kern, ta, tb, tc, tc2, p) != cudaSuccess) return kGemmErrCuda;
  return cudaGetLastError() == cudaSuccess ? kGemmOk : kGemmErrCuda;
}

template <int BN, int CG, int EPI>
int dispatch_major(const GemmParams& p, cudaStream_t s) {
  if (!p.a_mn && !p.b_mn) return launch<BN, CG, false, false, EPI>(p, s);
  if (!p.a_mn && p.b_mn) return launch<BN, CG, false, true, EPI>(p, s);
  if (p.a_mn && p.b_mn) return launch<BN, CG, true, true, EPI>(p, s);
  return launch<BN, CG, true, false, EPI>(p, s);
}

template <int BN, int CG>
int dispatch_epi(const GemmParams& p, cudaStream_t s) {
  switch (p.epi) {
    case EPI_BF16: return dispatch_major<BN, CG, EPI_BF16>(p, s);
    case EPI_BIAS_GELU: return dispatch_major<BN, CG, EPI_BIAS_GELU>(p, s);
    case EPI_F32: return dispatch_major<BN, CG, EPI_F32>(p, s);
    case EPI_DGELU: return dispatch_major<BN, CG, EPI_DGELU>(p, s);
    default: return kGemmErrShape;
  }
}

int g_force_cg = 0;  // test hook: 1 or 2 forces the CTA-group choice (0 = automatic)

// K-slice count for an accumulating fp32 GEMM: the S (slices >= 1024 deep) that best fills the
// last wave of `slots` concurrent tiles, charging each extra slice for its fp32 reduction traffic
// (measured: ~3% of the GEMM per extra slice at K = 16384, i.e. ~500/K).
// Raster group: 8 M-blocks by default. Weight-gradient GEMMs (fp32 accumulate, few output tiles,
// K = tokens) stream both operands from HBM: the raster runs fastest along the shorter tile dimension
// of C, so the co-resident tiles share the long operand panels (measured at the 1.4B MBS-32 shapes,
// DRAM bytes per launch: QKV wgrad 2.71 -> 2.23 GB, fc1 3.64 -> 3.17 GB with group 1; fc2 best at
// group >= num_m; `profiles/r02_gemm_group.txt`).
int choose_group(const GemmParams& p, int num_m, int num_n, int slots) {
  static const int forced = [] {
    const char* e = std::getenv("GPTB200_GEMM_GROUP");  // A/B switch: fixed group for every GEMM
    return e ? std::atoi(e) : 0;
  }();
  (void)slots;
  if (forced > 0) return forced;
  // measured on the long-K (K = tokens >= 16384) weight gradients of the data-parallel shapes; the
  // tensor-parallel ones (K = 2048..8192 tokens, large C) keep the group of 8
  if (p.epi == EPI_F32 && p.accumulate && p.K >= 16384) return num_m >= num_n ? 1 : num_m;
  return 8;
}

int choose_split(const GemmParams& p, int tiles, int slots) {
  if (p.split_k > 0) return p.split_k;
  if (p.epi != EPI_F32 || !p.accumulate) return 1;
  const int kblocks = p.K / kBK;
  int best = 1;
  double best_score = -1.0;
  for (int S = 1; S <= 8; ++S) {
    if (S > 1 && kblocks / S < 16) continue;
    const int units = tiles * S;
    const int waves = (units + slots - 1) / slots;
    const double score =
        static_cast<double>(units) / (static_cast<double>(waves) * slots) - (S - 1) * 500.0 / p.K;
    if (score > best_score + 1e-9) {
      best_score = score;
      best = S;
    }
  }
  return best;
}

}  // namespace

void gemm_force_cta_group(int cg) { g_force_cg = cg; }

int gemm_bf16(const GemmParams& p, cudaStream_t stream) {
  if (p.M <= 0 || p.N <= 0 || p.K <= 0) return kGemmErrShape;
  if (p.M % kBM != 0 || p.K % kBK != 0 || p.N % 64 != 0) return kGemmErrShape;
  if (p.epi == EPI_BIAS_GELU && p.C2 == nullptr) return kGemmErrShape;
  if (p.epi == EPI_DGELU && p.aux == nullptr) return kGemmErrShape;
  if (p.split_k > 1 && (p.epi != EPI_F32 || !p.accumulate || p.K / kBK < p.split_k)) return kGemmErrShape;
  if (p.colsum_part && ((p.epi != EPI_BF16 && p.epi != EPI_DGELU) || p.N % 128 != 0)) return kGemmErrShape;
  if (p.rowstat_part && (p.epi != EPI_BF16 || p.N % 128 != 0)) return kGemmErrShape;
  if (p.rowdot_out && (p.epi != EPI_BF16 || p.N % 128 != 0 || p.rowdot_seq <= 0 || p.M % p.rowdot_seq != 0))
    return kGemmErrShape;
  // CTA pairs (256 x 256 tiles) when the problem yields at least one full wave of pairs;
  // otherwise single-CTA 128 x BN tiles with the widest BN that still fills the machine.
  const bool pair_ok = p.M % 256 == 0 && p.N % 256 == 0;
  // >= ~85% of the pairs busy in a single wave beats 1.7 waves of single-CTA tiles
  const bool pair_wave = pair_ok && (p.M / 256) * (p.N / 256) * 8 >= (num_sms() / 2) * 7 - 8;
  GemmParams q = p;
  // 256 x 512 pair tiles: 25% less L2->SMEM operand traffic per FLOP (measured: 8192^3 sustained
  // 1281 -> 1325 TF/s under the power cap) but a single-buffered accumulator, so only for long K
  // when the bigger tiles still fill the waves (the training-step shapes do not qualify).
  const bool p512_ok = p.M % 256 == 0 && p.N % 512 == 0 && !(p.epi == EPI_F32 && p.accumulate);
  const int t512 = p512_ok ? (p.M / 256) * (p.N / 512) : 0, slots = num_sms() / 2;
  const bool p512_auto = p512_ok && p.K >= 8192 && t512 >= slots &&
                         static_cast<double>(t512) / (((t512 + slots - 1) / slots) * slots) >= 0.97;
  if ((g_force_cg == 3 && p512_ok) || (g_force_cg == 0 && p512_auto)) {
    q.split_k = choose_split(p, (p.M / 256) * (p.N / 512), num_sms() / 2);
    q.group_m = choose_group(p, p.M / 256, p.N / 512, num_sms() / 2);
    return dispatch_epi<512, 2>(q, stream);
  }
  if (g_force_cg == 2 ? pair_ok : (g_force_cg == 0 && pair_wave)) {
    q.split_k = choose_split(p, (p.M / 256) * (p.N / 256), num_sms() / 2);
    q.group_m = choose_group(p, p.M / 256, p.N / 256, num_sms() / 2);
    return dispatch_epi<256, 2>(q, stream);
  }
  const int bn = (p.N % 256 == 0) && (p.M / kBM) * (p.N / 256) >= num_sms() ? 256 : (p.N % 128 == 0 ? 128 : 64);
  q.split_k = choose_split(p, (p.M / kBM) * (p.N / bn), num_sms());
  q.group_m = choose_group(p, p.M / kBM, p.N / bn, num_sms());
  if (bn == 256) return dispatch_epi<256, 1>(q, stream);
  if (bn == 128) return dispatch_epi<128, 1>(q, stream);
  return dispatch_epi<64, 1>(q, stream);
}

}  // namespace gptb200
