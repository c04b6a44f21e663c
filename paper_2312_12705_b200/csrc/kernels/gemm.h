// Host-facing declaration of the sm_100a GEMM (see gemm_sm100.cu for the kernel).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace gptb200 {

enum GemmEpilogue {
  EPI_BF16 = 0,       // C(bf16) = acc (+ bias[n])
  EPI_BIAS_GELU = 1,  // C(bf16) = acc + bias[n];  C2(bf16) = gelu_tanh(C)
  EPI_F32 = 2,        // C(fp32) = acc, or C += acc when accumulate != 0
  EPI_DGELU = 3,      // C(bf16) = acc * gelu_tanh'(aux[m,n])
};

enum GemmStatus { kGemmOk = 0, kGemmErrShape = 1, kGemmErrTmap = 2, kGemmErrCuda = 3 };

struct GemmParams {
  int M = 0, N = 0, K = 0;
  const __nv_bfloat16* A = nullptr;
  int lda = 0;
  bool a_mn = false;  // A stored [K][M] (M contiguous) instead of [M][K]
  const __nv_bfloat16* B = nullptr;
  int ldb = 0;
  bool b_mn = false;  // B stored [K][N] instead of [N][K]
  void* C = nullptr;  // bf16 or fp32 depending on epi
  int ldc = 0;
  int epi = EPI_BF16;
  const __nv_bfloat16* bias = nullptr;  // [N]
  __nv_bfloat16* C2 = nullptr;          // second output (EPI_BIAS_GELU), ld = ldc
  const __nv_bfloat16* aux = nullptr;   // EPI_DGELU pre-activation
  int ldaux = 0;
  int accumulate = 0;
  // K slices per output tile (EPI_F32 with accumulate only): slices are reduced into C with fp32
  // vector atomics, which squares up the wave count of the few-tile, long-K weight-gradient GEMMs.
  // 0 = automatic, 1 = off.
  int split_k = 0;
  // Tile raster: groups of group_m M-blocks sweep all N-blocks (0 = automatic; see gemm_bf16).
  int group_m = 0;
  // Optional fused row-dot (EPI_BF16 only): rowdot_out[(m / seq * heads + n / hd) * seq + m % seq]
  // += sum over a head's hd columns of bf16(C[m, n]) * rowdot_b[m * ldc + n] (hd = 128; rowdot_out
  // zeroed by the caller). Used for the attention-backward D = rowsum(dO * O) on the dO GEMM.
  // Optional column partial sums of the stored bf16 C (EPI_DGELU / EPI_BF16, N % 128 == 0):
  // colsum_part[(m / 32) * N + n] = sum of C[m', n] over the 32-row block of m (deterministic;
  // reduce over the M/32 blocks afterwards). Used for the fc1 bias gradient from dGeLU(dgrad).
  float* colsum_part = nullptr;
  // Optional per-row softmax statistics of the stored bf16 C (EPI_BF16, N % 128 == 0): rowstat_part
  // [m * (N / 64) + n / 64] = (max, sum exp(x - max)) over the 64 columns [n, n + 64) of row m. The LM
  // head uses them so the cross-entropy statistics need not re-read the [M, V] logits.
  float2* rowstat_part = nullptr;
  float* rowdot_out = nullptr;
  const __nv_bfloat16* rowdot_b = nullptr;
  int rowdot_seq = 0, rowdot_heads = 0;
};

// Requires M % 128 == 0, K % 64 == 0, N % 64 == 0, 16-byte aligned rows.
int gemm_bf16(const GemmParams& p, cudaStream_t stream);

// Test hook: 0 = automatic tile choice, 1 = single-CTA tiles only, 2 = CTA pairs when divisible.
void gemm_force_cta_group(int cg);

}  // namespace gptb200
