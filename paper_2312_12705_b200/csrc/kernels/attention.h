// Causal flash attention (K5 forward, K6 backward) on tcgen05 / TMEM / TMA: attention_sm100.cu.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace gptb200 {

struct AttnShape {
  int batch = 0;     // sequences in the microbatch
  int seq = 0;       // s (multiple of 128)
  int heads = 0;     // heads on this TP rank
  int head_dim = 0;  // 64, 128 or 160
};

// qkv[M, 3*heads*hd] -> out[M, heads*hd], lse[batch, heads, seq] (log2 units).
int flash_attn_fwd(const AttnShape& a, const __nv_bfloat16* qkv, __nv_bfloat16* out, float* lse,
                   cudaStream_t st);

// tcgen05/TMEM forward (attention_sm100.cu); flash_attn_fwd dispatches to it.
int flash_attn_fwd_tc(const AttnShape& a, const __nv_bfloat16* qkv, __nv_bfloat16* out, float* lse,
                      cudaStream_t st);

// tcgen05 backward main kernel (hd 64 / 128 / 160): dK, dV into dqkv and dQ into the zeroed fp32 dq_acc
// (D must already hold rowsum(dO*O)).
int flash_attn_bwd_tc_main(const AttnShape& a, const __nv_bfloat16* qkv, const __nv_bfloat16* dout,
                           const float* lse, const float* D, float* dq_acc, __nv_bfloat16* dqkv,
                           cudaStream_t st, float* dbqkv = nullptr);

// Writes dqkv[M, 3*heads*hd]. Workspaces: D[batch*heads*seq] fp32, dq_acc[M*heads*hd] fp32.
// d_ready: D = rowsum(dO * O) was already produced (fused into the dO GEMM epilogue); only the
// dQ accumulator is cleared before the main kernel.
// dbqkv (fp32, 3*heads*hd, accumulated +=): the qkv bias gradient (column sums of dqkv) for hd 128,
// folded into the kernels; returns with it untouched for other head dims (the caller sums dqkv).
int flash_attn_bwd(const AttnShape& a, const __nv_bfloat16* qkv, const __nv_bfloat16* out,
                   const __nv_bfloat16* dout, const float* lse, float* D, float* dq_acc,
                   __nv_bfloat16* dqkv, cudaStream_t st, bool d_ready = false, float* dbqkv = nullptr);

}  // namespace gptb200
