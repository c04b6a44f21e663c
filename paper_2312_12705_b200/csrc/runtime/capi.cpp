// C-ABI entry points (include/trainplan/capi.h). Kernel-level wrappers live here; the
// session (train step) entries are in session_capi.cpp.
#include "trainplan/capi.h"

#include <cuda_runtime.h>

#include <string>

#include "kernels/gemm.h"
#include "runtime/status.h"

using namespace gptb200;

extern "C" {

const char* tp_last_error(void) { return last_error().c_str(); }

int tp_abi_version(void) { return 1; }

int tp_gemm_bf16(int M, int N, int K, const void* A, int lda, int a_mn, const void* B, int ldb,
                 int b_mn, void* C, int ldc, int epi, const void* bias, void* C2, const void* aux,
                 int ldaux, int accumulate, void* stream) {
  GemmParams p;
  p.M = M;
  p.N = N;
  p.K = K;
  p.A = static_cast<const __nv_bfloat16*>(A);
  p.lda = lda;
  p.a_mn = a_mn != 0;
  p.B = static_cast<const __nv_bfloat16*>(B);
  p.ldb = ldb;
  p.b_mn = b_mn != 0;
  p.C = C;
  p.ldc = ldc;
  p.epi = epi;
  p.bias = static_cast<const __nv_bfloat16*>(bias);
  p.C2 = static_cast<__nv_bfloat16*>(C2);
  p.aux = static_cast<const __nv_bfloat16*>(aux);
  p.ldaux = ldaux;
  p.accumulate = accumulate;
  int r = gemm_bf16(p, static_cast<cudaStream_t>(stream));
  switch (r) {
    case kGemmOk: return clear_error();
    case kGemmErrShape:
      return set_error(TP_ERR_INVALID, "tp_gemm_bf16: unsupported shape M=" + std::to_string(M) +
                                           " N=" + std::to_string(N) + " K=" + std::to_string(K));
    case kGemmErrTmap: return set_error(TP_ERR_CUDA, "tp_gemm_bf16: TMA descriptor encode failed");
    default: return set_cuda_error("tp_gemm_bf16");
  }
}

int tp_gemm_force_cta_group(int cg) {
  if (cg < 0 || cg > 3) return set_error(TP_ERR_INVALID, "tp_gemm_force_cta_group: cg must be 0..3");
  gemm_force_cta_group(cg);
  return clear_error();
}

}  // extern "C"

// ---------------------------------------------------------------- kernel-level wrappers
#include <cmath>

#include "kernels/attention.h"
#include "kernels/ops.h"

namespace {
int kstatus(int r, const char* where) {
  if (r == 0) return gptb200::clear_error();
  if (r == 1) return gptb200::set_error(TP_ERR_INVALID, std::string(where) + ": unsupported arguments");
  return gptb200::set_cuda_error(where);
}
gptb200::DropKey dkey(uint64_t seed, int step, int layer, int site, float p, int64_t base) {
  gptb200::DropKey k;
  k.seed = seed, k.step = step, k.layer = layer, k.site = site, k.p = p, k.elem_base = base;
  return k;
}
}  // namespace

extern "C" {

int tp_flash_attn_fwd(int batch, int seq, int heads, int head_dim, const void* qkv, void* out, void* lse,
                      void* stream) {
  return kstatus(flash_attn_fwd({batch, seq, heads, head_dim}, static_cast<const bf16*>(qkv), static_cast<bf16*>(out),
                                static_cast<float*>(lse), static_cast<cudaStream_t>(stream)),
                 "tp_flash_attn_fwd");
}

int tp_flash_attn_bwd(int batch, int seq, int heads, int head_dim, const void* qkv, const void* out, const void* dout,
                      const void* lse, void* D, void* dq_acc, void* dqkv, void* stream) {
  return kstatus(flash_attn_bwd({batch, seq, heads, head_dim}, static_cast<const bf16*>(qkv),
                                static_cast<const bf16*>(out), static_cast<const bf16*>(dout),
                                static_cast<const float*>(lse), static_cast<float*>(D), static_cast<float*>(dq_acc),
                                static_cast<bf16*>(dqkv), static_cast<cudaStream_t>(stream)),
                 "tp_flash_attn_bwd");
}

int tp_resid_layernorm_fwd(int rows, int d, const void* y, const void* bias, const void* resid, void* h_out,
                           const void* gamma, const void* beta, void* ln_out, void* mean, void* rstd, uint64_t seed,
                           int step, int layer, int site, float p, int64_t elem_base, void* stream) {
  ResidLnArgs a;
  a.rows = rows, a.d = d, a.seq = rows;
  a.y = static_cast<const bf16*>(y), a.bias = static_cast<const bf16*>(bias), a.resid = static_cast<const bf16*>(resid);
  a.drop = dkey(seed, step, layer, site, p, elem_base);
  a.h_out = static_cast<bf16*>(h_out);
  a.gamma = static_cast<const bf16*>(gamma), a.beta = static_cast<const bf16*>(beta);
  a.ln_out = static_cast<bf16*>(ln_out), a.mean = static_cast<float*>(mean), a.rstd = static_cast<float*>(rstd);
  return kstatus(resid_ln_fwd(a, static_cast<cudaStream_t>(stream)), "tp_resid_layernorm_fwd");
}

int tp_layernorm_bwd(int rows, int d, const void* x, const void* dy, const void* resid_grad, const void* gamma,
                     const void* mean, const void* rstd, void* dx, void* dxd, void* dgamma, void* dbeta, void* dbias,
                     uint64_t seed, int step, int layer, int site, float p, int64_t elem_base, void* workspace,
                     void* stream) {
  LnBwdArgs a;
  a.rows = rows, a.d = d;
  a.x = static_cast<const bf16*>(x), a.dy = static_cast<const bf16*>(dy);
  a.resid_grad = static_cast<const bf16*>(resid_grad), a.gamma = static_cast<const bf16*>(gamma);
  a.mean = static_cast<const float*>(mean), a.rstd = static_cast<const float*>(rstd);
  a.dx = static_cast<bf16*>(dx), a.dxd = static_cast<bf16*>(dxd);
  a.drop = dkey(seed, step, layer, site, p, elem_base);
  a.dgamma = static_cast<float*>(dgamma), a.dbeta = static_cast<float*>(dbeta), a.dbias = static_cast<float*>(dbias);
  a.workspace = static_cast<float*>(workspace);
  return kstatus(ln_bwd(a, static_cast<cudaStream_t>(stream)), "tp_layernorm_bwd");
}

size_t tp_layernorm_bwd_workspace_bytes(int rows, int d) { return ln_bwd_workspace_floats(rows, d) * sizeof(float); }

int tp_cross_entropy(int rows, int vocab, void* logits, const int32_t* labels, float scale, void* row_loss, void* stats,
                     void* stream) {
  auto st = static_cast<cudaStream_t>(stream);
  int r = xent_stats(static_cast<const bf16*>(logits), rows, vocab, labels, 0, static_cast<float*>(stats), st);
  if (r == 0)
    r = xent_finish(static_cast<bf16*>(logits), rows, vocab, labels, 0, static_cast<const float*>(stats), 1, scale,
                    static_cast<float*>(row_loss), st);
  return kstatus(r, "tp_cross_entropy");
}

int tp_adam_step(int64_t n, void* master, void* m, void* v, const void* grad, void* param_bf16, float lr, float beta1,
                 float beta2, float eps, float weight_decay, int step, void* stream) {
  AdamArgs a;
  a.n = n, a.master = static_cast<float*>(master), a.m = static_cast<float*>(m), a.v = static_cast<float*>(v);
  a.grad = static_cast<const float*>(grad), a.param = static_cast<bf16*>(param_bf16);
  a.lr = lr, a.beta1 = beta1, a.beta2 = beta2, a.eps = eps, a.weight_decay = weight_decay;
  a.bc1 = static_cast<float>(1.0 - std::pow(static_cast<double>(beta1), step));
  a.bc2 = static_cast<float>(1.0 - std::pow(static_cast<double>(beta2), step));
  return kstatus(adam_step(a, static_cast<cudaStream_t>(stream)), "tp_adam_step");
}

}  // extern "C"
