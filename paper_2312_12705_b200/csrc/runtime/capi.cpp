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

}  // extern "C"
