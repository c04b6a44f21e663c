/* C-ABI of the B200-native GPT train step (libtrainplan_b200.so).
 *
 * This is the drop-in boundary for the path the reference `trainplan` only models:
 * `trainplan::estimate()` (/root/reference/proj/include/trainplan/perf.hpp:42-44,
 * proj/src/perf.cpp:36-122) predicts the GPT decoder train step; the functions below run it.
 * The reference exposes a C++20 library with no FFI, so the C++ API in
 * include/trainplan/train.hpp is the primary binding and this header is the thin layer it
 * (and ctypes / cgo / JNI callers) sit on.
 *
 * Conventions (SURVEY.md §8b "What the B200 build must export"):
 *   - Every entry returns int status: TP_OK (0) or one of the TP_ERR_* codes; the message of
 *     the last failure on the calling thread is available from tp_last_error().
 *   - TP_ERR_INVALID mirrors the reference's std::invalid_argument for invalid configs
 *     (proj/src/perf.cpp:41-44); TP_ERR_OOM is the reported-state OOM (perf.cpp:49-53,
 *     search.hpp:59 FailureKind::Oom).
 *   - Kernel-level entries take device pointers and a cudaStream_t passed as void*; they are
 *     stream-ordered and asynchronous. Session entries own their device memory and streams.
 *   - A session is bound to one host thread and one GPU (one process per GPU).
 */
#ifndef TRAINPLAN_CAPI_H_
#define TRAINPLAN_CAPI_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TP_OK 0
#define TP_ERR_INVALID 1
#define TP_ERR_OOM 2
#define TP_ERR_CUDA 3
#define TP_ERR_NCCL 4
#define TP_ERR_INTERNAL 5
#define TP_ERR_UNSUPPORTED 6

/* Last error message of the calling thread ("" when none). */
const char* tp_last_error(void);
/* ABI version of this library. */
int tp_abi_version(void);

/* ------------------------------------------------------------------ plan (structural)
 * Mirrors of trainplan::ModelSpec (arch.hpp:10-20) and ParallelConfig (memory.hpp:17-32). */
typedef struct tp_model_spec {
  int num_layers, hidden_size, num_heads, vocab_size, seq_length;
} tp_model_spec;

typedef struct tp_parallel_config {
  int tp, pp, dp, mbs, gbs, zero_stage, interleave_v;
  int precision;        /* 0 FP16, 1 BF16, 2 FP32 (trainplan::Precision) */
  int grad_accum_fp32;  /* trainplan::GradAccumDtype::FP32 */
  int checkpoint_activations, flash_attention;
} tp_parallel_config;

typedef struct tp_validation {
  int ok, dp, num_microbatches, num_violations;
  char fields[16][24];
  int hard[16];
  char first_message[256];
} tp_validation;

/* trainplan::param_count (arch.cpp:48-62): out = {attention, ffn, embedding, total_exact,
 * total_approx, executed_total}. */
int tp_param_count(const tp_model_spec* m, uint64_t out[6]);
/* trainplan::model_flops_per_iteration (arch.cpp:64-92). */
int tp_model_flops(const tp_model_spec* m, int64_t batch, int ckpt, int factor, double* out);
/* trainplan::validate (search.cpp:23-84) on a cluster of num_nodes x gpus_per_node; with
 * kernel_checks != 0 the B200 kernel constraints are appended (validate_kernels). */
int tp_validate(const tp_model_spec* m, const tp_parallel_config* c, int num_nodes,
                int gpus_per_node, int kernel_checks, tp_validation* out);
/* Per-device pipeline order (pipesim.cpp:31-91): kind 0 GPipe, 1 1F1B, 2 interleaved. Writes
 * up to cap ops as (backward, microbatch, chunk) triples; *n = op count. */
int tp_pipeline_order(int kind, int p, int m, int v, int device, int* ops, int cap, int* n);
/* Rank layout (perf.cpp:15-20): rank = t + tp*(p + pp*d). out = {t, p, d}. */
int tp_rank_coords(int rank, int tp, int pp, int dp, int out[3]);

/* ------------------------------------------------------------------ K1-K4 GEMM
 * C[m,n] = sum_k A(m,k) B(n,k); A(m,k) = A[m*lda+k] (a_mn=0) or A[k*lda+m] (a_mn=1);
 * B(n,k) = B[n*ldb+k] (b_mn=0) or B[k*ldb+n] (b_mn=1). bf16 operands, fp32 accumulation.
 * epi: 0 = bf16 C (+bias), 1 = bf16 C = acc+bias and C2 = gelu_tanh(C),
 *      2 = fp32 C (= or += when accumulate), 3 = bf16 C = acc * gelu_tanh'(aux).
 * Requires M%128 == 0, K%64 == 0, N%64 == 0. */
int tp_gemm_bf16(int M, int N, int K, const void* A, int lda, int a_mn, const void* B, int ldb,
                 int b_mn, void* C, int ldc, int epi, const void* bias, void* C2, const void* aux,
                 int ldaux, int accumulate, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* TRAINPLAN_CAPI_H_ */
