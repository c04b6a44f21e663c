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
 *   - A session is bound to one host thread and one GPU (one process per GPU is the supported
 *     layout). Per-kernel attributes and SM counts are cached per device (thread-safe), so sessions
 *     on different GPUs of one process also work; the launch-variant counters and the GEMM
 *     tile-choice test hook (tp_gemm_force_cta_group) are process-wide.
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
#define TP_ERR_TIMEOUT 7 /* watchdog: a host wait exceeded the session timeout; communicators aborted */

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
/* Executable per-device plan Stage::step() runs for that order (runtime/pipe_exec.h): 6 ints per
 * action = {kind 0 fwd / 1 bwd, microbatch, chunk, activation slot, gradient buffer, flags}
 * (flags: 1 recv input, 2 send output, 4 LM head now, 8 deferred LM head, 16 last microbatch). */
int tp_pipeline_actions(int p, int m, int v, int device, int dh_ring, int forward_only, int* out, int cap, int* n);
/* Rank layout (perf.cpp:15-20): rank = t + tp*(p + pp*d). out = {t, p, d}. */
int tp_rank_coords(int rank, int tp, int pp, int dp, int out[3]);

/* ------------------------------------------------------------------ hardware counters
 * trainplan::parse_ncu_csv + hw_flops (include/trainplan/metrics.hpp), the B200 replacement of
 * the reference's parse_counter_csv / hw_flops over AMD SQ_INSTS_VALU_* counters
 * (proj/src/metrics.cpp:67-117). `text` is `ncu --csv` output (long or --page raw form); only
 * launches whose kernel name contains `kernel_filter` are summed (NULL or "" = all). */
typedef struct tp_hw_counters {
  uint64_t launches;
  uint64_t tensor_utc_bf16, tensor_utc_f16, tensor_hmma_bf16, tensor_hmma_f16; /* ncu math ops */
  uint64_t dram_read_bytes, dram_write_bytes, duration_ns;
  double tensor_flops, simt_flops, hw_flops; /* FLOPs (measured coefficients, metrics.hpp) */
  int num_warnings;                          /* unknown metrics skipped */
} tp_hw_counters;
int tp_ncu_parse_csv(const char* text, size_t len, const char* kernel_filter, tp_hw_counters* out);
/* The --metrics list tp_ncu_parse_csv understands, comma-separated, into buf (NUL-terminated). */
int tp_ncu_metric_list(char* buf, size_t cap);
/* trainplan::diagnose_mbs_mismatch (reference semantics, metrics.cpp:164-185): kind 0 consistent,
 * 1 micro-batch mismatch, 2 unexplained; ratio = model / hardware; message into msg. */
int tp_diagnose_mbs_mismatch(double model_tflops, double hw_tflops, int cfg_mbs, int ds_mbs, int* kind,
                             double* ratio, char* msg, size_t cap);

/* ------------------------------------------------------------------ K1-K4 GEMM
 * C[m,n] = sum_k A(m,k) B(n,k); A(m,k) = A[m*lda+k] (a_mn=0) or A[k*lda+m] (a_mn=1);
 * B(n,k) = B[n*ldb+k] (b_mn=0) or B[k*ldb+n] (b_mn=1). bf16 operands, fp32 accumulation.
 * epi: 0 = bf16 C (+bias), 1 = bf16 C = acc+bias and C2 = gelu_tanh(C),
 *      2 = fp32 C (= or += when accumulate), 3 = bf16 C = acc * gelu_tanh'(aux).
 * Requires M%128 == 0, K%64 == 0, N%64 == 0. */
int tp_gemm_bf16(int M, int N, int K, const void* A, int lda, int a_mn, const void* B, int ldb,
                 int b_mn, void* C, int ldc, int epi, const void* bias, void* C2, const void* aux,
                 int ldaux, int accumulate, void* stream);

/* Test/tuning hook: 0 = automatic GEMM tile choice, 1 = single-CTA 128xN tiles only, 3 = CTA-pair 256x512,
 * 2 = CTA-pair (cta_group::2) 256x256 tiles whenever M, N are multiples of 256. */
int tp_gemm_force_cta_group(int cg);

/* ------------------------------------------------------------------ K5/K6 flash attention
 * Causal; qkv[b*s, 3*heads*hd] (q | k | v heads, bf16) -> out[b*s, heads*hd], lse[b, heads, s]
 * (fp32, log2 units). Backward writes dqkv; workspaces D[b*heads*s], dq_acc[b*s*heads*hd] fp32. */
int tp_flash_attn_fwd(int batch, int seq, int heads, int head_dim, const void* qkv, void* out,
                      void* lse, void* stream);
int tp_flash_attn_bwd(int batch, int seq, int heads, int head_dim, const void* qkv,
                      const void* out, const void* dout, const void* lse, void* D, void* dq_acc,
                      void* dqkv, void* stream);

/* ------------------------------------------------------------------ K7/K9 LayerNorm + residual
 * h = resid + dropout(y + bias) (y may be NULL: h = resid); ln_out = LN(h)*gamma + beta (eps 1e-5)
 * with fp32 mean/rstd. Dropout keyed by (seed, step, layer, site, elem_base + row*d + col). */
int tp_resid_layernorm_fwd(int rows, int d, const void* y, const void* bias, const void* resid,
                           void* h_out, const void* gamma, const void* beta, void* ln_out,
                           void* mean, void* rstd, uint64_t seed, int step, int layer, int site,
                           float p, int64_t elem_base, void* stream);
/* dx = resid_grad + LN'(x; dy); dxd = dropout'(dx); dgamma, dbeta, dbias (+= fp32). */
int tp_layernorm_bwd(int rows, int d, const void* x, const void* dy, const void* resid_grad,
                     const void* gamma, const void* mean, const void* rstd, void* dx, void* dxd,
                     void* dgamma, void* dbeta, void* dbias, uint64_t seed, int step, int layer,
                     int site, float p, int64_t elem_base, void* workspace, void* stream);
size_t tp_layernorm_bwd_workspace_bytes(int rows, int d);

/* ------------------------------------------------------------------ K10 cross entropy (tp=1)
 * In place: logits[rows, V] (bf16) -> scale*(softmax - onehot); row_loss[rows] (fp32).
 * stats workspace: 3*rows floats. */
int tp_cross_entropy(int rows, int vocab, void* logits, const int32_t* labels, float scale,
                     void* row_loss, void* stats, void* stream);

/* ------------------------------------------------------------------ K11 Adam (one shard) */
int tp_adam_step(int64_t n, void* master, void* m, void* v, const void* grad, void* param_bf16,
                 float lr, float beta1, float beta2, float eps, float weight_decay, int step,
                 void* stream);

/* ------------------------------------------------------------------ train-step session
 * One rank of the distributed GPT train step (what trainplan::estimate models, perf.cpp:36-122).
 * Launch one process per GPU; rank 0 calls tp_nccl_unique_id and shares the 128 bytes with the
 * other ranks out of band (file, TCP store). world == 1 needs no id (nccl_id may be NULL). */
typedef struct tp_session tp_session;

typedef struct tp_train_options {
  uint64_t seed;      /* parameter init + dropout key (counter-based; see oracle/gpt_oracle.h) */
  float dropout;      /* hidden dropout p */
  float lr, beta1, beta2, eps, weight_decay; /* Adam with fp32 master weights */
} tp_train_options;

int tp_nccl_unique_id(unsigned char out[128]);
/* Validates (trainplan::validate + kernel constraints) and allocates everything; TP_ERR_INVALID
 * on a bad config, TP_ERR_OOM when it does not fit. */
int tp_session_create(const tp_model_spec* model, const tp_parallel_config* cfg,
                      const tp_train_options* opts, int rank, int world, int device,
                      const unsigned char* nccl_id, tp_session** out);
int tp_session_destroy(tp_session* s);
int tp_session_init_params(tp_session* s);
/* Global batch tokens [gbs][s+1] int32 (host or device pointer). */
int tp_session_upload_tokens(tp_session* s, const int32_t* tokens, int64_t n, int on_device);
/* One iteration on the uploaded tokens (asynchronous; loss stays on device). */
int tp_session_step(tp_session* s);
/* End-to-end iteration: H2D copy of host tokens, step, D2H read of the mean loss. */
int tp_session_train_step(tp_session* s, const int32_t* host_tokens, int64_t n, float* loss_out);
int tp_session_read_loss(tp_session* s, float* loss_out);
/* Forward-only mean loss of the uploaded batch with the current parameters. */
int tp_session_eval_loss(tp_session* s, float* loss_out);
int tp_session_sync(tp_session* s);
int tp_session_barrier(tp_session* s);
/* info = {present, rows, cols, offset, rseg, rstride, roff, coff, gcols}: the local shard of
 * global tensor `tensor_id` (oracle numbering) and its local->global index map. */
int tp_session_tensor_info(tp_session* s, int tensor_id, int64_t info[9]);
/* which: 0 bf16 working param, 1 fp32 grad of the last step, 2 fp32 master, 3 Adam m, 4 Adam v. */
int tp_session_read_tensor(tp_session* s, int which, int tensor_id, float* host_out);
/* Raw read of the rank's flat buffers: which 0 = bf16 params [P], 1 = fp32 grads [P] (after a step
 * only this rank's ZeRO shard [d*P/dp, (d+1)*P/dp) holds DP-reduced values), 2/3/4 = fp32 master /
 * Adam m / Adam v shard [P/dp]. offset and n in elements of that buffer. */
int tp_session_read_flat(tp_session* s, int which, int64_t offset, int64_t n, float* host_out);
/* ZeRO-1 buckets of the flat buffers: triples (flat_offset, length, master_offset); DP rank d owns
 * [flat_offset + d*length/dp, flat_offset + (d+1)*length/dp) of each bucket, stored contiguously
 * in its master/m/v shard at master_offset. Writes up to cap triples; *n = bucket count. */
int tp_session_buckets(tp_session* s, int64_t* out, int cap, int* n);
/* out = {flat_params, shard_params, device_bytes, microbatches, launches_last_step, rank, world, 0} */
/* out = {flat params, ZeRO shard params, device bytes, microbatches, kernel launches per step,
 * rank, world, TP mode (0 none, 1 ncclAllReduce, 2 NVLS allreduce kernel, 3 sequence parallel
 * with the LayerNorms fused with the NVLS reduce-scatter / allgather)}. */
int tp_session_info(tp_session* s, int64_t out[8]);

/* Live timing. Kernel classes: 0 GEMM, 1 attention fwd, 2 attention bwd, 3 LayerNorm/residual,
 * 4 other elementwise, 5 TP comm, 6 PP comm, 7 DP comm, 8 Adam. */
#define TP_KERNEL_CLASSES 9
typedef struct tp_kernel_times {
  double ms[TP_KERNEL_CLASSES];      /* summed launch durations (CUDA events, step stream) */
  int64_t launches[TP_KERNEL_CLASSES];
  double flops[TP_KERNEL_CLASSES];   /* algorithmic FLOPs of those launches */
  double bytes[TP_KERNEL_CLASSES];   /* algorithmic HBM bytes of those launches */
} tp_kernel_times;
/* Runs `steps` iterations on the uploaded tokens between two CUDA events on the session stream;
 * *ms = device time. With profile != 0 every launch is bracketed by events into *kt. */
int tp_session_time_steps(tp_session* s, int steps, int profile, float* ms, tp_kernel_times* kt);
/* Device ms of each step of the last tp_session_time_steps call (CUDA events recorded between
 * consecutive steps on the step stream, no host sync in between): out[0..min(n, steps)). */
int tp_session_step_times(tp_session* s, float* out, int n);
/* Watchdog for every host wait of the session (sync, loss read, timed steps): after `seconds`
 * without progress the session aborts its NCCL communicators (ncclCommAbort) and the call returns
 * TP_ERR_TIMEOUT (trainplan::FailureKind::Timeout, search.hpp:59); the session is unusable
 * afterwards and the process should exit (a kernel spinning on a dead peer cannot be cancelled).
 * seconds <= 0 waits forever. Default: $GPTB200_TIMEOUT_S, else 0. */
int tp_session_set_timeout(tp_session* s, double seconds);

/* Measured per-GPU footprint of the session in the categories of trainplan::MemoryReport
 * (memory.hpp:47-55): params = bf16 working copy + fp32 master (ZeRO shard), gradients = fp32
 * main grads, optimizer = Adam m + v (ZeRO shard), activations = stored / recomputed per-microbatch
 * tensors, workspace = per-op scratch; window = the NVLS symmetric window (TP > 1; the buffers
 * carved from it are also counted in their category); total = all device allocations + window. */
typedef struct tp_memory_report {
  uint64_t params_bytes, gradient_bytes, optimizer_bytes, activation_bytes, workspace_bytes;
  uint64_t window_bytes, total_bytes;
  int zero_stage; /* in effect: 1 sharded optimizer state, 0 replicated */
} tp_memory_report;
int tp_session_memory(tp_session* s, tp_memory_report* out);

/* Process-wide launch-variant counters of the kernel dispatchers (all sessions and devices):
 * 0 GEMM single-CTA tiles, 1 GEMM CTA-pair 256x256, 2 GEMM CTA-pair 256x512, 3 K-sliced fp32
 * GEMM, 4 attention fwd persistent, 5 attention fwd per-block, 6 attention bwd per-block,
 * 7 attention bwd persistent, 8 attention bwd hd 64, 9 attention bwd hd 160, 10 LayerNorm bwd
 * persistent bulk-copy, 11 LayerNorm bwd 32-row fused, 12 LayerNorm bwd two-pass, 13 attention
 * fwd two query tiles per CTA. */
#define TP_KERNEL_VARIANTS 14
int tp_variant_counts(int64_t out[TP_KERNEL_VARIANTS]);
int tp_variant_counts_reset(void);

/* Max over all ranks of *v (NCCL on the world communicator); identity when world == 1. */
int tp_session_allreduce_max(tp_session* s, float* v);
/* TP allreduce of one [mbs*s, d] bf16 activation buffer (the Megatron f/g operator), for tests and
 * microbenchmarks: mode 0 = automatic (NVLS in-switch reduction kernel when the TP group is one
 * multicast domain), 1 = ncclAllReduce. in/out are mbs*s*d bf16 bit patterns on the host. */
int tp_session_debug_tp_allreduce(tp_session* s, const uint16_t* in, uint16_t* out, int mode);
/* Average device ms per allreduce over `iters` (ctas 0 = default grid); *nvls = 1 if the
 * session's TP group uses the NVLS kernel. */
int tp_session_bench_tp_allreduce(tp_session* s, int iters, int mode, int ctas, float* ms, int* nvls);
/* Average device ms of one sequence-parallel LayerNorm kernel (mode 0: NVLS reduce-scatter + LN +
 * allgather forward, 1: backward) on the session's buffers, back to back (TP > 1 with SP only). */
int tp_session_bench_sp(tp_session* s, int iters, int mode, float* ms);

#ifdef __cplusplus
}
#endif

#endif /* TRAINPLAN_CAPI_H_ */
