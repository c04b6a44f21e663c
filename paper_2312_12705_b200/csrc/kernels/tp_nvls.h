// Tensor-parallel allreduce through NVSwitch multicast (NVLS): each rank reduces 1/tp of the
// buffer inside the switch (multimem.ld_reduce, fp32 accumulation) and broadcasts the result to
// every rank's copy (multimem.st). Per-rank NVLink traffic is ~1x the buffer each way, vs 2(tp-1)/tp
// for a ring. The buffer lives in one NCCL symmetric window registered on the TP communicator;
// NCCL 2.28's device API supplies the window / multicast mapping and the cross-GPU barrier, the
// data path is this kernel. Replaces ncclAllReduce for the Megatron f/g operators
// (/root/reference/proj/src/perf.cpp:62-102 models them as 4 allreduces per layer).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstddef>
#include <cstdint>

#include "kernels/ops.h"

namespace gptb200 {

struct NvlsContext;

// Collective over the TP communicator. Returns nullptr (and leaves NCCL state clean) when the
// TP group is not one NVLink/multicast domain; the caller then uses ncclAllReduce.
// The device barriers come in kNvlsBarrierSets sets of max_ctas: kernels that may run concurrently
// on different streams must use different sets (set 0: allreduce / step stream).
constexpr int kNvlsBarrierSets = 2;
NvlsContext* nvls_create(ncclComm_t tp_comm, size_t bytes, int max_ctas);
void nvls_destroy(NvlsContext* ctx, ncclComm_t tp_comm);
void* nvls_base(const NvlsContext* ctx);
size_t nvls_bytes(const NvlsContext* ctx);
// In-place sum of n bf16 over the TP group; buf must lie inside the window, n % (8*tp) == 0.
// Returns 0, or 1 for bad arguments, 2 for a launch error.
int nvls_allreduce_bf16(NvlsContext* ctx, void* buf, size_t n, cudaStream_t st, int ctas = 0);
// Byte offset of p inside the window, -1 when outside.
int64_t nvls_offset(const NvlsContext* ctx, const void* p);

// ---- Sequence-parallel norms fused with their collectives (Megatron-SP, PAPER.md:235-267 split
// of the row-parallel outputs). Rank t owns rows [row0, row0 + nrows) of the [M, d] microbatch
// activation; full-width [M, d] buffers live in the window, per-row state in local shards.
//
// Forward: for each own row R
//   y    = sum over TP ranks of the partial rows P[R]   (multimem.ld_reduce, in-switch; y_off >= 0)
//   h    = resid[R] + dropout(y + bias)                  (resid: own-row shard, or the [s, d]
//                                                          position table indexed R % seq)
//   h_out[R] = h (shard); ln = LN(h)*gamma + beta broadcast to every rank's ln buffer
//   (multimem.st, ln_off >= 0) with mean/rstd stored in the shard.
// y_off < 0: h = resid (pure LayerNorm of the shard, allgathered).
struct SpLnFwdArgs {
  int nrows = 0, row0 = 0, d = 0, seq = 1;
  int lane_set = 0;  // barrier-index set: kernels on different streams use different sets
  int bar_base = 0;  // (set by sp_ln_fwd: lane_set * max CTAs)
  int64_t y_off = -1;
  const bf16* bias = nullptr;
  const bf16* resid = nullptr;  // shard [nrows, d] or position table
  bool resid_pos_table = false;
  DropKey drop;                 // element index = elem_base + R * d + col (same masks as tp = 1)
  bf16* h_out = nullptr;        // shard [nrows, d] (optional)
  const bf16* gamma = nullptr;  // nullptr: no LayerNorm / no allgather
  const bf16* beta = nullptr;
  int64_t ln_off = -1;
  float* mean = nullptr;  // shard [nrows]
  float* rstd = nullptr;
};
int sp_ln_fwd(NvlsContext* ctx, const SpLnFwdArgs& a, cudaStream_t st);

// Backward: for each own row R
//   dy   = sum over TP ranks of P[R] (dy_off >= 0; the reduced row is also written back to this
//          rank's copy of P[R] for the column sums)
//   dx   = resid_grad[R] + LN'(x[R]; dy)  -> dx shard (optional)
//   dxd  = dropout'(dx) broadcast to every rank's buffer at dxd_off (allgather; optional)
// then dgamma/dbeta (+ dbias from dxd) column sums over the own rows (TP-partial: the caller sums
// them over TP once per step).
struct SpLnBwdArgs {
  int nrows = 0, row0 = 0, d = 0;
  int lane_set = 0;
  int bar_base = 0;  // (set by sp_ln_bwd)
  int64_t dy_off = -1;
  const bf16* x = nullptr;  // shard
  const bf16* gamma = nullptr;
  const float* mean = nullptr;
  const float* rstd = nullptr;
  const bf16* resid_grad = nullptr;  // shard (may alias dx)
  bf16* dx = nullptr;                // shard
  DropKey drop;
  int64_t dxd_off = -1;
  float* dgamma = nullptr;
  float* dbeta = nullptr;
  float* dbias = nullptr;
  float* workspace = nullptr;  // >= ln_bwd_workspace_floats(nrows, d)
};
int sp_ln_bwd(NvlsContext* ctx, const SpLnBwdArgs& a, cudaStream_t st);

}  // namespace gptb200
