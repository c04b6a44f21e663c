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

namespace gptb200 {

struct NvlsContext;

// Collective over the TP communicator. Returns nullptr (and leaves NCCL state clean) when the
// TP group is not one NVLink/multicast domain; the caller then uses ncclAllReduce.
NvlsContext* nvls_create(ncclComm_t tp_comm, size_t bytes, int max_ctas);
void nvls_destroy(NvlsContext* ctx, ncclComm_t tp_comm);
void* nvls_base(const NvlsContext* ctx);
size_t nvls_bytes(const NvlsContext* ctx);
// In-place sum of n bf16 over the TP group; buf must lie inside the window, n % (8*tp) == 0.
// Returns 0, or 1 for bad arguments, 2 for a launch error.
int nvls_allreduce_bf16(NvlsContext* ctx, void* buf, size_t n, cudaStream_t st, int ctas = 0);

}  // namespace gptb200
