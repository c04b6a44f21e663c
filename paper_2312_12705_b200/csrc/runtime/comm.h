// NCCL communicators of one rank: world, then TP / PP / DP / embedding-tie groups split with
// the reference's rank layout rank = t + tp*(p + pp*d) (proj/src/perf.cpp:15-20). These are the
// real collectives behind the reference's cost calls (perf.cpp:62-102, cluster.cpp:81-110).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <string>
#include <utility>
#include <vector>

#include "kernels/tp_nvls.h"
#include "trainplan/core.hpp"

namespace gptb200 {

struct CommError {
  int code;  // TP_ERR_*
  std::string msg;
};

class Comms {
 public:
  Comms() = default;
  ~Comms();
  Comms(const Comms&) = delete;
  Comms& operator=(const Comms&) = delete;

  // world_size == 1 creates no NCCL communicators at all.
  void init(const trainplan::ParallelConfig& cfg, int rank, int world, const ncclUniqueId* id);
  // Watchdog path: ncclCommAbort every communicator (no peer synchronisation, so it returns even
  // when a peer is dead or stuck); the NVLS window is leaked (its device state may be in use by a
  // kernel that never finishes). The process should exit afterwards.
  void abort();
  bool aborted = false;

  int rank = 0, world = 1;
  trainplan::RankCoords me;
  int tp = 1, pp = 1, dp = 1;
  ncclComm_t world_comm = nullptr;
  ncclComm_t tp_comm = nullptr;   // ranks sharing (p, d), ordered by t
  // Pipeline ring links, one 2-rank communicator per (link, direction) so every FIFO carries one
  // kind of message and is driven from one stream: [0] activations p -> p+1, [1] gradients p -> p-1
  // (mod pp; the wrap links pp-1 -> 0 / 0 -> pp-1 exist only for interleaved schedules).
  ncclComm_t link_send[2] = {nullptr, nullptr};
  ncclComm_t link_recv[2] = {nullptr, nullptr};
  std::vector<ncclComm_t> links_in_order;  // creation order (identical on all ranks) for teardown
  ncclComm_t dp_comm = nullptr;   // ranks sharing (t, p), ordered by d
  ncclComm_t emb_comm = nullptr;  // first & last stage of (t, d) when pp > 1 (tied embedding)

  // NVLS symmetric window on the TP communicator (tp > 1 and one multicast domain); buffers
  // carved from it are allreduced by the in-switch reduction kernel, others by ncclAllReduce.
  NvlsContext* tp_nvls = nullptr;
  void* init_tp_symmetric(size_t bytes);  // collective over TP; returns the window base or nullptr
  int tp_nvls_ctas = 0;                    // 0 = default grid

  // Collectives on `st` (no-ops for singleton groups). Throw CommError on failure.
  // mode: 0 = automatic (NVLS kernel when buf is in the window), 1 = force ncclAllReduce.
  void tp_allreduce_bf16(void* buf, size_t n, cudaStream_t st, int mode = 0) const;
  // Sum each (buffer, count) over TP in one ncclGroup.
  void tp_allreduce_f32_group(const std::vector<std::pair<float*, size_t>>& parts, cudaStream_t st) const;
  void tp_allgather_f32(const float* send, float* recv, size_t n_per_rank, cudaStream_t st) const;
  void dp_reduce_scatter_f32(float* buf, size_t n_per_rank, cudaStream_t st) const;  // in place
  void dp_allgather_bf16(void* buf, size_t n_per_rank, cudaStream_t st) const;       // in place
  void dp_allreduce_f32(float* buf, size_t n, cudaStream_t st) const;                 // ZeRO-0
  void emb_allreduce_f32(float* buf, size_t n, cudaStream_t st) const;
  void world_allreduce_f32(float* buf, size_t n, cudaStream_t st) const;
  // Pipeline p2p over the ring links: dir 0 = activations (to p+1 / from p-1), dir 1 = gradients
  // (to p-1 / from p+1).
  void pp_send(const void* buf, size_t n_bf16, int dir, cudaStream_t st) const;
  void pp_recv(void* buf, size_t n_bf16, int dir, cudaStream_t st) const;
};

void nccl_check(ncclResult_t r, const char* what);

}  // namespace gptb200
