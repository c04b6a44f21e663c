// NCCL communicators of one rank: world, then TP / PP / DP / embedding-tie groups split with
// the reference's rank layout rank = t + tp*(p + pp*d) (proj/src/perf.cpp:15-20). These are the
// real collectives behind the reference's cost calls (perf.cpp:62-102, cluster.cpp:81-110).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <string>

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

  int rank = 0, world = 1;
  trainplan::RankCoords me;
  int tp = 1, pp = 1, dp = 1;
  ncclComm_t world_comm = nullptr;
  ncclComm_t tp_comm = nullptr;   // ranks sharing (p, d), ordered by t
  ncclComm_t pp_comm = nullptr;   // ranks sharing (t, d), ordered by p
  ncclComm_t dp_comm = nullptr;   // ranks sharing (t, p), ordered by d
  ncclComm_t emb_comm = nullptr;  // first & last stage of (t, d) when pp > 1 (tied embedding)

  // Collectives on `st` (no-ops for singleton groups). Throw CommError on failure.
  void tp_allreduce_bf16(void* buf, size_t n, cudaStream_t st) const;
  void tp_allgather_f32(const float* send, float* recv, size_t n_per_rank, cudaStream_t st) const;
  void dp_reduce_scatter_f32(float* buf, size_t n_per_rank, cudaStream_t st) const;  // in place
  void dp_allgather_bf16(void* buf, size_t n_per_rank, cudaStream_t st) const;       // in place
  void emb_allreduce_f32(float* buf, size_t n, cudaStream_t st) const;
  void world_allreduce_f32(float* buf, size_t n, cudaStream_t st) const;
  // Pipeline p2p inside one ncclGroup: optional send to stage p+dir_send, optional recv.
  void pp_exchange(const void* send, int send_peer_stage, void* recv, int recv_peer_stage,
                   size_t n_bf16, cudaStream_t st) const;
};

void nccl_check(ncclResult_t r, const char* what);

}  // namespace gptb200
