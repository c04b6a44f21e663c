#include "runtime/comm.h"

#include "trainplan/capi.h"

namespace gptb200 {

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw CommError{TP_ERR_NCCL, std::string(what) + ": " + ncclGetErrorString(r)};
}

Comms::~Comms() {
  for (ncclComm_t* c : {&emb_comm, &dp_comm, &pp_comm, &tp_comm, &world_comm})
    if (*c) {
      ncclCommDestroy(*c);
      *c = nullptr;
    }
}

void Comms::init(const trainplan::ParallelConfig& cfg, int rank_, int world_, const ncclUniqueId* id) {
  rank = rank_;
  world = world_;
  tp = cfg.tp;
  pp = cfg.pp;
  dp = cfg.dp;
  me = trainplan::rank_coords(rank, cfg);
  if (world == 1) return;
  nccl_check(ncclCommInitRank(&world_comm, world, *id, rank), "ncclCommInitRank");
  auto split = [&](int color, int key, ncclComm_t* out, const char* what) {
    nccl_check(ncclCommSplit(world_comm, color, key, out, nullptr), what);
  };
  split(me.p + pp * me.d, me.t, &tp_comm, "split tp");
  split(me.t + tp * me.d, me.p, &pp_comm, "split pp");
  split(me.t + tp * me.p, me.d, &dp_comm, "split dp");
  const bool edge = pp > 1 && (me.p == 0 || me.p == pp - 1);
  split(edge ? me.t + tp * me.d : NCCL_SPLIT_NOCOLOR, me.p, &emb_comm, "split emb");
}

void Comms::tp_allreduce_bf16(void* buf, size_t n, cudaStream_t st) const {
  if (tp == 1) return;
  nccl_check(ncclAllReduce(buf, buf, n, ncclBfloat16, ncclSum, tp_comm, st), "tp allreduce");
}

void Comms::tp_allgather_f32(const float* send, float* recv, size_t n, cudaStream_t st) const {
  if (tp == 1) {
    if (send != recv) cudaMemcpyAsync(recv, send, n * sizeof(float), cudaMemcpyDeviceToDevice, st);
    return;
  }
  nccl_check(ncclAllGather(send, recv, n, ncclFloat, tp_comm, st), "tp allgather");
}

void Comms::dp_reduce_scatter_f32(float* buf, size_t n, cudaStream_t st) const {
  if (dp == 1) return;
  nccl_check(ncclReduceScatter(buf, buf + static_cast<size_t>(me.d) * n, n, ncclFloat, ncclSum, dp_comm, st),
             "dp reduce-scatter");
}

void Comms::dp_allgather_bf16(void* buf, size_t n, cudaStream_t st) const {
  if (dp == 1) return;
  auto* b = static_cast<uint16_t*>(buf);
  nccl_check(ncclAllGather(b + static_cast<size_t>(me.d) * n, b, n, ncclBfloat16, dp_comm, st), "dp allgather");
}

void Comms::emb_allreduce_f32(float* buf, size_t n, cudaStream_t st) const {
  if (!emb_comm) return;
  nccl_check(ncclAllReduce(buf, buf, n, ncclFloat, ncclSum, emb_comm, st), "embedding allreduce");
}

void Comms::world_allreduce_f32(float* buf, size_t n, cudaStream_t st) const {
  if (world == 1) return;
  nccl_check(ncclAllReduce(buf, buf, n, ncclFloat, ncclSum, world_comm, st), "world allreduce");
}

void Comms::pp_exchange(const void* send, int send_peer, void* recv, int recv_peer, size_t n,
                        cudaStream_t st) const {
  if (pp == 1 || (!send && !recv)) return;
  nccl_check(ncclGroupStart(), "group start");
  if (send) nccl_check(ncclSend(send, n, ncclBfloat16, send_peer, pp_comm, st), "pp send");
  if (recv) nccl_check(ncclRecv(recv, n, ncclBfloat16, recv_peer, pp_comm, st), "pp recv");
  nccl_check(ncclGroupEnd(), "group end");
}

}  // namespace gptb200
