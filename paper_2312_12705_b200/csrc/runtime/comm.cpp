#include "runtime/comm.h"

#include "trainplan/capi.h"

namespace gptb200 {

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw CommError{TP_ERR_NCCL, std::string(what) + ": " + ncclGetErrorString(r)};
}

void Comms::abort() {
  if (aborted) return;
  aborted = true;
  tp_nvls = nullptr;
  for (ncclComm_t& c : links_in_order) ncclCommAbort(c);
  links_in_order.clear();
  link_send[0] = link_send[1] = link_recv[0] = link_recv[1] = nullptr;
  for (ncclComm_t* c : {&emb_comm, &dp_comm, &tp_comm, &world_comm})
    if (*c) {
      ncclCommAbort(*c);
      *c = nullptr;
    }
}

Comms::~Comms() {
  if (aborted) return;
  if (tp_nvls) {
    nvls_destroy(tp_nvls, tp_comm);
    tp_nvls = nullptr;
  }
  // ncclCommDestroy synchronises with the peers: destroy in creation order on every rank
  for (ncclComm_t& c : links_in_order) ncclCommDestroy(c);
  links_in_order.clear();
  for (ncclComm_t* c : {&emb_comm, &dp_comm, &tp_comm, &world_comm})
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
  if (pp > 1) {
    for (int dir = 0; dir < 2; ++dir)
      for (int k = 0; k < pp; ++k) {
        const int dst = dir == 0 ? (k + 1) % pp : (k + pp - 1) % pp;
        const bool wrap = dir == 0 ? k == pp - 1 : k == 0;
        if (wrap && cfg.interleave_v == 1) continue;  // same decision on every rank
        ncclComm_t unused = nullptr;
        ncclComm_t* out = me.p == k ? &link_send[dir] : (me.p == dst ? &link_recv[dir] : &unused);
        const bool member = me.p == k || me.p == dst;
        split(member ? me.t + tp * me.d : NCCL_SPLIT_NOCOLOR, me.p == k ? 0 : 1, out, "split pipeline link");
        if (member) links_in_order.push_back(*out);
      }
  }
  split(me.t + tp * me.p, me.d, &dp_comm, "split dp");
  const bool edge = pp > 1 && (me.p == 0 || me.p == pp - 1);
  split(edge ? me.t + tp * me.d : NCCL_SPLIT_NOCOLOR, me.p, &emb_comm, "split emb");
}

void* Comms::init_tp_symmetric(size_t bytes) {
  if (tp == 1) return nullptr;
  tp_nvls = nvls_create(tp_comm, bytes, 148);
  return nvls_base(tp_nvls);
}

void Comms::tp_allreduce_bf16(void* buf, size_t n, cudaStream_t st, int mode) const {
  if (tp == 1) return;
  if (mode == 0 && tp_nvls) {
    const int r = nvls_allreduce_bf16(tp_nvls, buf, n, st, tp_nvls_ctas);
    if (r == 0) return;
    if (r == 2) throw CommError{TP_ERR_CUDA, "NVLS allreduce launch failed"};
    // r == 1: buffer outside the window -> NCCL
  }
  nccl_check(ncclAllReduce(buf, buf, n, ncclBfloat16, ncclSum, tp_comm, st), "tp allreduce");
}

void Comms::tp_allreduce_f32_group(const std::vector<std::pair<float*, size_t>>& parts, cudaStream_t st) const {
  if (tp == 1 || parts.empty()) return;
  nccl_check(ncclGroupStart(), "group start");
  for (const auto& p : parts) nccl_check(ncclAllReduce(p.first, p.first, p.second, ncclFloat, ncclSum, tp_comm, st), "tp allreduce f32");
  nccl_check(ncclGroupEnd(), "group end");
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

void Comms::dp_allreduce_f32(float* buf, size_t n, cudaStream_t st) const {
  if (dp == 1) return;
  nccl_check(ncclAllReduce(buf, buf, n, ncclFloat, ncclSum, dp_comm, st), "dp allreduce");
}

void Comms::emb_allreduce_f32(float* buf, size_t n, cudaStream_t st) const {
  if (!emb_comm) return;
  nccl_check(ncclAllReduce(buf, buf, n, ncclFloat, ncclSum, emb_comm, st), "embedding allreduce");
}

void Comms::world_allreduce_f32(float* buf, size_t n, cudaStream_t st) const {
  if (world == 1) return;
  nccl_check(ncclAllReduce(buf, buf, n, ncclFloat, ncclSum, world_comm, st), "world allreduce");
}

void Comms::pp_send(const void* buf, size_t n, int dir, cudaStream_t st) const {
  if (!link_send[dir]) throw CommError{TP_ERR_INVALID, "pipeline send on a missing link"};
  nccl_check(ncclSend(buf, n, ncclBfloat16, 1, link_send[dir], st), "pp send");
}

void Comms::pp_recv(void* buf, size_t n, int dir, cudaStream_t st) const {
  if (!link_recv[dir]) throw CommError{TP_ERR_INVALID, "pipeline recv on a missing link"};
  nccl_check(ncclRecv(buf, n, ncclBfloat16, 0, link_recv[dir], st), "pp recv");
}

}  // namespace gptb200
