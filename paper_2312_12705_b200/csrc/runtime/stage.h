// One rank's share of the GPT train step: its pipeline stage's layers, TP-sharded, with the
// ZeRO-1 optimizer shard of its DP group. Executes what trainplan::estimate() models
// (/root/reference/proj/src/perf.cpp:36-122) on sm_100a kernels + NCCL.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "kernels/ops.h"
#include "runtime/comm.h"
#include "runtime/pipe_exec.h"
#include "trainplan/core.hpp"

namespace gptb200 {

struct TrainOptions {
  uint64_t seed = 1234;  // init + dropout key
  float dropout = 0.f;   // hidden dropout (embedding, attention-out, mlp-out)
  float lr = 1e-4f, beta1 = 0.9f, beta2 = 0.95f, eps = 1e-8f, weight_decay = 0.f;
};

struct StepError {
  int code;
  std::string msg;
};

// Local shard of one global parameter tensor inside the stage's flat buffers.
struct ParamSlot {
  int tensor_id = 0;
  int64_t rows = 0, cols = 0, offset = 0;
  int64_t rseg = 1, rstride = 0, roff = 0, coff = 0, gcols = 1;  // local -> global index map
  float stddev = 0.f, constant = 0.f;
};

// Per-layer tensors kept for backward (or recomputed under activation checkpointing).
struct LayerActs {
  bf16 *a = nullptr, *qkv = nullptr, *o = nullptr, *hmid = nullptr, *m2 = nullptr, *u = nullptr,
       *g = nullptr;
  float *mu1 = nullptr, *rs1 = nullptr, *mu2 = nullptr, *rs2 = nullptr, *lse = nullptr;
};

// Kernel classes for the live per-launch timing (CUDA events on the step stream).
enum KernelClass { K_GEMM = 0, K_ATTN_FWD, K_ATTN_BWD, K_NORM, K_ELEM, K_COMM_TP, K_COMM_PP, K_COMM_DP, K_ADAM, K_NUM };

struct KernelTimes {
  double ms[K_NUM] = {};
  long launches[K_NUM] = {};
  double flops[K_NUM] = {};  // algorithmic FLOPs (GEMM 2MNK; attention causal)
  double bytes[K_NUM] = {};  // algorithmic HBM bytes (norm / elementwise / Adam)
};

// ZeRO-1 bucket: a contiguous range of the flat buffers (padded to a multiple of 64*dp); DP rank
// d owns [off + d*len/dp, off + (d+1)*len/dp), stored in the master/m/v shard at master_off.
struct Bucket {
  int64_t off = 0, len = 0, master_off = 0;
};

// Device-memory categories of the session (MemoryReport, /root/reference/proj/include/trainplan/
// memory.hpp:47-55): parameters = bf16 working copy + fp32 master shard, gradients = fp32 main grads,
// optimizer = Adam m + v shards, activations = everything kept or recomputed per microbatch,
// workspace = per-op scratch (the reference's framework overhead).
enum MemCategory { MEM_PARAMS = 0, MEM_GRADS, MEM_OPTIMIZER, MEM_ACTIVATIONS, MEM_WORKSPACE, MEM_NUM };

struct StepTimes {  // milliseconds of the last step on this rank (CUDA events)
  float total = 0, tp_comm = 0, pp_comm = 0, dp_comm = 0, optimizer = 0;
};

class Stage {
 public:
  Stage(const trainplan::ModelSpec& model, const trainplan::ParallelConfig& resolved,
        const TrainOptions& opts, int rank, int world, int device, const void* nccl_id);
  ~Stage();
  Stage(const Stage&) = delete;
  Stage& operator=(const Stage&) = delete;

  void init_params();
  // Global batch tokens [gbs, s+1] (inputs = [:, :s], labels = [:, 1:]); host or device src.
  void upload_tokens(const int32_t* src, int64_t n, bool src_on_device);
  // One iteration: zero grads, 1F1B over the microbatches, tied-embedding + DP reductions,
  // ZeRO-1 Adam, parameter allgather. Loss stays on device (read_loss).
  void step();
  float read_loss();  // mean CE of the last step over the global batch (blocking)
  void sync();
  void barrier();

  const ParamSlot* slot(int tensor_id) const;
  // which: 0 = working bf16 param, 1 = fp32 grad (accumulated this step), 2 = fp32 master
  // (dp must be 1 or the tensor must lie in this rank's ZeRO shard), 3 = Adam m, 4 = Adam v.
  void read_tensor(int which, int tensor_id, float* host) const;
  void read_flat(int which, int64_t offset, int64_t n, float* host) const;
  // Forward-only loss of the uploaded batch with the current parameters (no update).
  float eval_loss();

  const std::vector<Bucket>& buckets() const { return buckets_; }
  int64_t flat_params() const { return P_; }
  int64_t shard_params() const { return shard_; }
  size_t device_bytes() const { return dev_bytes_; }
  // Bytes per MemCategory (HBM allocations plus buffers carved from the NVLS window) and the window.
  size_t category_bytes(int c) const { return cat_bytes_[c]; }
  size_t window_bytes() const { return window_bytes_; }
  // ZeRO stage in effect: 1 = optimizer state sharded over DP (reduce-scatter + allgather),
  // 0 = replicated (gradient allreduce, every rank updates every parameter).
  int zero_stage() const { return zero_; }
  // This rank's optimizer range of bucket b: flat offset and length.
  int64_t own_offset(const Bucket& b) const { return zero_ ? b.off + comms_.me.d * (b.len / cfg_.dp) : b.off; }
  int64_t own_len(const Bucket& b) const { return zero_ ? b.len / cfg_.dp : b.len; }
  // Watchdog: host waits on the session's streams give up after `seconds` (<= 0: wait forever),
  // abort the NCCL communicators and throw TP_ERR_TIMEOUT; the session is unusable afterwards.
  void set_timeout(double seconds) { timeout_s_ = seconds; }
  bool poisoned() const { return poisoned_; }
  StepTimes last_times() const { return times_; }
  int microbatches() const { return m_; }
  int kernel_launches_per_step() const { return launches_; }
  // Runs `steps` iterations bracketed by CUDA events on the step stream; returns device ms.
  // With profile, every launch is bracketed too and summed per KernelClass into *kt.
  float time_steps(int steps, bool profile, KernelTimes* kt);
  // Device ms of each step of the last time_steps call (events between consecutive steps).
  const std::vector<float>& step_times() const { return step_ms_; }
  float allreduce_max(float v);
  // TP allreduce of the [M, d] bf16 activation buffer (test / microbenchmark hooks).
  // mode 0 = automatic (NVLS when available), 1 = ncclAllReduce. in/out: M*d bf16 bit patterns.
  void debug_tp_allreduce(const uint16_t* in, uint16_t* out, int mode);
  float bench_tp_allreduce(int iters, int mode, int ctas);
  // Average device ms of one sequence-parallel LayerNorm kernel on this session's buffers
  // (mode 0: forward reduce-scatter + LN + allgather, 1: backward), back to back (microbenchmark).
  float bench_sp(int iters, int mode);
  bool tp_uses_nvls() const { return comms_.tp_nvls != nullptr; }
  // 0: no TP; 1: ncclAllReduce; 2: NVLS allreduce kernel; 3: sequence parallel (fused NVLS norms)
  int tp_mode() const { return cfg_.tp == 1 ? 0 : (sp_ ? 3 : (comms_.tp_nvls ? 2 : 1)); }

 private:
  struct LayerW {
    const bf16 *ln1g, *ln1b, *wqkv, *bqkv, *wo, *bo, *ln2g, *ln2b, *w1, *b1, *w2, *b2;
  };
  struct LayerG {
    float *ln1g, *ln1b, *wqkv, *bqkv, *wo, *bo, *ln2g, *ln2b, *w1, *b1, *w2, *b2;
  };
  struct Slot {
    std::vector<bf16*> h;         // Ll+1 residual-stream tensors [M, d]
    std::vector<LayerActs> acts;  // per layer (empty under checkpointing)
    int32_t* inputs = nullptr;    // [M]
    int32_t* labels = nullptr;    // [M]
  };

  void* alloc(size_t bytes, int cat = MEM_WORKSPACE);
  void wait(cudaStream_t st, const char* what);
  void build_layout();
  void allocate();
  LayerW w(int l) const;
  LayerG gr(int l) const;
  LayerActs& acts_for(int slot, int l);

  // One pipeline op on chunk c (layers [c*Lc, (c+1)*Lc) of this device; virtual stage c*pp + p).
  void forward_op(int mb, int c, int slot, bool head_now);
  void backward_op(int mb, int c, int slot, bf16* dh, bool head_late);
  void layer_fwd(int li, LayerActs& A, const bf16* hin, bf16* hout, int slot);
  void layer_recompute(int l, LayerActs& A, const bf16* hin);
  void layer_bwd(int l, LayerActs& A, const bf16* hin, bf16* dh, bf16* dy2);
  void head_and_loss(int slot);
  void final_ln(const bf16* h);  // final LayerNorm of the last virtual stage into hf_/muf_/rsf_
  void head_bwd(bf16* dh_out);
  void adam_bucket(int bucket, cudaStream_t st);
  void grads_ready(int bucket);  // last microbatch's grads of `bucket` final: start its reduce-scatter
  void prepare_tokens(int mb, int slot);
  void run_action(const PipeAction& a);
  void pp_recv(void* buf, int dir);
  void pp_send(const void* buf, int dir, cudaEvent_t done);
  void join_sends();

  void gemm_fwd(const bf16* X, const bf16* W, const bf16* bias, bf16* Y, int M, int N, int K, int epi = 0,
                bf16* C2 = nullptr);
  void gemm_dgrad(const bf16* dY, const bf16* W, bf16* dX, int M, int N, int K, int epi = 0,
                  const bf16* aux = nullptr, const bf16* rowdot_b = nullptr, float* colsum_part = nullptr);
  void gemm_wgrad(const bf16* dY, const bf16* X, float* dW, int M, int N, int K);
  void ck(int status, const char* what);
  friend struct KScope;
  struct KScope {  // brackets the enclosed launches on `stream` (default: the step stream)
    Stage* s;
    int k;
    size_t idx;
    cudaStream_t stream;
    KScope(Stage* st, int kind, double flops = 0, double bytes = 0, cudaStream_t on = nullptr);
    ~KScope();
  };
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pool_;
  std::vector<int> ev_kind_;
  size_t ev_used_ = 0;
  bool profile_ = false;
  KernelTimes prof_acc_;
  void tp_allreduce(bf16* buf);
  int64_t woff(const void* p) const;  // window offset of an SP buffer (throws when outside)
  void sp_fwd(const SpLnFwdArgs& a);
  void sp_bwd(const SpLnBwdArgs& a);
  template <typename F>
  void sp_bwd_overlapped(const SpLnBwdArgs& a, F&& independent);
  cudaStream_t sp_st_ = nullptr;
  cudaEvent_t sp_fork_ = nullptr, sp_join_ = nullptr;
  // recompute prefetch (SP + checkpointing): see backward_op / RecomputeOnSide
  bool rc_overlap_ = false;
  LayerActs scratch2_;
  bf16* rc_tmp_ = nullptr;
  cudaStream_t rc_st_ = nullptr;
  cudaEvent_t rc_fork_ = nullptr, rc_done_[2] = {nullptr, nullptr};
  int sp_lane_set_ = 0;
  struct RecomputeOnSide {
    Stage* s;
    cudaStream_t st;
    bf16* tmp;
    explicit RecomputeOnSide(Stage* st);
    ~RecomputeOnSide();
  };
  friend struct RecomputeOnSide;
  int64_t slot_offset(int tid) const { return slot(tid)->offset; }

  trainplan::ModelSpec model_;
  trainplan::ParallelConfig cfg_;
  TrainOptions opts_;
  Comms comms_;
  int device_ = 0;
  cudaStream_t st_ = nullptr;
  std::vector<void*> allocations_;
  size_t dev_bytes_ = 0;
  size_t cat_bytes_[MEM_NUM] = {};
  size_t window_bytes_ = 0;
  int zero_ = 1;
  double timeout_s_ = 0.0;
  bool poisoned_ = false;

  // shape
  // Ll_ local layers = v_ chunks of Lc_ layers; local layer li is global layer glayer(li).
  int glayer(int li) const { return ((li / Lc_) * cfg_.pp + comms_.me.p) * Lc_ + li % Lc_; }
  bool first_vs(int c) const { return first_ && c == 0; }
  bool last_vs(int c) const { return last_ && c == v_ - 1; }
  int L_ = 0, Ll_ = 0, Lc_ = 0, v_ = 1, d_ = 0, dt_ = 0, ht_ = 0, hd_ = 0, V_ = 0, Vt_ = 0, s_ = 0;
  int mbs_ = 1, M_ = 0, m_ = 1, nslots_ = 1;
  // Sequence parallelism (tp > 1 with an NVLS window): this rank owns rows [row0_, row0_ + Ms_)
  // of every [M, d] residual-stream tensor; LayerNorms run on those rows fused with the TP
  // reduce-scatter / allgather (kernels/tp_nvls.h). Without SP, Ms_ == M_ and row0_ == 0.
  bool sp_ = false;
  int Ms_ = 0, row0_ = 0;
  bool first_ = true, last_ = true, ckpt_ = false;
  int step_no_ = 0;
  int cur_mb_ = 0;
  int launches_ = 0;

  // parameters
  std::vector<ParamSlot> slots_;
  std::vector<int> slot_index_;  // tensor_id -> index in slots_ or -1
  std::vector<Bucket> buckets_;  // [0] = embeddings, then one per local layer (last + final LN)
  std::vector<int> layer_bucket_;
  cudaStream_t comm_st_ = nullptr;
  std::vector<cudaEvent_t> bucket_ev_;
  cudaEvent_t comm_done_ = nullptr;
  bool overlap_rs_ = false, in_last_bwd_ = false;
  int64_t P_ = 0, shard_ = 0;
  bf16* params_ = nullptr;
  float *grads_ = nullptr, *master_ = nullptr, *adam_m_ = nullptr, *adam_v_ = nullptr;

  // activations / workspaces
  std::vector<Slot> slots_act_;
  LayerActs scratch_;  // checkpointing recompute buffers
  int32_t* tokens_ = nullptr;
  // pipeline p2p: sends on one side stream per direction, buffer-reuse events
  cudaStream_t send_st_[2] = {nullptr, nullptr};
  cudaEvent_t op_ev_ = nullptr, send_done_ev_[2] = {nullptr, nullptr};
  std::vector<cudaEvent_t> slot_send_ev_;
  cudaEvent_t dh_send_ev_[kDhRing] = {};
  std::vector<PipeAction> plan_, eval_plan_;
  bf16* dh_[kDhRing] = {};
  bf16 *tmp_md_ = nullptr, *dy_ = nullptr, *du_ = nullptr, *dm_ = nullptr,
       *do_ = nullptr, *dqkv_ = nullptr;
  float *attn_D_ = nullptr, *dq_acc_ = nullptr, *ws_ = nullptr;
  float* colpart_ = nullptr;  // [M/32][4d/t] column partials of the dGeLU dgrad (fc1 bias grad)
  bf16* hf_ = nullptr;
  float *muf_ = nullptr, *rsf_ = nullptr;
  bf16* logits_ = nullptr;
  float2* rowstat_ = nullptr;  // [M][Vt/64] (max, sum exp) partials of the LM-head epilogue
  float *xstats_ = nullptr, *xall_ = nullptr, *row_loss_ = nullptr, *loss_acc_ = nullptr;
  StepTimes times_;
  std::vector<float> step_ms_;
};

}  // namespace gptb200
