// The per-rank train step. See stage.h; data flow per decoder layer (TP-local sizes,
// M = mbs*s tokens, dt = d/tp):
//   fwd: a=LN1(h) -> qkv=a.Wqkv^T+b -> o=flash(qkv) -> y=o.Wo^T -> TP allreduce ->
//        hmid=h+drop(y+bo), m2=LN2(hmid) -> u=m2.W1^T+b1, g=gelu(u) -> y2=g.W2^T -> TP allreduce
//        -> hout=hmid+drop(y2+b2), next LN fused into the same kernel.
//   bwd: the mirror image; every dgrad GEMM of a column-parallel layer is followed by the TP
//        allreduce of its input gradient (Megatron f/g operators).
#include "runtime/stage.h"

#include <chrono>
#include <cmath>
#include <cstdio>
#include <thread>
#include <cstdlib>
#include <cstring>

#include "kernels/attention.h"
#include "kernels/gemm.h"
#include "trainplan/capi.h"

namespace gptb200 {

using trainplan::PipeOp;
using trainplan::ScheduleKind;

namespace {
constexpr int kPerLayer = 16;  // tensor ids per layer (oracle numbering)
enum LayerTensor { LN1G = 0, LN1B, WQKV, BQKV, WO, BO, LN2G, LN2B, W1, B1, W2, B2 };
constexpr int kEmbedLayer = 0xFFFF;

int64_t align64(int64_t x) { return (x + 63) / 64 * 64; }
}  // namespace

void Stage::ck(int status, const char* what) {
  ++launches_;
  if (status != 0) {
    cudaError_t e = cudaGetLastError();
    throw StepError{e == cudaErrorMemoryAllocation ? TP_ERR_OOM : (status == 1 ? TP_ERR_INVALID : TP_ERR_CUDA),
                    std::string(what) + " failed (status " + std::to_string(status) + ", " +
                        cudaGetErrorString(e) + ")"};
  }
}

Stage::KScope::KScope(Stage* st, int kind, double flops, double bytes, cudaStream_t on)
    : s(st), k(kind), idx(0), stream(on ? on : st->st_) {
  if (!s->profile_) return;
  if (s->ev_used_ == s->ev_pool_.size()) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    s->ev_pool_.push_back({a, b});
    s->ev_kind_.push_back(0);
  }
  idx = s->ev_used_++;
  s->ev_kind_[idx] = kind;
  s->prof_acc_.launches[kind] += 1;
  s->prof_acc_.flops[kind] += flops;
  s->prof_acc_.bytes[kind] += bytes;
  cudaEventRecord(s->ev_pool_[idx].first, stream);
}

Stage::KScope::~KScope() {
  if (!s->profile_) return;
  cudaEventRecord(s->ev_pool_[idx].second, stream);
}

Stage::Stage(const trainplan::ModelSpec& model, const trainplan::ParallelConfig& cfg, const TrainOptions& opts,
             int rank, int world, int device, const void* nccl_id)
    : model_(model), cfg_(cfg), opts_(opts), device_(device) {
  if (cudaSetDevice(device) != cudaSuccess) throw StepError{TP_ERR_CUDA, "cudaSetDevice failed"};
  if (cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking) != cudaSuccess)
    throw StepError{TP_ERR_CUDA, "cudaStreamCreate failed"};
  try {
    comms_.init(cfg, rank, world, static_cast<const ncclUniqueId*>(nccl_id));
  } catch (const CommError& e) {
    throw StepError{e.code, e.msg};
  }
  L_ = model.num_layers;
  d_ = model.hidden_size;
  V_ = model.vocab_size;
  s_ = model.seq_length;
  v_ = std::max(cfg.interleave_v, 1);
  Lc_ = L_ / (cfg.pp * v_);
  Ll_ = Lc_ * v_;
  dt_ = d_ / cfg.tp;
  ht_ = model.num_heads / cfg.tp;
  hd_ = d_ / model.num_heads;
  Vt_ = V_ / cfg.tp;
  mbs_ = cfg.mbs;
  M_ = mbs_ * s_;
  m_ = cfg.num_microbatches();
  first_ = comms_.me.p == 0;
  last_ = comms_.me.p == cfg.pp - 1;
  ckpt_ = cfg.checkpoint_activations;
  zero_ = cfg.zero_stage >= 1 ? 1 : 0;
  if (const char* t = std::getenv("GPTB200_TIMEOUT_S")) timeout_s_ = std::atof(t);
  plan_ = pipeline_actions(cfg.pp, m_, v_, comms_.me.p, kDhRing, false);
  eval_plan_ = pipeline_actions(cfg.pp, m_, v_, comms_.me.p, kDhRing, true);
  nslots_ = pipeline_slots(plan_);
  build_layout();
  allocate();
}

Stage::~Stage() {
  if (poisoned_) return;  // a kernel may still spin on a dead peer: leak rather than hang
  if (st_) cudaStreamSynchronize(st_);
  for (int i = 0; i < 2; ++i)
    if (send_st_[i]) {
      cudaStreamSynchronize(send_st_[i]);
      cudaStreamDestroy(send_st_[i]);
      cudaEventDestroy(send_done_ev_[i]);
    }
  if (rc_st_) {
    cudaStreamSynchronize(rc_st_);
    cudaStreamDestroy(rc_st_);
    cudaEventDestroy(rc_fork_);
    for (auto& e : rc_done_) cudaEventDestroy(e);
  }
  if (sp_st_) {
    cudaStreamSynchronize(sp_st_);
    cudaStreamDestroy(sp_st_);
    cudaEventDestroy(sp_fork_);
    cudaEventDestroy(sp_join_);
  }
  for (auto& e : slot_send_ev_) cudaEventDestroy(e);
  for (auto& e : dh_send_ev_)
    if (e) cudaEventDestroy(e);
  if (op_ev_) cudaEventDestroy(op_ev_);
  if (comm_st_) {
    cudaStreamSynchronize(comm_st_);
    for (auto& e : bucket_ev_) cudaEventDestroy(e);
    cudaEventDestroy(comm_done_);
    cudaStreamDestroy(comm_st_);
  }
  for (auto& e : ev_pool_) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  for (void* p : allocations_) cudaFree(p);
  if (st_) cudaStreamDestroy(st_);
}

void* Stage::alloc(size_t bytes, int cat) {
  void* p = nullptr;
  bytes = (bytes + 255) / 256 * 256;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw StepError{e == cudaErrorMemoryAllocation ? TP_ERR_OOM : TP_ERR_CUDA,
                    "cudaMalloc(" + std::to_string(bytes) + ") failed: " + cudaGetErrorString(e)};
  }
  allocations_.push_back(p);
  dev_bytes_ += bytes;
  cat_bytes_[cat] += bytes;
  return p;
}

// Flat stage-local parameter layout; every tensor starts on a 64-element boundary (TMA and
// 16-byte vector alignment). The local->global index map reproduces Megatron's TP split:
// QKV rows by head within each of q/k/v, fc1 rows, W_o / fc2 columns, vocab rows of wte.
void Stage::build_layout() {
  const int t = comms_.me.t;
  const float std_base = 0.02f;
  const float std_out = static_cast<float>(0.02 / std::sqrt(2.0 * L_));
  int64_t off = 0;
  auto add = [&](int tid, int64_t rows, int64_t cols, int64_t rseg, int64_t rstride, int64_t roff, int64_t coff,
                 int64_t gcols, float sd, float cst) {
    ParamSlot s;
    s.tensor_id = tid;
    s.rows = rows;
    s.cols = cols;
    s.offset = off;
    s.rseg = rseg;
    s.rstride = rstride;
    s.roff = roff;
    s.coff = coff;
    s.gcols = gcols;
    s.stddev = sd;
    s.constant = cst;
    slots_.push_back(s);
    off = align64(off + rows * cols);
  };
  const int64_t d = d_, dt = dt_, Vt = Vt_;
  const int64_t q = static_cast<int64_t>(cfg_.dp) * 64;
  int64_t bucket_start = 0;
  auto close_bucket = [&]() {
    off = (off + q - 1) / q * q;
    Bucket b;
    b.off = bucket_start;
    b.len = off - bucket_start;
    b.master_off = buckets_.empty() ? 0 : buckets_.back().master_off + own_len(buckets_.back());
    buckets_.push_back(b);
    bucket_start = off;
  };
  if (first_ || last_) add(0, Vt, d, Vt, 0, t * Vt, 0, d, std_base, 0.f);
  if (first_) add(1, s_, d, s_, 0, 0, 0, d, std_base, 0.f);
  close_bucket();  // bucket 0: embeddings (possibly empty)
  for (int l = 0; l < Ll_; ++l) {
    const int b = 2 + kPerLayer * glayer(l);
    add(b + LN1G, d, 1, d, 0, 0, 0, 1, 0.f, 1.f);
    add(b + LN1B, d, 1, d, 0, 0, 0, 1, 0.f, 0.f);
    add(b + WQKV, 3 * dt, d, dt, d, t * dt, 0, d, std_base, 0.f);
    add(b + BQKV, 3 * dt, 1, dt, d, t * dt, 0, 1, 0.f, 0.f);
    add(b + WO, d, dt, d, 0, 0, t * dt, d, std_out, 0.f);
    add(b + BO, d, 1, d, 0, 0, 0, 1, 0.f, 0.f);
    add(b + LN2G, d, 1, d, 0, 0, 0, 1, 0.f, 1.f);
    add(b + LN2B, d, 1, d, 0, 0, 0, 1, 0.f, 0.f);
    add(b + W1, 4 * dt, d, 4 * dt, 0, t * 4 * dt, 0, d, std_base, 0.f);
    add(b + B1, 4 * dt, 1, 4 * dt, 0, t * 4 * dt, 0, 1, 0.f, 0.f);
    add(b + W2, d, 4 * dt, d, 0, 0, t * 4 * dt, 4 * d, std_out, 0.f);
    add(b + B2, d, 1, d, 0, 0, 0, 1, 0.f, 0.f);
    if (l == Ll_ - 1 && last_) {  // final LN grads are final before the last layer's
      add(2 + kPerLayer * L_, d, 1, d, 0, 0, 0, 1, 0.f, 1.f);
      add(2 + kPerLayer * L_ + 1, d, 1, d, 0, 0, 0, 1, 0.f, 0.f);
    }
    close_bucket();
    layer_bucket_.push_back(static_cast<int>(buckets_.size()) - 1);
  }
  P_ = off;
  shard_ = zero_ ? P_ / cfg_.dp : P_;
  slot_index_.assign(2 + kPerLayer * L_ + 2, -1);
  for (size_t i = 0; i < slots_.size(); ++i) slot_index_[slots_[i].tensor_id] = static_cast<int>(i);
}

void Stage::allocate() {
  const size_t M = M_, d = d_, dt = dt_;
  params_ = static_cast<bf16*>(alloc(P_ * sizeof(bf16), MEM_PARAMS));
  grads_ = static_cast<float*>(alloc(P_ * sizeof(float), MEM_GRADS));
  master_ = static_cast<float*>(alloc(shard_ * sizeof(float), MEM_PARAMS));
  adam_m_ = static_cast<float*>(alloc(shard_ * sizeof(float), MEM_OPTIMIZER));
  adam_v_ = static_cast<float*>(alloc(shard_ * sizeof(float), MEM_OPTIMIZER));
  tokens_ = static_cast<int32_t*>(alloc(static_cast<size_t>(cfg_.gbs) * (s_ + 1) * sizeof(int32_t)));

  // TP > 1: full-width buffers that a collective reads or writes on every rank live in one NCCL
  // symmetric window (NVSwitch multicast). With sequence parallelism (SP) that is the row-parallel
  // partial sums (tmp_md_, dm_), the allgathered LayerNorm outputs (a, m2, hf_) and the allgathered
  // input gradient dy_; the residual stream and per-row state shrink to this rank's M/tp rows.
  const size_t Md = M * d;
  const bool sp_wanted = cfg_.tp > 1 && M_ % cfg_.tp == 0 && !(std::getenv("GPTB200_TP_SP") &&
                                                                  std::getenv("GPTB200_TP_SP")[0] == '0');
  size_t sym_elems = 2 * Md;  // tmp_md_, dm_
  // SP + checkpointing with >= 2 layers per chunk: recompute of layer l-1 runs on its own stream
  // during layer l's backward, so the scratch activations are double-buffered by layer parity and the
  // recompute has its own partial-sum buffer (window: a, m2 per scratch set + rc_tmp_).
  const bool rc_overlap = cfg_.tp > 1 && ckpt_ && Lc_ >= 2;
  if (sp_wanted)
    sym_elems += Md + (last_ ? Md : 0) + (ckpt_ ? (rc_overlap ? 5 : 2) : 2 * static_cast<size_t>(nslots_) * Lc_) * Md;
  char* sym = static_cast<char*>(comms_.init_tp_symmetric(sym_elems * 2));
  sp_ = sp_wanted && sym != nullptr;
  Ms_ = sp_ ? M_ / cfg_.tp : M_;
  row0_ = sp_ ? comms_.me.t * Ms_ : 0;
  size_t sym_used = 0;
  window_bytes_ = sym ? nvls_bytes(comms_.tp_nvls) : 0;
  auto full = [&](size_t elems, int cat) -> bf16* {  // [M, d]-class buffer: window when SP/NVLS, else HBM
    if (sym) {
      bf16* p = reinterpret_cast<bf16*>(sym + sym_used);
      sym_used += (elems * 2 + 255) / 256 * 256;
      cat_bytes_[cat] += (elems * 2 + 255) / 256 * 256;
      return p;
    }
    return static_cast<bf16*>(alloc(elems * 2, cat));
  };
  constexpr int ACT = MEM_ACTIVATIONS;
  const size_t Ms = Ms_;
  auto layer_acts = [&](LayerActs& A) {
    A.a = sp_ ? full(Md, ACT) : static_cast<bf16*>(alloc(Md * 2, ACT));
    A.qkv = static_cast<bf16*>(alloc(M * 3 * dt * 2, ACT));
    A.o = static_cast<bf16*>(alloc(M * dt * 2, ACT));
    A.hmid = static_cast<bf16*>(alloc(Ms * d * 2, ACT));
    A.m2 = sp_ ? full(Md, ACT) : static_cast<bf16*>(alloc(Md * 2, ACT));
    A.u = static_cast<bf16*>(alloc(M * 4 * dt * 2, ACT));
    A.g = static_cast<bf16*>(alloc(M * 4 * dt * 2, ACT));
    A.mu1 = static_cast<float*>(alloc(Ms * 4, ACT));
    A.rs1 = static_cast<float*>(alloc(Ms * 4, ACT));
    A.mu2 = static_cast<float*>(alloc(Ms * 4, ACT));
    A.rs2 = static_cast<float*>(alloc(Ms * 4, ACT));
    A.lse = static_cast<float*>(alloc(static_cast<size_t>(mbs_) * ht_ * s_ * 4, ACT));
  };
  tmp_md_ = full(Md, MEM_WORKSPACE);
  dm_ = full(Md, MEM_WORKSPACE);
  slots_act_.resize(nslots_);
  for (auto& S : slots_act_) {
    S.h.resize(Lc_ + 1);
    for (auto& h : S.h) h = static_cast<bf16*>(alloc(Ms * d * 2, ACT));
    if (!ckpt_) {
      S.acts.resize(Lc_);
      for (auto& A : S.acts) layer_acts(A);
    }
    S.inputs = static_cast<int32_t*>(alloc(M * 4, ACT));
    S.labels = static_cast<int32_t*>(alloc(M * 4, ACT));
  }
  if (ckpt_) layer_acts(scratch_);
  rc_overlap_ = sp_ && rc_overlap;
  if (rc_overlap_) {
    layer_acts(scratch2_);
    rc_tmp_ = full(Md, MEM_WORKSPACE);
    cudaStreamCreateWithFlags(&rc_st_, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&rc_fork_, cudaEventDisableTiming);
    for (auto& e : rc_done_) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  }
  for (auto& b : dh_) b = static_cast<bf16*>(alloc(Ms * d * 2));
  dy_ = sp_ ? full(Md, MEM_WORKSPACE) : static_cast<bf16*>(alloc(Md * 2));
  du_ = static_cast<bf16*>(alloc(M * 4 * dt * 2));
  do_ = static_cast<bf16*>(alloc(M * dt * 2));
  dqkv_ = static_cast<bf16*>(alloc(M * 3 * dt * 2));
  attn_D_ = static_cast<float*>(alloc(static_cast<size_t>(mbs_) * ht_ * s_ * 4));
  dq_acc_ = static_cast<float*>(alloc(M * dt * 4));
  size_t ws = std::max({colsum_workspace_floats(M_, 4 * dt_), colsum_workspace_floats(M_, 3 * dt_),
                        ln_bwd_workspace_floats(M_, d_)});
  ws_ = static_cast<float*>(alloc(ws * 4));
  colpart_ = static_cast<float*>(alloc(static_cast<size_t>(M_ / 32) * 4 * dt * 4));
  if (last_) {
    hf_ = sp_ ? full(Md, ACT) : static_cast<bf16*>(alloc(Md * 2, ACT));
    muf_ = static_cast<float*>(alloc(Ms * 4, ACT));
    rsf_ = static_cast<float*>(alloc(Ms * 4, ACT));
    logits_ = static_cast<bf16*>(alloc(M * static_cast<size_t>(Vt_) * 2, ACT));
    xstats_ = static_cast<float*>(alloc(M * 3 * 4));
    // (max, sum exp) per row and 64 logits, written by the LM-head GEMM epilogue
    if (Vt_ % 128 == 0) rowstat_ = static_cast<float2*>(alloc(M * static_cast<size_t>(Vt_ / 64) * 8));
    xall_ = static_cast<float*>(alloc(M * 3 * 4 * cfg_.tp));
    row_loss_ = static_cast<float*>(alloc(M * 4));
  }
  loss_acc_ = static_cast<float*>(alloc(4));
  if (sp_) {
    cudaStreamCreateWithFlags(&sp_st_, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&sp_fork_, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&sp_join_, cudaEventDisableTiming);
  }
  if (cfg_.pp > 1) {
    for (int i = 0; i < 2; ++i) {
      cudaStreamCreateWithFlags(&send_st_[i], cudaStreamNonBlocking);
      cudaEventCreateWithFlags(&send_done_ev_[i], cudaEventDisableTiming);
    }
    slot_send_ev_.resize(nslots_);
    for (auto& e : slot_send_ev_) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    for (auto& e : dh_send_ev_) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&op_ev_, cudaEventDisableTiming);
  }
  overlap_rs_ = true;  // per-bucket RS -> Adam -> AG pipelined on a side stream during backward
  if (overlap_rs_) {
    cudaStreamCreateWithFlags(&comm_st_, cudaStreamNonBlocking);
    bucket_ev_.resize(buckets_.size());
    for (auto& e : bucket_ev_) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&comm_done_, cudaEventDisableTiming);
  }
}

const ParamSlot* Stage::slot(int tid) const {
  if (tid < 0 || tid >= static_cast<int>(slot_index_.size()) || slot_index_[tid] < 0) return nullptr;
  return &slots_[slot_index_[tid]];
}

Stage::LayerW Stage::w(int l) const {
  const int b = 2 + kPerLayer * glayer(l);
  auto p = [&](int j) { return params_ + slot(b + j)->offset; };
  return {p(LN1G), p(LN1B), p(WQKV), p(BQKV), p(WO), p(BO), p(LN2G), p(LN2B), p(W1), p(B1), p(W2), p(B2)};
}

Stage::LayerG Stage::gr(int l) const {
  const int b = 2 + kPerLayer * glayer(l);
  auto p = [&](int j) { return grads_ + slot(b + j)->offset; };
  return {p(LN1G), p(LN1B), p(WQKV), p(BQKV), p(WO), p(BO), p(LN2G), p(LN2B), p(W1), p(B1), p(W2), p(B2)};
}

LayerActs& Stage::acts_for(int slot, int l) {
  if (ckpt_) return (rc_overlap_ && (l & 1)) ? scratch2_ : scratch_;  // parity sets when recompute overlaps
  return slots_act_[slot].acts[l % Lc_];
}

void Stage::init_params() {
  cudaMemsetAsync(grads_, 0, P_ * sizeof(float), st_);
  for (const auto& s : slots_) {
    InitArgs a;
    a.dst = grads_ + s.offset;
    a.rows = s.rows;
    a.cols = s.cols;
    a.rseg = s.rseg;
    a.rstride = s.rstride;
    a.roff = s.roff;
    a.coff = s.coff;
    a.gcols = s.gcols;
    a.seed = opts_.seed;
    a.tensor_id = s.tensor_id;
    // same expression as orc_init_value's scale (bit-identical values)
    a.scale = s.stddev > 0.f ? static_cast<float>(static_cast<double>(s.stddev) * std::sqrt(3.0) / 16777216.0) : 0.f;
    a.constant = s.constant;
    ck(init_tensor(a, st_), "init_tensor");
  }
  ck(cast_f32_bf16(grads_, params_, P_, st_), "cast params");
  for (const Bucket& b : buckets_) {
    const int64_t n = own_len(b);
    if (n) cudaMemcpyAsync(master_ + b.master_off, grads_ + own_offset(b), n * sizeof(float),
                           cudaMemcpyDeviceToDevice, st_);
  }
  cudaMemsetAsync(adam_m_, 0, shard_ * sizeof(float), st_);
  cudaMemsetAsync(adam_v_, 0, shard_ * sizeof(float), st_);
  cudaMemsetAsync(grads_, 0, P_ * sizeof(float), st_);
  step_no_ = 0;
  sync();
}

void Stage::upload_tokens(const int32_t* src, int64_t n, bool on_device) {
  const int64_t need = static_cast<int64_t>(cfg_.gbs) * (s_ + 1);
  if (n != need) throw StepError{TP_ERR_INVALID, "token count " + std::to_string(n) + " != gbs*(s+1) = " + std::to_string(need)};
  cudaError_t e = cudaMemcpyAsync(tokens_, src, n * sizeof(int32_t),
                                  on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st_);
  if (e != cudaSuccess) throw StepError{TP_ERR_CUDA, std::string("token upload: ") + cudaGetErrorString(e)};
}

// ------------------------------------------------------------------------------ GEMM helpers
void Stage::gemm_fwd(const bf16* X, const bf16* W, const bf16* bias, bf16* Y, int M, int N, int K, int epi, bf16* C2) {
  KScope prof(this, K_GEMM, 2.0 * M * N * K);
  GemmParams p;
  p.M = M, p.N = N, p.K = K;
  p.A = X, p.lda = K, p.a_mn = false;
  p.B = W, p.ldb = K, p.b_mn = false;
  p.C = Y, p.ldc = N, p.epi = epi, p.bias = bias, p.C2 = C2;
  ck(gemm_bf16(p, st_), "gemm fwd");
}

// dX[M,K] = dY[M,N] . W[N,K]
void Stage::gemm_dgrad(const bf16* dY, const bf16* W, bf16* dX, int M, int N, int K, int epi, const bf16* aux,
                       const bf16* rowdot_b, float* colsum_part) {
  KScope prof(this, K_GEMM, 2.0 * M * N * K);
  GemmParams p;
  p.M = M, p.N = K, p.K = N;
  p.A = dY, p.lda = N, p.a_mn = false;
  p.B = W, p.ldb = K, p.b_mn = true;
  p.C = dX, p.ldc = K, p.epi = epi, p.aux = aux, p.ldaux = K;
  p.colsum_part = colsum_part;
  if (rowdot_b) {  // attention backward's D = rowsum(dO * O) from the dO epilogue
    cudaMemsetAsync(attn_D_, 0, static_cast<size_t>(mbs_) * ht_ * s_ * sizeof(float), st_);
    p.rowdot_out = attn_D_, p.rowdot_b = rowdot_b, p.rowdot_seq = s_, p.rowdot_heads = ht_;
  }
  ck(gemm_bf16(p, st_), "gemm dgrad");
}

// dW[N,K] += dY[M,N]^T . X[M,K]   (fp32 main grad)
void Stage::gemm_wgrad(const bf16* dY, const bf16* X, float* dW, int M, int N, int K) {
  KScope prof(this, K_GEMM, 2.0 * M * N * K);
  GemmParams p;
  p.M = N, p.N = K, p.K = M;
  p.A = dY, p.lda = N, p.a_mn = true;
  p.B = X, p.ldb = K, p.b_mn = true;
  p.C = dW, p.ldc = K, p.epi = EPI_F32, p.accumulate = 1;
  ck(gemm_bf16(p, st_), "gemm wgrad");
}

// ------------------------------------------------------------------------------ forward
void Stage::prepare_tokens(int mb, int slot) {
  const int64_t sample0 = static_cast<int64_t>(comms_.me.d) * (cfg_.gbs / cfg_.dp) + static_cast<int64_t>(mb) * mbs_;
  ck(split_tokens(tokens_ + sample0 * (s_ + 1), mbs_, s_, slots_act_[slot].inputs, slots_act_[slot].labels, st_),
     "split_tokens");
}

static DropKey drop_key(const TrainOptions& o, int step, int layer, int site, int64_t sample0, int s, int d) {
  DropKey k;
  k.seed = o.seed;
  k.step = step;
  k.layer = layer;
  k.site = site;
  k.p = o.dropout;
  k.elem_base = sample0 * s * static_cast<int64_t>(d);
  return k;
}

void Stage::layer_fwd(int l, LayerActs& A, const bf16* hin, bf16* hout, int slot) {
  const int lg = glayer(l);
  const LayerW W = w(l);
  const bool next_in_chunk = (l + 1) % Lc_ != 0;
  const int64_t sample0 = static_cast<int64_t>(comms_.me.d) * (cfg_.gbs / cfg_.dp) +
                          static_cast<int64_t>(cur_mb_) * mbs_;
  gemm_fwd(A.a, W.wqkv, W.bqkv, A.qkv, M_, 3 * dt_, d_);
  {
    KScope prof(this, K_ATTN_FWD, 2.0 * mbs_ * ht_ * static_cast<double>(s_) * s_ * hd_);
    ck(flash_attn_fwd({mbs_, s_, ht_, hd_}, A.qkv, A.o, A.lse, st_), "flash fwd");
  }
  gemm_fwd(A.o, W.wo, nullptr, tmp_md_, M_, d_, dt_);
  if (sp_) {
    SpLnFwdArgs f;
    f.nrows = Ms_, f.row0 = row0_, f.d = d_, f.seq = s_;
    f.y_off = woff(tmp_md_), f.bias = W.bo, f.resid = hin;
    f.drop = drop_key(opts_, step_no_, lg, 0, sample0, s_, d_);
    f.h_out = A.hmid, f.gamma = W.ln2g, f.beta = W.ln2b, f.ln_off = woff(A.m2), f.mean = A.mu2, f.rstd = A.rs2;
    sp_fwd(f);
    gemm_fwd(A.m2, W.w1, W.b1, A.u, M_, 4 * dt_, d_, EPI_BIAS_GELU, A.g);
    gemm_fwd(A.g, W.w2, nullptr, tmp_md_, M_, d_, 4 * dt_);
    SpLnFwdArgs f2;
    f2.nrows = Ms_, f2.row0 = row0_, f2.d = d_, f2.seq = s_;
    f2.y_off = woff(tmp_md_), f2.bias = W.b2, f2.resid = A.hmid;
    f2.drop = drop_key(opts_, step_no_, lg, 1, sample0, s_, d_);
    f2.h_out = hout;
    const bool next_in_chunk_sp = (l + 1) % Lc_ != 0;
    if (next_in_chunk_sp) {
      LayerActs& N = acts_for(slot, l + 1);
      const LayerW Wn = w(l + 1);
      f2.gamma = Wn.ln1g, f2.beta = Wn.ln1b, f2.ln_off = woff(N.a), f2.mean = N.mu1, f2.rstd = N.rs1;
    } else if (last_vs(l / Lc_)) {
      f2.gamma = params_ + slot_offset(2 + kPerLayer * L_);
      f2.beta = params_ + slot_offset(2 + kPerLayer * L_ + 1);
      f2.ln_off = woff(hf_), f2.mean = muf_, f2.rstd = rsf_;
    }
    sp_fwd(f2);
    return;
  }
  tp_allreduce(tmp_md_);
  ResidLnArgs r;
  r.rows = M_, r.d = d_, r.seq = s_;
  r.y = tmp_md_, r.bias = W.bo, r.resid = hin;
  r.drop = drop_key(opts_, step_no_, lg, 0, sample0, s_, d_);
  r.h_out = A.hmid, r.gamma = W.ln2g, r.beta = W.ln2b, r.ln_out = A.m2, r.mean = A.mu2, r.rstd = A.rs2;
  {
    KScope prof(this, K_NORM, 0, 8.0 * M_ * d_);
    ck(resid_ln_fwd(r, st_), "resid+ln2");
  }
  gemm_fwd(A.m2, W.w1, W.b1, A.u, M_, 4 * dt_, d_, EPI_BIAS_GELU, A.g);
  gemm_fwd(A.g, W.w2, nullptr, tmp_md_, M_, d_, 4 * dt_);
  tp_allreduce(tmp_md_);
  ResidLnArgs r2;
  r2.rows = M_, r2.d = d_, r2.seq = s_;
  r2.y = tmp_md_, r2.bias = W.b2, r2.resid = A.hmid;
  r2.drop = drop_key(opts_, step_no_, lg, 1, sample0, s_, d_);
  r2.h_out = hout;
  if (next_in_chunk || last_vs(l / Lc_)) {
    if (next_in_chunk) {
      LayerActs& N = acts_for(slot, l + 1);
      const LayerW Wn = w(l + 1);
      r2.gamma = Wn.ln1g, r2.beta = Wn.ln1b, r2.ln_out = N.a, r2.mean = N.mu1, r2.rstd = N.rs1;
    } else {
      r2.gamma = params_ + slot_offset(2 + kPerLayer * L_);
      r2.beta = params_ + slot_offset(2 + kPerLayer * L_ + 1);
      r2.ln_out = hf_, r2.mean = muf_, r2.rstd = rsf_;
    }
  }
  {
    KScope prof(this, K_NORM, 0, 8.0 * M_ * d_);
    ck(resid_ln_fwd(r2, st_), "resid+ln1");
  }
}

void Stage::layer_recompute(int l, LayerActs& A, const bf16* hin) {
  const int lg = glayer(l);
  const LayerW W = w(l);
  const int64_t sample0 = static_cast<int64_t>(comms_.me.d) * (cfg_.gbs / cfg_.dp) +
                          static_cast<int64_t>(cur_mb_) * mbs_;
  if (sp_) {
    SpLnFwdArgs f;
    f.nrows = Ms_, f.row0 = row0_, f.d = d_, f.seq = s_;
    f.resid = hin, f.gamma = W.ln1g, f.beta = W.ln1b, f.ln_off = woff(A.a), f.mean = A.mu1, f.rstd = A.rs1;
    sp_fwd(f);
    gemm_fwd(A.a, W.wqkv, W.bqkv, A.qkv, M_, 3 * dt_, d_);
    {
      KScope prof(this, K_ATTN_FWD, 2.0 * mbs_ * ht_ * static_cast<double>(s_) * s_ * hd_);
      ck(flash_attn_fwd({mbs_, s_, ht_, hd_}, A.qkv, A.o, A.lse, st_), "flash fwd");
    }
    gemm_fwd(A.o, W.wo, nullptr, tmp_md_, M_, d_, dt_);
    SpLnFwdArgs f2;
    f2.nrows = Ms_, f2.row0 = row0_, f2.d = d_, f2.seq = s_;
    f2.y_off = woff(tmp_md_), f2.bias = W.bo, f2.resid = hin;
    f2.drop = drop_key(opts_, step_no_, lg, 0, sample0, s_, d_);
    f2.h_out = A.hmid, f2.gamma = W.ln2g, f2.beta = W.ln2b, f2.ln_off = woff(A.m2), f2.mean = A.mu2, f2.rstd = A.rs2;
    sp_fwd(f2);
    gemm_fwd(A.m2, W.w1, W.b1, A.u, M_, 4 * dt_, d_, EPI_BIAS_GELU, A.g);
    return;
  }
  ResidLnArgs r0;
  r0.rows = M_, r0.d = d_, r0.seq = s_;
  r0.resid = hin, r0.gamma = W.ln1g, r0.beta = W.ln1b, r0.ln_out = A.a, r0.mean = A.mu1, r0.rstd = A.rs1;
  {
    KScope prof(this, K_NORM, 0, 8.0 * M_ * d_);
    ck(resid_ln_fwd(r0, st_), "recompute ln1");
  }
  gemm_fwd(A.a, W.wqkv, W.bqkv, A.qkv, M_, 3 * dt_, d_);
  {
    KScope prof(this, K_ATTN_FWD, 2.0 * mbs_ * ht_ * static_cast<double>(s_) * s_ * hd_);
    ck(flash_attn_fwd({mbs_, s_, ht_, hd_}, A.qkv, A.o, A.lse, st_), "flash fwd");
  }
  gemm_fwd(A.o, W.wo, nullptr, tmp_md_, M_, d_, dt_);
  tp_allreduce(tmp_md_);
  ResidLnArgs r;
  r.rows = M_, r.d = d_, r.seq = s_;
  r.y = tmp_md_, r.bias = W.bo, r.resid = hin;
  r.drop = drop_key(opts_, step_no_, lg, 0, sample0, s_, d_);
  r.h_out = A.hmid, r.gamma = W.ln2g, r.beta = W.ln2b, r.ln_out = A.m2, r.mean = A.mu2, r.rstd = A.rs2;
  {
    KScope prof(this, K_NORM, 0, 8.0 * M_ * d_);
    ck(resid_ln_fwd(r, st_), "recompute ln2");
  }
  gemm_fwd(A.m2, W.w1, W.b1, A.u, M_, 4 * dt_, d_, EPI_BIAS_GELU, A.g);
}

void Stage::tp_allreduce(bf16* buf) {
  if (cfg_.tp == 1) return;
  ++launches_;
  KScope prof(this, K_COMM_TP, 0, 2.0 * M_ * d_);
  try {
    comms_.tp_allreduce_bf16(buf, static_cast<size_t>(M_) * d_, st_);
  } catch (const CommError& e) {
    throw StepError{e.code, e.msg};
  }
}

void Stage::forward_op(int mb, int c, int slot, bool head_now) {
  cur_mb_ = mb;
  Slot& S = slots_act_[slot];
  if (first_vs(c) || last_vs(c)) prepare_tokens(mb, slot);
  const int l0 = c * Lc_;
  LayerActs& A0 = acts_for(slot, l0);
  const LayerW W0 = w(l0);
  ResidLnArgs r;
  r.rows = M_, r.d = d_, r.seq = s_;
  r.gamma = W0.ln1g, r.beta = W0.ln1b, r.ln_out = A0.a, r.mean = A0.mu1, r.rstd = A0.rs1;
  if (sp_) {  // embedding partials reduce-scattered / LN1 allgathered in one NVLS kernel
    SpLnFwdArgs f;
    f.nrows = Ms_, f.row0 = row0_, f.d = d_, f.seq = s_;
    if (first_vs(c)) {
      ck(embed_lookup(S.inputs, M_, params_ + slot_offset(0), comms_.me.t * Vt_, Vt_, d_, tmp_md_, st_), "embed");
      const int64_t sample0 = static_cast<int64_t>(comms_.me.d) * (cfg_.gbs / cfg_.dp) + static_cast<int64_t>(mb) * mbs_;
      f.y_off = woff(tmp_md_), f.resid = params_ + slot_offset(1), f.resid_pos_table = true;
      f.drop = drop_key(opts_, step_no_, kEmbedLayer, 2, sample0, s_, d_);
      f.h_out = S.h[0];
    } else {
      f.resid = S.h[0];
    }
    f.gamma = W0.ln1g, f.beta = W0.ln1b, f.ln_off = woff(A0.a), f.mean = A0.mu1, f.rstd = A0.rs1;
    sp_fwd(f);
    for (int l = 0; l < Lc_; ++l) layer_fwd(l0 + l, acts_for(slot, l0 + l), S.h[l], S.h[l + 1], slot);
    if (last_vs(c) && head_now) head_and_loss(slot);
    return;
  }
  if (first_vs(c)) {
    ck(embed_lookup(S.inputs, M_, params_ + slot_offset(0), comms_.me.t * Vt_, Vt_, d_, tmp_md_, st_), "embed");
    tp_allreduce(tmp_md_);
    const int64_t sample0 = static_cast<int64_t>(comms_.me.d) * (cfg_.gbs / cfg_.dp) + static_cast<int64_t>(mb) * mbs_;
    r.y = tmp_md_, r.resid = params_ + slot_offset(1), r.resid_pos_table = true;
    r.drop = drop_key(opts_, step_no_, kEmbedLayer, 2, sample0, s_, d_);
    r.h_out = S.h[0];
  } else {
    r.resid = S.h[0];
  }
  {
    KScope prof(this, K_NORM, 0, 8.0 * M_ * d_);
    ck(resid_ln_fwd(r, st_), "embed+ln1");
  }
  for (int l = 0; l < Lc_; ++l) layer_fwd(l0 + l, acts_for(slot, l0 + l), S.h[l], S.h[l + 1], slot);
  if (last_vs(c) && head_now) head_and_loss(slot);
}

void Stage::final_ln(const bf16* h) {
  if (sp_) {
    SpLnFwdArgs f;
    f.nrows = Ms_, f.row0 = row0_, f.d = d_, f.seq = s_;
    f.resid = h;
    f.gamma = params_ + slot_offset(2 + kPerLayer * L_);
    f.beta = params_ + slot_offset(2 + kPerLayer * L_ + 1);
    f.ln_off = woff(hf_), f.mean = muf_, f.rstd = rsf_;
    sp_fwd(f);
    return;
  }
  ResidLnArgs r;
  r.rows = M_, r.d = d_, r.seq = s_;
  r.resid = h;
  r.gamma = params_ + slot_offset(2 + kPerLayer * L_);
  r.beta = params_ + slot_offset(2 + kPerLayer * L_ + 1);
  r.ln_out = hf_, r.mean = muf_, r.rstd = rsf_;
  KScope prof(this, K_NORM, 0, 4.0 * M_ * d_);
  ck(resid_ln_fwd(r, st_), "final ln");
}

// hf_ (final LN output of this microbatch) -> vocab-parallel logits -> CE; logits_ is left holding
// the loss-scaled softmax - onehot for head_bwd.
void Stage::head_and_loss(int slot) {
  Slot& S = slots_act_[slot];
  if (rowstat_) {  // LM head with the softmax statistics in its epilogue: no extra pass over the logits
    {
      KScope prof(this, K_GEMM, 2.0 * M_ * Vt_ * d_);
      GemmParams p;
      p.M = M_, p.N = Vt_, p.K = d_;
      p.A = hf_, p.lda = d_;
      p.B = params_ + slot_offset(0), p.ldb = d_;
      p.C = logits_, p.ldc = Vt_, p.epi = EPI_BF16;
      p.rowstat_part = rowstat_;
      ck(gemm_bf16(p, st_), "lm head");
    }
    ck(xent_stats_from_parts(logits_, rowstat_, M_, Vt_, S.labels, comms_.me.t * Vt_, xstats_, st_), "xent stats");
  } else {
    gemm_fwd(hf_, params_ + slot_offset(0), nullptr, logits_, M_, Vt_, d_);
    ck(xent_stats(logits_, M_, Vt_, S.labels, comms_.me.t * Vt_, xstats_, st_), "xent stats");
  }
  try {
    comms_.tp_allgather_f32(xstats_, xall_, static_cast<size_t>(M_) * 3, st_);
  } catch (const CommError& e) {
    throw StepError{e.code, e.msg};
  }
  const float scale = static_cast<float>(1.0 / (static_cast<double>(cfg_.gbs) * s_));
  ck(xent_finish(logits_, M_, Vt_, S.labels, comms_.me.t * Vt_, xall_, cfg_.tp, scale, row_loss_, st_), "xent finish");
  if (comms_.me.t == 0) ck(accumulate_sum(row_loss_, M_, loss_acc_, st_), "loss sum");
}

// ------------------------------------------------------------------------------ backward
void Stage::head_bwd(bf16* dh) {
  // logits_ holds scale*(softmax - onehot). Vocab-parallel: partial dX summed over TP.
  gemm_dgrad(logits_, params_ + slot_offset(0), tmp_md_, M_, Vt_, d_);
  if (!sp_) tp_allreduce(tmp_md_);  // SP: reduced in the final-LN backward kernel
  gemm_wgrad(logits_, hf_, grads_ + slot_offset(0), M_, Vt_, d_);
}

void Stage::layer_bwd(int l, LayerActs& A, const bf16* hin, bf16* dh, bf16* dy2) {
  const int lg = glayer(l);
  const LayerW W = w(l);
  const LayerG G = gr(l);
  const bool drop_on = opts_.dropout > 0.f;
  const bool fuse_d = hd_ == 128 && dt_ % 128 == 0;  // D computed in the W_o dgrad epilogue
  const int64_t sample0 = static_cast<int64_t>(comms_.me.d) * (cfg_.gbs / cfg_.dp) +
                          static_cast<int64_t>(cur_mb_) * mbs_;
  // MLP branch
  gemm_dgrad(dy2, W.w2, du_, M_, d_, 4 * dt_, EPI_DGELU, A.u, nullptr, colpart_);  // + db1 partials
  gemm_wgrad(dy2, A.g, G.w2, M_, d_, 4 * dt_);
  {
    KScope prof(this, K_ELEM);
    ck(reduce_col_partials(colpart_, M_ / 32, 4 * dt_, G.b1, st_), "db1");
  }
  gemm_dgrad(du_, W.w1, dm_, M_, 4 * dt_, d_);
  if (sp_) {
    // the fused reduce-scatter + LN2 backward needs only the dgrad partials: it runs on the SP
    // stream while the independent fc1 weight-gradient GEMM runs here (NVLink under tensor work)
    SpLnBwdArgs g;
    g.nrows = Ms_, g.row0 = row0_, g.d = d_, g.workspace = ws_;
    g.dy_off = woff(dm_), g.x = A.hmid, g.gamma = W.ln2g, g.mean = A.mu2, g.rstd = A.rs2;
    g.resid_grad = dh, g.dx = dh;
    g.drop = drop_key(opts_, step_no_, lg, 0, sample0, s_, d_);
    g.dxd_off = woff(dy_), g.dgamma = G.ln2g, g.dbeta = G.ln2b, g.dbias = G.bo;
    sp_bwd_overlapped(g, [&] { gemm_wgrad(du_, A.m2, G.w1, M_, 4 * dt_, d_); });
    gemm_dgrad(dy_, W.wo, do_, M_, d_, dt_, EPI_BF16, nullptr, fuse_d ? A.o : nullptr);
    gemm_wgrad(dy_, A.o, G.wo, M_, d_, dt_);
    {
      KScope prof(this, K_ATTN_BWD, 5.0 * mbs_ * ht_ * static_cast<double>(s_) * s_ * hd_);
      // hd 128: the qkv bias gradient is folded into the attention backward kernels
      ck(flash_attn_bwd({mbs_, s_, ht_, hd_}, A.qkv, A.o, do_, A.lse, attn_D_, dq_acc_, dqkv_, st_, fuse_d, G.bqkv),
         "flash bwd");
    }
    if (hd_ != 128) {
      KScope prof(this, K_ELEM);
      ck(colsum_bf16(dqkv_, M_, 3 * dt_, G.bqkv, ws_, st_), "dbqkv");
    }
    gemm_dgrad(dqkv_, W.wqkv, dm_, M_, 3 * dt_, d_);
    SpLnBwdArgs g1;
    g1.nrows = Ms_, g1.row0 = row0_, g1.d = d_, g1.workspace = ws_;
    g1.dy_off = woff(dm_), g1.x = hin, g1.gamma = W.ln1g, g1.mean = A.mu1, g1.rstd = A.rs1;
    g1.resid_grad = dh, g1.dx = dh, g1.dgamma = G.ln1g, g1.dbeta = G.ln1b;
    if (l % Lc_ > 0) {  // preceding branch: MLP of layer l-1 in this chunk
      g1.drop = drop_key(opts_, step_no_, lg - 1, 1, sample0, s_, d_);
      g1.dxd_off = woff(dy_), g1.dbias = gr(l - 1).b2;
    } else if (first_vs(l / Lc_)) {  // embedding dropout; dy_ feeds the embedding backward
      g1.drop = drop_key(opts_, step_no_, kEmbedLayer, 2, sample0, s_, d_);
      g1.dxd_off = woff(dy_);
    }
    sp_bwd_overlapped(g1, [&] { gemm_wgrad(dqkv_, A.a, G.wqkv, M_, 3 * dt_, d_); });
    return;
  }
  tp_allreduce(dm_);
  gemm_wgrad(du_, A.m2, G.w1, M_, 4 * dt_, d_);
  LnBwdArgs b;
  b.rows = M_, b.d = d_;
  b.x = A.hmid, b.dy = dm_, b.resid_grad = dh, b.gamma = W.ln2g, b.mean = A.mu2, b.rstd = A.rs2;
  b.dx = dh;
  b.drop = drop_key(opts_, step_no_, lg, 0, sample0, s_, d_);
  b.dxd = drop_on ? dy_ : dh;
  b.dgamma = G.ln2g, b.dbeta = G.ln2b, b.dbias = G.bo, b.workspace = ws_;
  {
    KScope prof(this, K_NORM, 0, 10.0 * M_ * d_);
    ck(ln_bwd(b, st_), "ln2 bwd");
  }
  const bf16* dya = drop_on ? dy_ : dh;
  // attention branch
  gemm_dgrad(dya, W.wo, do_, M_, d_, dt_, EPI_BF16, nullptr, fuse_d ? A.o : nullptr);
  gemm_wgrad(dya, A.o, G.wo, M_, d_, dt_);
  {
    KScope prof(this, K_ATTN_BWD, 5.0 * mbs_ * ht_ * static_cast<double>(s_) * s_ * hd_);
    ck(flash_attn_bwd({mbs_, s_, ht_, hd_}, A.qkv, A.o, do_, A.lse, attn_D_, dq_acc_, dqkv_, st_, fuse_d, G.bqkv),
       "flash bwd");
  }
  if (hd_ != 128) {
    KScope prof(this, K_ELEM);
    ck(colsum_bf16(dqkv_, M_, 3 * dt_, G.bqkv, ws_, st_), "dbqkv");
  }
  gemm_dgrad(dqkv_, W.wqkv, dm_, M_, 3 * dt_, d_);
  tp_allreduce(dm_);
  gemm_wgrad(dqkv_, A.a, G.wqkv, M_, 3 * dt_, d_);
  LnBwdArgs c;
  c.rows = M_, c.d = d_;
  c.x = hin, c.dy = dm_, c.resid_grad = dh, c.gamma = W.ln1g, c.mean = A.mu1, c.rstd = A.rs1;
  c.dx = dh;
  c.dgamma = G.ln1g, c.dbeta = G.ln1b, c.workspace = ws_;
  if (l % Lc_ > 0) {  // preceding branch: MLP of layer l-1 in this chunk
    c.drop = drop_key(opts_, step_no_, lg - 1, 1, sample0, s_, d_);
    c.dxd = drop_on ? dy_ : dh;
    c.dbias = gr(l - 1).b2;
  } else if (first_vs(l / Lc_)) {  // preceding branch: embedding dropout
    c.drop = drop_key(opts_, step_no_, kEmbedLayer, 2, sample0, s_, d_);
    c.dxd = drop_on ? dy_ : dh;
  }
  {
    KScope prof(this, K_NORM, 0, 10.0 * M_ * d_);
    ck(ln_bwd(c, st_), "ln1 bwd");
  }
}

void Stage::backward_op(int mb, int c, int slot, bf16* dh, bool head_late) {
  cur_mb_ = mb;
  Slot& S = slots_act_[slot];
  const bool drop_on = opts_.dropout > 0.f;
  const int l_last = (c + 1) * Lc_ - 1;
  const int64_t sample0 = static_cast<int64_t>(comms_.me.d) * (cfg_.gbs / cfg_.dp) + static_cast<int64_t>(mb) * mbs_;
  if (sp_) {
    // chunk output: final LN backward (last virtual stage) or the received gradient; either way
    // the dropout' of the last layer's MLP branch is allgathered into dy_ for that MLP backward
    SpLnBwdArgs g;
    g.nrows = Ms_, g.row0 = row0_, g.d = d_, g.workspace = ws_;
    g.drop = drop_key(opts_, step_no_, glayer(l_last), 1, sample0, s_, d_);
    g.dxd_off = woff(dy_), g.dbias = gr(l_last).b2;
    if (last_vs(c)) {
      if (head_late) {
        final_ln(S.h[Lc_]);
        head_and_loss(slot);
      }
      head_bwd(dh);
      const int f = 2 + kPerLayer * L_;
      g.dy_off = woff(tmp_md_), g.x = S.h[Lc_], g.gamma = params_ + slot_offset(f), g.mean = muf_, g.rstd = rsf_;
      g.dx = dh, g.dgamma = grads_ + slot_offset(f), g.dbeta = grads_ + slot_offset(f + 1);
    } else {
      g.resid_grad = dh;  // received gradient of the chunk output (shard); dh itself is unchanged
    }
    sp_bwd(g);
    const bool prefetch = ckpt_ && rc_overlap_ && !profile_;
    for (int l = Lc_ - 1; l >= 0; --l) {
      const int li = c * Lc_ + l;
      LayerActs& A = acts_for(slot, li);
      if (ckpt_) {
        if (prefetch && l < Lc_ - 1)
          cudaStreamWaitEvent(st_, rc_done_[li & 1], 0);  // recompute(li) ran on rc_st_ meanwhile
        else
          layer_recompute(li, A, S.h[l]);
      }
      if (prefetch && l >= 1) {  // recompute(li - 1) on rc_st_ while layer li's backward runs here
        cudaEventRecord(rc_fork_, st_);  // its scratch set was last read by layer li + 1 (issued above)
        cudaStreamWaitEvent(rc_st_, rc_fork_, 0);
        RecomputeOnSide side(this);
        layer_recompute(li - 1, acts_for(slot, li - 1), S.h[l - 1]);
        cudaEventRecord(rc_done_[(li - 1) & 1], rc_st_);
      }
      layer_bwd(li, A, S.h[l], dh, dy_);
      if (in_last_bwd_) grads_ready(layer_bucket_[li]);
    }
    if (first_vs(c))
      ck(embed_bwd(S.inputs, M_, dy_, comms_.me.t * Vt_, Vt_, d_, s_, grads_ + slot_offset(0), grads_ + slot_offset(1), st_),
         "embed bwd");
    return;
  }
  LnBwdArgs b;
  b.rows = M_, b.d = d_, b.workspace = ws_;
  b.drop = drop_key(opts_, step_no_, glayer(l_last), 1, sample0, s_, d_);
  b.dxd = drop_on ? dy_ : dh;
  b.dbias = gr(l_last).b2;
  if (last_vs(c)) {
    if (head_late) {  // another microbatch's forward ran since ours: rebuild the head input
      final_ln(S.h[Lc_]);
      head_and_loss(slot);
    }
    head_bwd(dh);
    const int f = 2 + kPerLayer * L_;
    b.x = S.h[Lc_], b.dy = tmp_md_, b.gamma = params_ + slot_offset(f), b.mean = muf_, b.rstd = rsf_;
    b.dx = dh, b.dgamma = grads_ + slot_offset(f), b.dbeta = grads_ + slot_offset(f + 1);
  } else {
    b.resid_grad = dh;  // received gradient of the chunk output
    b.dx = nullptr;
    if (!drop_on) b.dxd = nullptr;
  }
  {
    KScope prof(this, K_NORM, 0, 10.0 * M_ * d_);
    ck(ln_bwd(b, st_), "final ln / stage-boundary bwd");
  }
  for (int l = Lc_ - 1; l >= 0; --l) {
    const int li = c * Lc_ + l;
    LayerActs& A = acts_for(slot, li);
    if (ckpt_) layer_recompute(li, A, S.h[l]);
    layer_bwd(li, A, S.h[l], dh, drop_on ? dy_ : dh);
    if (in_last_bwd_) grads_ready(layer_bucket_[li]);
  }
  if (first_vs(c)) {
    const bf16* g = drop_on ? dy_ : dh;
    ck(embed_bwd(S.inputs, M_, g, comms_.me.t * Vt_, Vt_, d_, s_, grads_ + slot_offset(0), grads_ + slot_offset(1), st_),
       "embed bwd");
  }
}

// ------------------------------------------------------------------------------ SP helpers
int64_t Stage::woff(const void* p) const {
  const int64_t o = nvls_offset(comms_.tp_nvls, p);
  if (o < 0) throw StepError{TP_ERR_INVALID, "sequence-parallel buffer outside the symmetric window"};
  return o;
}

// Issue the enclosed recompute on rc_st_: launches go to that stream, its row-parallel partials to
// rc_tmp_, and its SP kernels use NVLS barrier set 1 (they may run concurrently with set-0 kernels).
Stage::RecomputeOnSide::RecomputeOnSide(Stage* st) : s(st), st(st->st_), tmp(st->tmp_md_) {
  s->st_ = s->rc_st_;
  s->tmp_md_ = s->rc_tmp_;
  s->sp_lane_set_ = 1;
}

Stage::RecomputeOnSide::~RecomputeOnSide() {
  s->st_ = st;
  s->tmp_md_ = tmp;
  s->sp_lane_set_ = 0;
}

void Stage::sp_fwd(const SpLnFwdArgs& a_in) {
  ++launches_;
  KScope prof(this, K_COMM_TP, 0, (a_in.y_off >= 0 ? 2.0 : 0.0) * M_ * d_ + 6.0 * Ms_ * d_);
  SpLnFwdArgs a = a_in;
  a.lane_set = sp_lane_set_;
  const int r = sp_ln_fwd(comms_.tp_nvls, a, st_);
  if (r != 0) throw StepError{r == 1 ? TP_ERR_INVALID : TP_ERR_CUDA, "sequence-parallel LN forward failed"};
}

// SP backward on sp_st_ concurrently with `independent` (a weight-gradient GEMM) on st_; the step
// stream joins before the next consumer of dh / dy_. SP kernels stay totally ordered on every rank.
template <typename F>
void Stage::sp_bwd_overlapped(const SpLnBwdArgs& a, F&& independent) {
  if (profile_ || !sp_st_) {  // profiled pass: keep every launch on the timed stream
    independent();
    sp_bwd(a);
    return;
  }
  cudaEventRecord(sp_fork_, st_);
  cudaStreamWaitEvent(sp_st_, sp_fork_, 0);
  launches_ += 3;
  const int r = sp_ln_bwd(comms_.tp_nvls, a, sp_st_);
  if (r != 0) throw StepError{r == 1 ? TP_ERR_INVALID : TP_ERR_CUDA, "sequence-parallel LN backward failed"};
  independent();
  cudaEventRecord(sp_join_, sp_st_);
  cudaStreamWaitEvent(st_, sp_join_, 0);
}

void Stage::sp_bwd(const SpLnBwdArgs& a) {
  launches_ += 3;
  KScope prof(this, K_COMM_TP, 0, (a.dy_off >= 0 ? 2.0 : 0.0) * M_ * d_ + 10.0 * Ms_ * d_);
  const int r = sp_ln_bwd(comms_.tp_nvls, a, st_);
  if (r != 0) throw StepError{r == 1 ? TP_ERR_INVALID : TP_ERR_CUDA, "sequence-parallel LN backward failed"};
}

// ------------------------------------------------------------------------------ step
// Adam on this rank's slice of one bucket, on `st` (fp32 master/m/v, writes the bf16 copy).
void Stage::adam_bucket(int bucket, cudaStream_t st) {
  const Bucket& b = buckets_[bucket];
  const int64_t n = own_len(b);
  if (!n) return;
  AdamArgs a;
  a.lr = opts_.lr, a.beta1 = opts_.beta1, a.beta2 = opts_.beta2, a.eps = opts_.eps, a.weight_decay = opts_.weight_decay;
  a.bc1 = static_cast<float>(1.0 - std::pow(static_cast<double>(opts_.beta1), step_no_));
  a.bc2 = static_cast<float>(1.0 - std::pow(static_cast<double>(opts_.beta2), step_no_));
  const int64_t own = own_offset(b);
  a.n = n, a.master = master_ + b.master_off, a.m = adam_m_ + b.master_off, a.v = adam_v_ + b.master_off;
  a.grad = grads_ + own, a.param = params_ + own;
  ck(adam_step(a, st), "adam");
}

// The bucket's gradients are final on the compute stream (last microbatch): on the side stream,
// reduce-scatter them over DP (in place), run Adam on the owned slice and allgather the updated
// bf16 slices — all while backward continues with earlier layers (whose parameters are
// untouched by this bucket's update).
void Stage::grads_ready(int bucket) {
  const Bucket& b = buckets_[bucket];
  if (!b.len) return;
  cudaEventRecord(bucket_ev_[bucket], st_);
  cudaStreamWaitEvent(comm_st_, bucket_ev_[bucket], 0);
  try {
    if (sp_) {  // LayerNorm / row-parallel bias grads were summed over this rank's rows only
      std::vector<std::pair<float*, size_t>> parts;
      for (int li = 0; li < Ll_; ++li) {
        if (layer_bucket_[li] != bucket) continue;
        const LayerG G = gr(li);
        for (float* g : {G.ln1g, G.ln1b, G.bo, G.ln2g, G.ln2b, G.b2}) parts.push_back({g, static_cast<size_t>(d_)});
        if (li == Ll_ - 1 && last_) {
          parts.push_back({grads_ + slot_offset(2 + kPerLayer * L_), static_cast<size_t>(d_)});
          parts.push_back({grads_ + slot_offset(2 + kPerLayer * L_ + 1), static_cast<size_t>(d_)});
        }
      }
      comms_.tp_allreduce_f32_group(parts, comm_st_);
    }
    if (bucket == 0 && cfg_.pp > 1 && (first_ || last_))
      comms_.emb_allreduce_f32(grads_ + slot_offset(0), static_cast<size_t>(Vt_) * d_, comm_st_);
    // DP collectives are timed on the comm stream (K_COMM_DP: overlapped with backward; the exposed
    // part is the K_ADAM tail of step())
    if (cfg_.dp > 1) {
      KScope prof(this, K_COMM_DP, 0, (zero_ ? 4.0 : 8.0) * b.len, comm_st_);
      if (zero_) comms_.dp_reduce_scatter_f32(grads_ + b.off, b.len / cfg_.dp, comm_st_);
      else comms_.dp_allreduce_f32(grads_ + b.off, b.len, comm_st_);  // ZeRO-0 (perf.cpp:101)
    }
    adam_bucket(bucket, comm_st_);
    if (cfg_.dp > 1 && zero_) {
      KScope prof(this, K_COMM_DP, 0, 2.0 * b.len, comm_st_);
      comms_.dp_allgather_bf16(params_ + b.off, b.len / cfg_.dp, comm_st_);
    }
  } catch (const CommError& e) {
    throw StepError{e.code, e.msg};
  }
}

// Pipeline p2p of one plan action (runtime/pipe_exec.h): receive on the compute stream before the
// op; send on the direction's side stream after it, recording the buffer's send-done event.
void Stage::pp_recv(void* buf, int dir) {
  ++launches_;
  KScope prof(this, K_COMM_PP);
  comms_.pp_recv(buf, static_cast<size_t>(Ms_) * d_, dir, st_);  // SP: this rank's rows only
}

void Stage::pp_send(const void* buf, int dir, cudaEvent_t done) {
  ++launches_;
  cudaEventRecord(op_ev_, st_);
  cudaStreamWaitEvent(send_st_[dir], op_ev_, 0);
  comms_.pp_send(buf, static_cast<size_t>(Ms_) * d_, dir, send_st_[dir]);
  cudaEventRecord(done, send_st_[dir]);
}

void Stage::run_action(const PipeAction& a) {
  static const bool trace = std::getenv("GPTB200_TRACE_PIPE") != nullptr;
  if (trace)
    std::fprintf(stderr, "[stage %d] %s mb %d chunk %d slot %d dh %d flags %d\n", comms_.me.p,
                 a.kind == PA_FWD ? "F" : "B", a.microbatch, a.chunk, a.slot, a.dh, a.flags);
  if (a.kind == PA_FWD) {
    Slot& S = slots_act_[a.slot];
    if (cfg_.pp > 1) cudaStreamWaitEvent(st_, slot_send_ev_[a.slot], 0);  // h[Lc] of the slot's last use sent
    if (a.flags & PA_RECV) pp_recv(S.h[0], 0);
    forward_op(a.microbatch, a.chunk, a.slot, (a.flags & PA_HEAD) != 0);
    if (a.flags & PA_SEND) pp_send(S.h[Lc_], 0, slot_send_ev_[a.slot]);
  } else {
    bf16* dh = dh_[a.dh];
    if (cfg_.pp > 1) cudaStreamWaitEvent(st_, dh_send_ev_[a.dh], 0);
    if (a.flags & PA_RECV) pp_recv(dh, 1);
    in_last_bwd_ = (a.flags & PA_LAST_MB) != 0;
    backward_op(a.microbatch, a.chunk, a.slot, dh, (a.flags & PA_HEAD_LATE) != 0);
    in_last_bwd_ = false;
    if (a.flags & PA_SEND) pp_send(dh, 1, dh_send_ev_[a.dh]);
  }
}

void Stage::join_sends() {
  for (int i = 0; i < 2; ++i)
    if (send_st_[i]) {
      cudaEventRecord(send_done_ev_[i], send_st_[i]);
      cudaStreamWaitEvent(st_, send_done_ev_[i], 0);
    }
}

void Stage::step() {
  ++step_no_;
  launches_ = 0;
  cudaMemsetAsync(grads_, 0, P_ * sizeof(float), st_);
  cudaMemsetAsync(loss_acc_, 0, sizeof(float), st_);
  try {
    for (const PipeAction& a : plan_) run_action(a);
    join_sends();
    grads_ready(0);  // embeddings (tied wte: after the first/last-stage allreduce)
    {
      KScope prof(this, K_ADAM);  // exposed tail of the side-stream optimizer pipeline
      cudaEventRecord(comm_done_, comm_st_);
      cudaStreamWaitEvent(st_, comm_done_, 0);
    }
    comms_.world_allreduce_f32(loss_acc_, 1, st_);
  } catch (const CommError& e) {
    throw StepError{e.code, e.msg};
  }
}

float Stage::read_loss() {
  float v = 0.f;
  cudaMemcpyAsync(&v, loss_acc_, sizeof(float), cudaMemcpyDeviceToHost, st_);
  wait(st_, "read loss");
  return static_cast<float>(v / (static_cast<double>(cfg_.gbs) * s_));
}

float Stage::eval_loss() {
  cudaMemsetAsync(loss_acc_, 0, sizeof(float), st_);
  try {
    for (const PipeAction& a : eval_plan_) run_action(a);
    join_sends();
    comms_.world_allreduce_f32(loss_acc_, 1, st_);
  } catch (const CommError& e) {
    throw StepError{e.code, e.msg};
  }
  return read_loss();
}

void Stage::sync() { wait(st_, "stream sync"); }

// Host wait with a watchdog. Spins briefly (the common case: the step is about to finish), then
// polls with a growing sleep. On timeout the communicators are aborted so peers blocked in NCCL
// return errors instead of hanging, and the session is marked unusable (a kernel spinning on a
// dead peer's barrier cannot be cancelled: the process should exit).
void Stage::wait(cudaStream_t st, const char* what) {
  if (poisoned_) throw StepError{TP_ERR_TIMEOUT, std::string(what) + ": session aborted by the watchdog"};
  if (timeout_s_ <= 0) {
    const cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) throw StepError{TP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e)};
    return;
  }
  using clock = std::chrono::steady_clock;
  const auto t0 = clock::now();
  for (int it = 0;; ++it) {
    const cudaError_t e = cudaStreamQuery(st);
    if (e == cudaSuccess) return;
    if (e != cudaErrorNotReady) throw StepError{TP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e)};
    const double waited = std::chrono::duration<double>(clock::now() - t0).count();
    if (waited > timeout_s_) {
      poisoned_ = true;
      comms_.abort();
      throw StepError{TP_ERR_TIMEOUT, std::string(what) + ": no progress after " + std::to_string(waited) +
                                          " s (watchdog); NCCL communicators aborted"};
    }
    if (it < 2000) continue;  // ~ the first millisecond: spin
    std::this_thread::sleep_for(std::chrono::microseconds(it < 4000 ? 20 : 200));
  }
}

void Stage::barrier() {
  if (comms_.world > 1) {
    float* one = loss_acc_;  // any device float works; value is irrelevant after the step read
    (void)one;
    float* tmp = static_cast<float*>(ws_);
    try {
      comms_.world_allreduce_f32(tmp, 1, st_);
    } catch (const CommError& e) {
      throw StepError{e.code, e.msg};
    }
  }
  sync();
}

void Stage::read_flat(int which, int64_t offset, int64_t n, float* host) const {
  const int64_t len = (which <= 1) ? P_ : shard_;
  if (offset < 0 || n < 0 || offset + n > len) throw StepError{TP_ERR_INVALID, "read_flat: range out of bounds"};
  const_cast<Stage*>(this)->wait(st_, "read_flat");
  if (which == 0) {
    std::vector<uint16_t> tmp(n);
    cudaMemcpy(tmp.data(), params_ + offset, n * 2, cudaMemcpyDeviceToHost);
    for (int64_t i = 0; i < n; ++i) {
      uint32_t u = static_cast<uint32_t>(tmp[i]) << 16;
      std::memcpy(&host[i], &u, 4);
    }
    return;
  }
  const float* base = which == 1 ? grads_ : which == 2 ? master_ : which == 3 ? adam_m_ : adam_v_;
  cudaMemcpy(host, base + offset, n * 4, cudaMemcpyDeviceToHost);
}

void Stage::read_tensor(int which, int tid, float* host) const {
  const ParamSlot* s = slot(tid);
  if (!s) throw StepError{TP_ERR_INVALID, "tensor " + std::to_string(tid) + " not on this rank"};
  const int64_t n = s->rows * s->cols;
  const_cast<Stage*>(this)->wait(st_, "read_tensor");
  if (which == 0) {
    std::vector<uint16_t> tmp(n);
    cudaMemcpy(tmp.data(), params_ + s->offset, n * 2, cudaMemcpyDeviceToHost);
    for (int64_t i = 0; i < n; ++i) {
      uint32_t u = static_cast<uint32_t>(tmp[i]) << 16;
      std::memcpy(&host[i], &u, 4);
    }
    return;
  }
  const float* base = nullptr;
  int64_t off = s->offset;
  if (which == 1) {
    base = grads_;
  } else {
    int64_t moff = -1;
    for (const Bucket& b : buckets_) {
      const int64_t per = own_len(b), own = own_offset(b);
      if (off >= own && off + n <= own + per) moff = b.master_off + (off - own);
    }
    if (moff < 0) throw StepError{TP_ERR_INVALID, "tensor outside this rank's ZeRO shard"};
    off = moff;
    base = which == 2 ? master_ : (which == 3 ? adam_m_ : adam_v_);
  }
  cudaMemcpy(host, base + off, n * 4, cudaMemcpyDeviceToHost);
}

}  // namespace gptb200

namespace gptb200 {

float Stage::time_steps(int steps, bool profile, KernelTimes* kt) {
  // one event between consecutive steps (no host sync inside the timed region): the total and the
  // per-step device times (step_ms_) for the spread
  std::vector<cudaEvent_t> ev(static_cast<size_t>(steps) + 1);
  for (auto& e : ev) cudaEventCreate(&e);
  auto destroy = [&] {
    for (auto& e : ev) cudaEventDestroy(e);
  };
  profile_ = profile;
  ev_used_ = 0;
  prof_acc_ = KernelTimes{};
  cudaEventRecord(ev[0], st_);
  try {
    for (int i = 0; i < steps; ++i) {
      step();
      cudaEventRecord(ev[i + 1], st_);
    }
  } catch (...) {
    profile_ = false;
    destroy();
    throw;
  }
  sync();
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ev[0], ev[steps]);
  step_ms_.assign(steps, 0.f);
  for (int i = 0; i < steps; ++i) cudaEventElapsedTime(&step_ms_[i], ev[i], ev[i + 1]);
  if (profile && kt) {
    *kt = prof_acc_;
    for (int k = 0; k < K_NUM; ++k) kt->ms[k] = 0;
    for (size_t i = 0; i < ev_used_; ++i) {
      float e = 0.f;
      cudaEventElapsedTime(&e, ev_pool_[i].first, ev_pool_[i].second);
      kt->ms[ev_kind_[i]] += e;
    }
  }
  profile_ = false;
  destroy();
  return ms;
}

void Stage::debug_tp_allreduce(const uint16_t* in, uint16_t* out, int mode) {
  const size_t n = static_cast<size_t>(M_) * d_;
  cudaMemcpyAsync(tmp_md_, in, n * 2, cudaMemcpyHostToDevice, st_);
  try {
    comms_.tp_allreduce_bf16(tmp_md_, n, st_, mode);
  } catch (const CommError& e) {
    throw StepError{e.code, e.msg};
  }
  cudaMemcpyAsync(out, tmp_md_, n * 2, cudaMemcpyDeviceToHost, st_);
  sync();
}

float Stage::bench_tp_allreduce(int iters, int mode, int ctas) {
  const size_t n = static_cast<size_t>(M_) * d_;
  comms_.tp_nvls_ctas = ctas;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  try {
    for (int i = 0; i < 3; ++i) comms_.tp_allreduce_bf16(tmp_md_, n, st_, mode);
    cudaEventRecord(a, st_);
    for (int i = 0; i < iters; ++i) comms_.tp_allreduce_bf16(tmp_md_, n, st_, mode);
    cudaEventRecord(b, st_);
  } catch (const CommError& e) {
    comms_.tp_nvls_ctas = 0;
    throw StepError{e.code, e.msg};
  }
  sync();
  comms_.tp_nvls_ctas = 0;
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return ms / std::max(iters, 1);
}

float Stage::bench_sp(int iters, int mode) {
  if (!sp_) throw StepError{TP_ERR_UNSUPPORTED, "bench_sp: the session does not run sequence parallelism"};
  LayerActs& A = acts_for(0, 0);
  const LayerW W = w(0);
  auto launch = [&] {
    if (mode == 0) {
      SpLnFwdArgs f;
      f.nrows = Ms_, f.row0 = row0_, f.d = d_, f.seq = s_;
      f.y_off = woff(tmp_md_), f.bias = W.bo, f.resid = slots_act_[0].h[0];
      f.drop = drop_key(opts_, 1, 0, 0, 0, s_, d_);
      f.h_out = A.hmid, f.gamma = W.ln2g, f.beta = W.ln2b, f.ln_off = woff(A.m2), f.mean = A.mu2, f.rstd = A.rs2;
      sp_fwd(f);
    } else {
      SpLnBwdArgs g;
      g.nrows = Ms_, g.row0 = row0_, g.d = d_, g.workspace = ws_;
      g.dy_off = woff(dm_), g.x = A.hmid, g.gamma = W.ln2g, g.mean = A.mu2, g.rstd = A.rs2;
      g.resid_grad = dh_[0], g.dx = dh_[0];
      g.drop = drop_key(opts_, 1, 0, 0, 0, s_, d_);
      g.dxd_off = woff(dy_), g.dgamma = gr(0).ln2g, g.dbeta = gr(0).ln2b, g.dbias = gr(0).bo;
      sp_bwd(g);
    }
  };
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) launch();
  cudaEventRecord(a, st_);
  for (int i = 0; i < iters; ++i) launch();
  cudaEventRecord(b, st_);
  sync();
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return ms / std::max(iters, 1);
}

float Stage::allreduce_max(float v) {
  if (comms_.world == 1) return v;
  float* d = ws_;
  cudaMemcpyAsync(d, &v, sizeof(float), cudaMemcpyHostToDevice, st_);
  try {
    nccl_check(ncclAllReduce(d, d, 1, ncclFloat, ncclMax, comms_.world_comm, st_), "allreduce max");
  } catch (const CommError& e) {
    throw StepError{e.code, e.msg};
  }
  float out = 0.f;
  cudaMemcpyAsync(&out, d, sizeof(float), cudaMemcpyDeviceToHost, st_);
  sync();
  return out;
}

}  // namespace gptb200
