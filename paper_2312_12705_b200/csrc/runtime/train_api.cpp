// C++ drop-in layer (include/trainplan/train.hpp) on top of the C-ABI.
#include "trainplan/train.hpp"

#include <cstdio>
#include <new>
#include <random>
#include <stdexcept>

namespace trainplan {

namespace {

void throw_for(int rc, const char* where) {
  if (rc == TP_OK) return;
  std::string msg = std::string(where) + ": " + tp_last_error();
  if (rc == TP_ERR_INVALID) throw std::invalid_argument(msg);
  if (rc == TP_ERR_OOM) throw std::bad_alloc();
  throw std::runtime_error(msg);
}

tp_model_spec to_c(const ModelSpec& m) {
  return {m.num_layers, m.hidden_size, m.num_heads, m.vocab_size, m.seq_length};
}

tp_parallel_config to_c(const ParallelConfig& c) {
  tp_parallel_config o{};
  o.tp = c.tp;
  o.pp = c.pp;
  o.dp = c.dp;
  o.mbs = c.mbs;
  o.gbs = c.gbs;
  o.zero_stage = c.zero_stage;
  o.interleave_v = c.interleave_v;
  o.precision = c.precision == Precision::BF16 ? 1 : (c.precision == Precision::FP32 ? 2 : 0);
  o.grad_accum_fp32 = c.grad_accum_dtype == GradAccumDtype::FP32 ? 1 : 0;
  o.checkpoint_activations = c.checkpoint_activations ? 1 : 0;
  o.flash_attention = c.flash_attention ? 1 : 0;
  return o;
}

std::vector<std::int32_t> synthetic_tokens(std::uint64_t seed, std::int64_t n, int vocab) {
  std::mt19937_64 gen(seed);
  std::vector<std::int32_t> t(static_cast<std::size_t>(n));
  for (auto& x : t) x = static_cast<std::int32_t>(gen() % static_cast<std::uint64_t>(vocab));
  return t;
}

}  // namespace

std::array<unsigned char, 128> nccl_unique_id() {
  std::array<unsigned char, 128> id{};
  throw_for(tp_nccl_unique_id(id.data()), "nccl_unique_id");
  return id;
}

TrainSession::TrainSession(const ModelSpec& model, const ParallelConfig& cfg, const TrainOptions& o,
                           const DistributedContext& dist) {
  const tp_model_spec m = to_c(model);
  const tp_parallel_config c = to_c(cfg);
  const tp_train_options t{o.seed, o.dropout, o.lr, o.beta1, o.beta2, o.eps, o.weight_decay};
  throw_for(tp_session_create(&m, &c, &t, dist.rank, dist.world, dist.device,
                              dist.nccl_id ? dist.nccl_id->data() : nullptr, &s_),
            "TrainSession");
}

TrainSession::~TrainSession() {
  if (s_) tp_session_destroy(s_);
}

TrainSession::TrainSession(TrainSession&& o) noexcept : s_(o.s_) { o.s_ = nullptr; }

void TrainSession::init_params() { throw_for(tp_session_init_params(s_), "init_params"); }

float TrainSession::train_step(const std::vector<std::int32_t>& tokens) {
  float l = 0.f;
  throw_for(tp_session_train_step(s_, tokens.data(), static_cast<std::int64_t>(tokens.size()), &l), "train_step");
  return l;
}

void TrainSession::upload(const std::int32_t* tokens, std::size_t n) {
  throw_for(tp_session_upload_tokens(s_, tokens, static_cast<std::int64_t>(n), 0), "upload");
}

void TrainSession::step() { throw_for(tp_session_step(s_), "step"); }

float TrainSession::loss() {
  float l = 0.f;
  throw_for(tp_session_read_loss(s_, &l), "loss");
  return l;
}

float TrainSession::time_steps(int steps, tp_kernel_times* kt) {
  float ms = 0.f;
  tp_kernel_times tmp;
  throw_for(tp_session_time_steps(s_, steps, kt != nullptr, &ms, kt ? kt : &tmp), "time_steps");
  return ms;
}

float TrainSession::allreduce_max(float v) {
  throw_for(tp_session_allreduce_max(s_, &v), "allreduce_max");
  return v;
}

ThroughputEstimate measure(const ModelSpec& model, const ParallelConfig& cfg, const ClusterSpec& cluster,
                           const MeasureOptions& opts) {
  ValidationResult val = validate(model, cfg, cluster);
  if (val.ok) validate_kernels(model, val.resolved, val);
  if (!val.ok) throw std::invalid_argument("unvalidated configuration: " + val.hard_violations().front().message);
  const ParallelConfig rc = val.resolved;
  ThroughputEstimate est;
  std::optional<TrainSession> sess;
  try {
    sess.emplace(model, rc, opts.train, opts.dist);
  } catch (const std::bad_alloc&) {
    est.oom = true;  // a reported state, as in the reference (perf.cpp:49-53)
    return est;
  }
  sess->init_params();
  const auto tokens = synthetic_tokens(opts.train.seed, static_cast<std::int64_t>(rc.gbs) * (model.seq_length + 1),
                                       model.vocab_size);
  sess->upload(tokens.data(), tokens.size());
  if (opts.warmup > 0) sess->time_steps(opts.warmup);
  const float ms = sess->allreduce_max(sess->time_steps(opts.steps));
  tp_kernel_times kt{};
  const float ms_prof = sess->time_steps(opts.steps, &kt);
  est.iter_time = ms / 1e3 / opts.steps;
  const double flops = model_flops_per_iteration(model, rc.gbs, rc.checkpoint_activations);
  est.flops_per_gpu = flops / (est.iter_time * cluster.world_size());
  est.peak_fraction = cluster.peak_flops_per_gpu > 0 ? est.flops_per_gpu / cluster.peak_flops_per_gpu : 0.0;
  const double scale = est.iter_time / (ms_prof / 1e3 / opts.steps);  // profiled pass -> timed pass
  auto sec = [&](int k) { return kt.ms[k] / 1e3 / opts.steps * scale; };
  est.breakdown.tp_comm = sec(5);
  est.breakdown.pp_comm = sec(6);
  est.breakdown.dp_comm = sec(7);
  est.breakdown.compute = sec(0) + sec(1) + sec(2) + sec(3) + sec(4) + sec(8);
  est.breakdown.bubble = std::max(0.0, est.iter_time - est.breakdown.compute - est.breakdown.tp_comm -
                                           est.breakdown.pp_comm - est.breakdown.dp_comm);
  return est;
}

std::optional<ParallelConfig> measured_config_from_point(const SearchPoint& point, const ClusterSpec& base) {
  ClusterSpec cluster = base;
  cluster.num_nodes = point.nodes;
  const long long world = cluster.world_size();
  const long long shards = static_cast<long long>(point.tp) * point.pp;
  if (point.tp < 1 || point.pp < 1 || point.mbs < 1 || point.gas < 1 || world % shards != 0) return std::nullopt;
  ParallelConfig cfg;
  cfg.tp = point.tp;
  cfg.pp = point.pp;
  cfg.dp = static_cast<int>(world / shards);
  cfg.mbs = point.mbs;
  cfg.gbs = point.mbs * point.gas * cfg.dp;
  cfg.zero_stage = point.zero1 ? 1 : 0;
  cfg.precision = Precision::BF16;
  cfg.grad_accum_dtype = GradAccumDtype::FP32;
  cfg.checkpoint_activations = true;
  cfg.flash_attention = true;
  return cfg;
}

Evaluator make_measured_evaluator(const ModelSpec& model, const ClusterSpec& base, const MeasureOptions& opts) {
  return [model, base, opts](const SearchPoint& point) {
    TrialRecord rec;
    rec.point = point;
    const auto cfg = measured_config_from_point(point, base);
    ClusterSpec cluster = base;
    cluster.num_nodes = point.nodes;
    if (!cfg || !validate(model, *cfg, cluster).ok) {
      rec.failure_kind = FailureKind::Invalid;
      return rec;
    }
    try {
      const ThroughputEstimate est = measure(model, *cfg, cluster, opts);
      if (est.oom) {
        rec.failure_kind = FailureKind::Oom;
        return rec;
      }
      rec.objective = est.flops_per_gpu / 1e12;
      rec.wall_time = est.iter_time * (opts.warmup + 2 * opts.steps);
    } catch (const std::invalid_argument&) {
      rec.failure_kind = FailureKind::Invalid;
    }
    return rec;
  };
}

std::string megatron_log_line(long iteration, long total, const ThroughputEstimate& est, double lr, float loss,
                              long global_batch) {
  char buf[512];
  std::snprintf(buf, sizeof(buf),
                " iteration %8ld/%8ld | consumed samples: %12ld | elapsed time per iteration (ms): %.1f | "
                "learning rate: %.3E | global batch size: %5ld | lm loss: %.6E | TFLOPs: %.2f |",
                iteration, total, iteration * global_batch, est.iter_time * 1e3, lr, global_batch,
                static_cast<double>(loss), est.flops_per_gpu / 1e12);
  return buf;
}

}  // namespace trainplan
