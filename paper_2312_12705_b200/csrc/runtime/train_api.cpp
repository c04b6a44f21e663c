// C++ drop-in layer (include/trainplan/train.hpp) on top of the C-ABI.
#include "trainplan/train.hpp"

#include <chrono>
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
  if (rc == TP_ERR_TIMEOUT) throw StepTimeout(msg);
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

void TrainSession::set_timeout(double seconds) { throw_for(tp_session_set_timeout(s_, seconds), "set_timeout"); }

MemoryReport TrainSession::memory_report(std::uint64_t mem_per_gpu) {
  tp_memory_report m{};
  throw_for(tp_session_memory(s_, &m), "memory_report");
  MemoryReport r;
  r.params_bytes = m.params_bytes;
  r.gradient_bytes = m.gradient_bytes;
  r.optimizer_bytes = m.optimizer_bytes;
  r.activation_bytes = m.activation_bytes;
  r.total_bytes = m.total_bytes;
  const std::uint64_t named = r.params_bytes + r.gradient_bytes + r.optimizer_bytes + r.activation_bytes;
  r.overhead_bytes = r.total_bytes > named ? r.total_bytes - named : 0;  // workspace + unused window
  r.fits = mem_per_gpu == 0 || r.total_bytes <= mem_per_gpu;
  return r;
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
  float ms = 0.f, ms_prof = 0.f;
  tp_kernel_times kt{};
  try {
    TrainSession sess(model, rc, opts.train, opts.dist);
    if (opts.timeout_s > 0) sess.set_timeout(opts.timeout_s);
    sess.init_params();
    const auto tokens = synthetic_tokens(opts.train.seed, static_cast<std::int64_t>(rc.gbs) * (model.seq_length + 1),
                                         model.vocab_size);
    sess.upload(tokens.data(), tokens.size());
    if (opts.warmup > 0) sess.time_steps(opts.warmup);
    ms = sess.allreduce_max(sess.time_steps(opts.steps));
    ms_prof = sess.time_steps(opts.steps, &kt);
  } catch (const std::bad_alloc&) {
    est.oom = true;  // a reported state wherever the allocation failed (perf.cpp:49-53)
    return est;
  }
  est.iter_time = ms / 1e3 / opts.steps;
  const double flops = model_flops_per_iteration(model, rc.gbs, rc.checkpoint_activations);
  est.flops_per_gpu = flops / (est.iter_time * cluster.world_size());
  est.peak_fraction = cluster.peak_flops_per_gpu > 0 ? est.flops_per_gpu / cluster.peak_flops_per_gpu : 0.0;
  const double scale = est.iter_time / (ms_prof / 1e3 / opts.steps);  // profiled pass -> timed pass
  auto sec = [&](int k) { return kt.ms[k] / 1e3 / opts.steps * scale; };
  est.breakdown.tp_comm = sec(5);
  est.breakdown.pp_comm = sec(6);
  // class 7 (the DP collectives on the comm stream) overlaps backward; what the step waits for is
  // the exposed optimizer-pipeline tail (class 8), reported as dp_comm when there is a DP group
  const bool dp_group = rc.dp > 1;
  est.breakdown.dp_comm = dp_group ? sec(8) : 0.0;
  est.breakdown.compute = sec(0) + sec(1) + sec(2) + sec(3) + sec(4) + (dp_group ? 0.0 : sec(8));
  est.breakdown.bubble = std::max(0.0, est.iter_time - est.breakdown.compute - est.breakdown.tp_comm -
                                           est.breakdown.pp_comm - est.breakdown.dp_comm);
  return est;
}

MemoryReport measured_memory_per_gpu(const ModelSpec& model, const ParallelConfig& cfg, const ClusterSpec& cluster,
                                     const DistributedContext& dist) {
  ValidationResult val = validate(model, cfg, cluster);
  if (val.ok) validate_kernels(model, val.resolved, val);
  if (!val.ok) throw std::invalid_argument("unvalidated configuration: " + val.hard_violations().front().message);
  try {
    TrainSession sess(model, val.resolved, TrainOptions{}, dist);
    return sess.memory_report(cluster.mem_per_gpu);
  } catch (const std::bad_alloc&) {
    return MemoryReport{};  // fits = false
  }
}

std::optional<ParallelConfig> measured_config_from_point(const SearchPoint& point, const ClusterSpec& base) {
  auto cfg = config_from_point(point, base);  // the reference's mapping (perf.cpp:161-181) ...
  if (cfg) {                                  // ... computed in bf16 with fp32 main grads
    cfg->precision = Precision::BF16;
    cfg->grad_accum_dtype = GradAccumDtype::FP32;
  }
  return cfg;
}

Evaluator make_measured_evaluator(const ModelSpec& model, const ClusterSpec& base, const MeasureOptions& opts) {
  return [model, base, opts](const SearchPoint& point) {
    const auto t0 = std::chrono::steady_clock::now();
    TrialRecord rec;
    rec.point = point;
    const auto cfg = measured_config_from_point(point, base);
    ClusterSpec cluster = base;
    cluster.num_nodes = point.nodes;
    ValidationResult val;
    if (cfg) {
      val = validate(model, *cfg, cluster);
      if (val.ok) validate_kernels(model, val.resolved, val);
    }
    if (!cfg || !val.ok) {
      rec.failure_kind = FailureKind::Invalid;
    } else {
      try {
        const ThroughputEstimate est = measure(model, *cfg, cluster, opts);
        if (est.oom)
          rec.failure_kind = FailureKind::Oom;
        else
          rec.objective = est.flops_per_gpu / 1e12;
      } catch (const std::bad_alloc&) {
        rec.failure_kind = FailureKind::Oom;
      } catch (const StepTimeout&) {
        rec.failure_kind = FailureKind::Timeout;
      } catch (const std::exception&) {  // invalid argument or a CUDA / NCCL failure: the point does not run
        rec.failure_kind = FailureKind::Invalid;
      }
    }
    rec.wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
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
