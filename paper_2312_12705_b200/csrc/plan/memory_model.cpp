// The reference's footprint model and the small perf.hpp helpers the step path uses, restated
// (semantics per function citation; tests/test_memory_model.py compares every result with the
// reference library compiled from its own sources). The executed step's MEASURED footprint in the
// same categories is TrainSession::memory_report (runtime/train_api.cpp).
#include <stdexcept>
#include <string>

#include "trainplan/b200.hpp"
#include "trainplan/perf.hpp"

namespace trainplan {

namespace {

using u64 = std::uint64_t;
using u128 = unsigned __int128;

u64 div_up(u64 a, u64 b) { return (a + b - 1) / b; }

}  // namespace

// arch.cpp:94-101 — 6 N D, exact in 128 bits.
double training_budget(std::uint64_t params, std::uint64_t tokens) {
  const u128 n = static_cast<u128>(params) * 6u;
  if (params != 0 && n / 6u != params) throw std::overflow_error("training budget overflows 128 bits");
  if (tokens != 0 && n > ~u128{0} / tokens) throw std::overflow_error("training budget overflows 128 bits");
  return static_cast<double>(n * tokens);
}

double training_budget(const ModelSpec& spec, std::uint64_t tokens) {
  return training_budget(param_count(spec).total_approx, tokens);
}

// memory.cpp:30-39
BytesPerParam bytes_per_param(Precision precision) {
  if (precision == Precision::FP32) return {4, 4, 4};
  if (precision == Precision::FP16 || precision == Precision::BF16) return {6, 4, 4};
  throw std::invalid_argument("unknown precision");
}

// memory.cpp:41-60 — per layer 34 s b d + 5 a s^2 b bytes (2-byte activations); checkpointing keeps
// the 2 s b d layer inputs of the stage plus one layer's working set; both divided by tp.
std::uint64_t activation_bytes(const ModelSpec& model, const ParallelConfig& cfg) {
  if (cfg.tp < 1 || cfg.pp < 1 || cfg.mbs < 0) throw std::invalid_argument("unvalidated configuration");
  if (cfg.mbs == 0) return 0;
  const u64 s = static_cast<u64>(model.seq_length), d = static_cast<u64>(model.hidden_size),
            a = static_cast<u64>(model.num_heads), b = static_cast<u64>(cfg.mbs), tp = static_cast<u64>(cfg.tp);
  const u64 layers = div_up(static_cast<u64>(model.num_layers), static_cast<u64>(cfg.pp));
  const u64 layer_set = s * b * (34 * d + 5 * a * s);
  if (!cfg.checkpoint_activations) return div_up(layer_set * layers, tp);
  return div_up(2 * s * b * d * layers + layer_set, tp);
}

// memory.cpp:62-93 — params / grads / optimizer bytes over the TP x PP shard, ZeRO stage k shards
// the first k of (optimizer, gradients, params) over DP; fp32 gradient accumulation under a half
// precision adds 4 B/param.
MemoryReport memory_per_gpu_for_params(std::uint64_t total_params, const ModelSpec& model, const ParallelConfig& cfg,
                                       const ClusterSpec& cluster, const MemoryOptions& opts) {
  if (cfg.tp < 1 || cfg.pp < 1 || cfg.dp < 1 || cfg.mbs < 0 || cfg.gbs < 1 || cfg.interleave_v < 1 ||
      cfg.zero_stage < 0 || cfg.zero_stage > 3)
    throw std::invalid_argument("unvalidated configuration");
  BytesPerParam bpp = bytes_per_param(cfg.precision);
  if (opts.optimizer_bytes_per_param > 0) bpp.optim_b = opts.optimizer_bytes_per_param;
  const bool fp32_accum = cfg.grad_accum_dtype == GradAccumDtype::FP32 && cfg.precision != Precision::FP32;
  const u64 grad_b = static_cast<u64>(bpp.grad_b) + (fp32_accum ? 4 : 0);
  const u64 shards = static_cast<u64>(cfg.tp) * static_cast<u64>(cfg.pp), dp = static_cast<u64>(cfg.dp);
  MemoryReport r;
  r.params_bytes = div_up(total_params * static_cast<u64>(bpp.param_b), shards);
  r.gradient_bytes = div_up(total_params * grad_b, shards);
  r.optimizer_bytes = div_up(total_params * static_cast<u64>(bpp.optim_b), shards);
  if (cfg.zero_stage >= 1) r.optimizer_bytes = div_up(r.optimizer_bytes, dp);
  if (cfg.zero_stage >= 2) r.gradient_bytes = div_up(r.gradient_bytes, dp);
  if (cfg.zero_stage >= 3) r.params_bytes = div_up(r.params_bytes, dp);
  r.activation_bytes = opts.include_activations ? activation_bytes(model, cfg) : 0;
  r.overhead_bytes = opts.framework_overhead_bytes;
  r.total_bytes = r.params_bytes + r.gradient_bytes + r.optimizer_bytes + r.activation_bytes + r.overhead_bytes;
  r.fits = r.total_bytes <= cluster.mem_per_gpu;
  return r;
}

// memory.cpp:95-98
MemoryReport memory_per_gpu(const ModelSpec& model, const ParallelConfig& cfg, const ClusterSpec& cluster,
                            const MemoryOptions& opts) {
  return memory_per_gpu_for_params(param_count(model).total_exact, model, cfg, cluster, opts);
}

// perf.cpp:151-159 — PAPER.md:526: fewer microbatches than stages leaves the pipeline unsaturated.
std::optional<std::string> saturation_check(const ParallelConfig& cfg) {
  if (cfg.pp <= 1) return std::nullopt;
  const int m = cfg.num_microbatches();
  if (m >= cfg.pp) return std::nullopt;
  return "pipeline unsaturated: " + std::to_string(m) + " microbatches for " + std::to_string(cfg.pp) +
         " stages; increase gbs or gradient accumulation";
}

// perf.cpp:161-181
std::optional<ParallelConfig> config_from_point(const SearchPoint& point, const ClusterSpec& base_cluster) {
  ClusterSpec cluster = base_cluster;
  cluster.num_nodes = point.nodes;
  const long long world = cluster.world_size(), shards = static_cast<long long>(point.tp) * point.pp;
  if (point.tp < 1 || point.pp < 1 || point.mbs < 1 || point.gas < 1 || world % shards != 0) return std::nullopt;
  ParallelConfig cfg;
  cfg.tp = point.tp;
  cfg.pp = point.pp;
  cfg.dp = static_cast<int>(world / shards);
  cfg.mbs = point.mbs;
  cfg.gbs = point.mbs * point.gas * cfg.dp;
  cfg.zero_stage = point.zero1 ? 1 : 0;
  cfg.precision = Precision::FP16;
  cfg.checkpoint_activations = true;
  cfg.flash_attention = true;
  return cfg;
}

// perf.cpp:209-217
PointValidator make_point_validator(const ModelSpec& model, const ClusterSpec& base_cluster) {
  return [model, base_cluster](const SearchPoint& point) {
    const auto cfg = config_from_point(point, base_cluster);
    if (!cfg) return false;
    ClusterSpec cluster = base_cluster;
    cluster.num_nodes = point.nodes;
    return validate(model, *cfg, cluster).ok;
  };
}

}  // namespace trainplan
