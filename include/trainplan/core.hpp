// trainplan public types and structural functions for the GPT train-step hot path.
//
// This is the subset of the reference API (/root/reference/proj/include/trainplan/*.hpp) that
// the train step sits behind, restated so that code written against the reference compiles
// unchanged against this library: same namespace, type names, field names, defaults and
// error conventions. The per-header forwarding files (arch.hpp, memory.hpp, cluster.hpp,
// search.hpp, pipesim.hpp, perf.hpp) include this file.
//
// Reference anchors:
//   ModelSpec / param_count / model_flops_per_iteration   arch.hpp:10-48, src/arch.cpp:35-101
//   ParallelConfig / Precision / GradAccumDtype           memory.hpp:11-32, src/memory.cpp:20-28
//   ClusterSpec / GpuId / GroupKind                       cluster.hpp:11-44
//   Violation / ValidationResult / validate               search.hpp:14-35, src/search.cpp:23-84
//   ScheduleKind / 1F1B order                             pipesim.hpp:8, src/pipesim.cpp:41-91
//   ThroughputBreakdown / ThroughputEstimate              perf.hpp:18-32
//   SearchPoint / FailureKind / TrialRecord / Evaluator   search.hpp:47-78
#pragma once

#include <cstdint>
#include <functional>
#include <string>
#include <vector>

namespace trainplan {

// ---------------------------------------------------------------- model shape
struct ModelSpec {
  int num_layers = 1;   // L
  int hidden_size = 1;  // d
  int num_heads = 1;    // a
  int vocab_size = 1;   // V
  int seq_length = 1;   // s

  // Human-readable shape problems (positivity, d % a); empty when clean. Never throws.
  std::vector<std::string> validate() const;
};

// Exact split of the reference's parameter convention: QKV 3d^2 and FFN 8d^2 per layer plus
// tied embedding V*d and learned positions s*d; total_approx = 12*L*d^2. The executed model
// additionally carries W_o (d^2), biases and LayerNorm parameters per layer; see
// executed_param_count().
struct ParamBreakdown {
  std::uint64_t attention_params = 0;
  std::uint64_t ffn_params = 0;
  std::uint64_t embedding_params = 0;
  std::uint64_t total_exact = 0;
  std::uint64_t total_approx = 0;
};

ParamBreakdown param_count(const ModelSpec& spec);

// Parameters of the executed network: 12*L*d^2 + 13*L*d + V*d + s*d + 2*d.
std::uint64_t executed_param_count(const ModelSpec& spec);

// Model FLOPs of one iteration over batch_size sequences (the metric numerator):
// 24*c*B*s*L*d^2*(1 + s/(6d) + V/(16Ld)), c = checkpoint_factor with activation
// checkpointing, else 3. Exact in 128-bit integers; std::overflow_error on overflow,
// std::invalid_argument on a non-positive shape or bad factor.
double model_flops_per_iteration(const ModelSpec& spec, std::int64_t batch_size,
                                 bool checkpoint_activations, int checkpoint_factor = 4);

// ---------------------------------------------------------------- parallel layout
enum class Precision { FP16, BF16, FP32 };
enum class GradAccumDtype { FP16, FP32 };

struct ParallelConfig {
  int tp = 1;
  int pp = 1;
  int dp = 0;  // 0: derive from the cluster in validate()
  int mbs = 1;
  int gbs = 1;
  int zero_stage = 0;
  int interleave_v = 1;
  Precision precision = Precision::FP16;
  GradAccumDtype grad_accum_dtype = GradAccumDtype::FP16;
  bool checkpoint_activations = false;
  bool flash_attention = false;

  // gbs / (mbs * dp); std::invalid_argument while dp is unbound or mbs < 1.
  int num_microbatches() const;
};

// ---------------------------------------------------------------- cluster
struct ClusterSpec {
  int num_nodes = 1;
  int gpus_per_node = 8;
  std::uint64_t mem_per_gpu = 0;
  double peak_flops_per_gpu = 0.0;
  double bw_same_card = 0.0;
  double bw_intra_node = 0.0;
  double bw_inter_node = 0.0;
  double link_latency_intra = 0.0;
  double link_latency_inter = 0.0;
  double hbm_bandwidth = 0.0;

  int world_size() const { return num_nodes * gpus_per_node; }
};

struct GpuId {
  int node = 0;
  int local = 0;
  friend bool operator==(const GpuId&, const GpuId&) = default;
};

enum class GroupKind { TP, PP, DP };

// One 8x B200 NVLink-5/NVSwitch box: 180 GB HBM3e, 2.25 PFLOP/s dense bf16, 900 GB/s per
// direction to every peer (uniform tiers), 8 TB/s HBM.
ClusterSpec b200_preset(int num_nodes = 1, int gpus_per_node = 8);

// ---------------------------------------------------------------- validation
struct Violation {
  std::string field;
  std::string message;
  bool hard = true;
};

struct ValidationResult {
  std::vector<Violation> violations;
  ParallelConfig resolved;
  int num_microbatches = 0;
  bool ok = false;

  std::vector<Violation> hard_violations() const;
};

// The config gate of the reference (world factorization, L % pp, d % tp, a % tp, ZeRO-3 with
// PP, gbs % (mbs*dp); TP wider than a node is a soft warning). Never throws.
ValidationResult validate(const ModelSpec& model, const ParallelConfig& cfg,
                          const ClusterSpec& cluster);

// Additional hard constraints of the B200 kernels (vocab and head split, GEMM tile
// divisibility, head dim, activation-checkpointing support). Appends to `res`.
void validate_kernels(const ModelSpec& model, const ParallelConfig& cfg, ValidationResult& res);

// ---------------------------------------------------------------- rank layout
// Megatron-style rank order used by the reference (src/perf.cpp:15-20): tp fastest, then pp,
// then dp: rank = t + tp * (p + pp * d).
struct RankCoords {
  int t = 0, p = 0, d = 0;
};
RankCoords rank_coords(int rank, const ParallelConfig& resolved);
int rank_of(const RankCoords& c, const ParallelConfig& resolved);

// ---------------------------------------------------------------- pipeline schedule
enum class ScheduleKind { GPipe, OneF1B, Interleaved1F1B };

struct PipeOp {
  bool backward = false;
  int microbatch = 0;
  int chunk = 0;
  friend bool operator==(const PipeOp&, const PipeOp&) = default;
};

// Per-device execution order, identical to the order the reference simulates
// (src/pipesim.cpp:31-91): 1F1B warm-up min(p-1-device, m) forwards, then F/B pairs, then the
// cool-down backwards; GPipe all forwards then all backwards; interleaved per pipesim.
std::vector<PipeOp> pipeline_order(ScheduleKind kind, int p, int m, int v, int device);

// ---------------------------------------------------------------- step reports
struct ThroughputBreakdown {
  double compute = 0.0;
  double tp_comm = 0.0;
  double pp_comm = 0.0;
  double dp_comm = 0.0;
  double bubble = 0.0;
};

struct ThroughputEstimate {
  double iter_time = 0.0;
  double flops_per_gpu = 0.0;
  double peak_fraction = 0.0;
  ThroughputBreakdown breakdown;
  bool oom = false;
};

// ---------------------------------------------------------------- search plumbing
struct SearchPoint {
  int pp = 1;
  int tp = 1;
  int mbs = 1;
  int gas = 1;
  bool zero1 = false;
  int nodes = 1;
  friend bool operator==(const SearchPoint&, const SearchPoint&) = default;
};

enum class FailureKind { None, Oom, Invalid, Timeout };

struct TrialRecord {
  SearchPoint point;
  double objective = 0.0;  // TFLOPS/GPU
  FailureKind failure_kind = FailureKind::None;
  double wall_time = 0.0;
  bool failed() const { return failure_kind != FailureKind::None; }
};

using Evaluator = std::function<TrialRecord(const SearchPoint&)>;
using PointValidator = std::function<bool(const SearchPoint&)>;

}  // namespace trainplan
