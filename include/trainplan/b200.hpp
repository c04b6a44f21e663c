// B200 additions to the trainplan API: what the executed step needs beyond the reference's
// declarations (which live, restated, in arch/cluster/memory/search/pipesim/perf/metrics.hpp and
// can equally come from the reference's own include directory). Everything here is defined by
// libtrainplan_b200.so (csrc/plan/plan.cpp).
#pragma once

#include <cstdint>
#include <vector>

#include "trainplan/arch.hpp"
#include "trainplan/cluster.hpp"
#include "trainplan/memory.hpp"
#include "trainplan/pipesim.hpp"
#include "trainplan/search.hpp"

namespace trainplan {

// Parameters of the executed network: 12 L d^2 + 13 L d + V d + s d + 2 d (param_count's
// convention plus W_o, biases and LayerNorms).
std::uint64_t executed_param_count(const ModelSpec& spec);

// One 8x B200 NVLink-5 / NVSwitch box: 180 GB HBM3e, 2.25 PFLOP/s dense bf16, 900 GB/s per
// direction to every peer (uniform tiers), 8 TB/s HBM.
ClusterSpec b200_preset(int num_nodes = 1, int gpus_per_node = 8);

// Hard constraints of the B200 kernels (head dim 64/128/160, vocab and head split over TP, GEMM
// and attention tile divisibility, bf16 compute, ZeRO stage <= 1, interleaving needs PP).
// Appends violations to `res` (and clears res.ok on any).
void validate_kernels(const ModelSpec& model, const ParallelConfig& cfg, ValidationResult& res);

// Megatron rank layout of the reference (perf.cpp:15-20): rank = t + tp * (p + pp * d).
struct RankCoords {
  int t = 0, p = 0, d = 0;
};
RankCoords rank_coords(int rank, const ParallelConfig& resolved);
int rank_of(const RankCoords& c, const ParallelConfig& resolved);

// One pipeline op of a device's schedule.
struct PipeOp {
  bool backward = false;
  int microbatch = 0;
  int chunk = 0;
  friend bool operator==(const PipeOp&, const PipeOp&) = default;
};

// Per-device execution order, identical to the order the reference's simulate() runs
// (pipesim.cpp:31-91): 1F1B warm-up min(p-1-device, m) forwards, F/B pairs, cool-down backwards;
// GPipe; interleaved 1F1B. This is the order the executor follows.
std::vector<PipeOp> pipeline_order(ScheduleKind kind, int p, int m, int v, int device);

}  // namespace trainplan
