// Reference-side code using the B200 step through the reference's own API — the drop-in check.
//
// Written the way a `trainplan` user writes it: only <trainplan/*.hpp> headers, the reference's
// planner functions (run_search, estimate, calibrate, simulate, cluster costs, util) and the B200
// library's measured counterparts (train.hpp). tests/test_dropin.py compiles this translation unit
// twice — against this repo's restated headers alone, and with the reference's own include
// directory FIRST (so every reference header comes from /root/reference and only train.hpp /
// b200.hpp / capi.h from this repo) — and links libtrainplan_b200.so plus the reference library
// compiled from its sources (oracle/_ref/libtrainplan_ref.a, test infrastructure).
//
//   dropin_search cpu   planner-only calls (no GPU): run_search over the analytic evaluator,
//                       simulate, calibrate, memory_per_gpu, saturation_check, cluster costs
//   dropin_search gpu   run_search driven by make_measured_evaluator on this GPU, calibrate()
//                       fed the measured observations (-> a B200 kernel_efficiency), an OOM
//                       point, and the measured footprint next to memory_per_gpu at the 1.4B shape
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "trainplan/cluster.hpp"
#include "trainplan/memory.hpp"
#include "trainplan/metrics.hpp"
#include "trainplan/perf.hpp"
#include "trainplan/pipesim.hpp"
#include "trainplan/search.hpp"
#include "trainplan/train.hpp"
#include "trainplan/util.hpp"

using namespace trainplan;

static const char* kind_name(FailureKind k) {
  switch (k) {
    case FailureKind::None: return "none";
    case FailureKind::Oom: return "oom";
    case FailureKind::Invalid: return "invalid";
    case FailureKind::Timeout: return "timeout";
  }
  return "?";
}

static void print_history(const SearchResult& r) {
  std::printf("\"history\": [");
  for (size_t i = 0; i < r.history.size(); ++i) {
    const TrialRecord& t = r.history[i];
    std::printf("%s{\"pp\": %d, \"tp\": %d, \"mbs\": %d, \"gas\": %d, \"zero1\": %d, \"objective\": %.6g, "
                "\"failure\": \"%s\", \"wall_time\": %.6g}",
                i ? ", " : "", t.point.pp, t.point.tp, t.point.mbs, t.point.gas, t.point.zero1 ? 1 : 0, t.objective,
                kind_name(t.failure_kind), t.wall_time);
  }
  std::printf("], \"best_objective\": %.6g", r.best ? r.best->objective : -1.0);
}

static void print_mem(const char* name, const MemoryReport& m) {
  std::printf("\"%s\": {\"params\": %llu, \"gradients\": %llu, \"optimizer\": %llu, \"activations\": %llu, "
              "\"overhead\": %llu, \"total\": %llu, \"fits\": %d}",
              name, (unsigned long long)m.params_bytes, (unsigned long long)m.gradient_bytes,
              (unsigned long long)m.optimizer_bytes, (unsigned long long)m.activation_bytes,
              (unsigned long long)m.overhead_bytes, (unsigned long long)m.total_bytes, m.fits ? 1 : 0);
}

static int run_cpu() {
  const ModelSpec model{24, 2048, 16, 51200, 2048};
  const ClusterSpec cl = b200_preset(1, 8);
  SearchSpace space;
  space.pp = {1, 2};
  space.tp = {1, 2, 4};
  space.mbs_min = 1;
  space.mbs_max = 8;
  space.gas = {1, 2, 4};
  const SearchResult r = run_search(space, 12, make_estimate_evaluator(model, cl), 7, make_point_validator(model, cl), 1);
  std::printf("{");
  print_history(r);
  const auto tl = simulate(ScheduleKind::OneF1B, 2, 4, 1, StageTiming{});
  std::printf(", \"sim_events\": %zu, \"sim_bubble_ratio\": %.6g", tl.events.size(), tl.bubble_ratio);
  std::vector<ThroughputObservation> obs;
  for (int tp : {1, 2}) {
    ParallelConfig c;
    c.tp = tp, c.pp = 1, c.dp = 8 / tp, c.mbs = 4, c.gbs = 4 * (8 / tp), c.zero_stage = 1, c.flash_attention = true;
    ThroughputObservation o{model, c, cl, 0.0};
    EfficiencyKnobs k;
    k.kernel_efficiency = 0.42;
    o.measured_tflops_per_gpu = estimate(model, c, cl, k).flops_per_gpu / 1e12;
    obs.push_back(o);
  }
  std::printf(", \"calibrated_synthetic\": %.6g", calibrate(EfficiencyKnobs{}, obs).kernel_efficiency);
  ParallelConfig c;
  c.tp = 2, c.pp = 2, c.dp = 2, c.mbs = 1, c.gbs = 2, c.zero_stage = 1;
  const auto sat = saturation_check(c);
  std::printf(", \"saturation\": \"%s\"", sat ? sat->c_str() : "");
  std::printf(", ");
  print_mem("model_mem", memory_per_gpu(model, c, cl));
  ProcessGroup g{{GpuId{0, 0}, GpuId{0, 1}}, GroupKind::TP};
  std::printf(", \"allreduce_s\": %.6g, \"fmt\": \"%s\"}\n", allreduce_time(cl, g, 1e9), format_double(0.5).c_str());
  return 0;
}

static int run_gpu() {
  // 4 layers of the GPT-1.4B shape (d 2048, 16 heads, s 2048), reduced vocabulary: big enough that
  // the measured points sit in the regime the step model describes
  const ModelSpec tiny{4, 2048, 16, 8192, 2048};
  const ClusterSpec cl = b200_preset(1, 1);
  MeasureOptions mo;
  mo.warmup = 2;
  mo.steps = 3;
  mo.timeout_s = 120;
  SearchSpace space;  // one GPU: pp = tp = 1; tune mbs, gradient accumulation and ZeRO
  space.mbs_min = 1;
  space.mbs_max = 8;
  space.gas = {1, 2};
  const Evaluator ev = make_measured_evaluator(tiny, cl, mo);
  const SearchResult r = run_search(space, 6, ev, 11, make_point_validator(tiny, cl), 1);
  std::printf("{");
  print_history(r);
  // calibrate the reference's step model to the measured B200 points of this search
  std::vector<ThroughputObservation> obs;
  for (const TrialRecord& t : r.history) {
    if (t.failed()) continue;
    auto cfg = measured_config_from_point(t.point, cl);
    obs.push_back({tiny, *cfg, cl, t.objective});
  }
  const EfficiencyKnobs k = calibrate(EfficiencyKnobs{}, obs);
  std::printf(", \"observations\": %zu, \"calibrated_kernel_efficiency\": %.6g", obs.size(), k.kernel_efficiency);
  // a point whose parameters cannot fit: GPT-175B shape on one GPU
  const ModelSpec big{96, 12288, 96, 51200, 2048};
  const TrialRecord oom = make_measured_evaluator(big, cl, mo)(SearchPoint{1, 1, 1, 1, true, 1});
  std::printf(", \"oom_failure\": \"%s\"", kind_name(oom.failure_kind));
  // measured footprint vs the reference's model at the 1.4B shape (config 2, MBS 8, 1 GPU)
  const ModelSpec m14{24, 2048, 16, 51200, 2048};
  ParallelConfig c;
  c.tp = 1, c.pp = 1, c.dp = 1, c.mbs = 8, c.gbs = 8, c.zero_stage = 1;
  c.precision = Precision::BF16, c.grad_accum_dtype = GradAccumDtype::FP32, c.flash_attention = true;
  MemoryOptions adam;
  adam.optimizer_bytes_per_param = 8;  // m + v (the reference's default counts momentum only)
  std::printf(", \"executed_params\": %llu, ", (unsigned long long)executed_param_count(m14));
  print_mem("model_mem", memory_per_gpu(m14, c, cl, adam));
  std::printf(", ");
  print_mem("measured_mem", measured_memory_per_gpu(m14, c, cl));
  std::printf("}\n");
  return 0;
}

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
  return gpu ? run_gpu() : run_cpu();
}
