// Drop-in C++ API exercise (GPU): TrainSession, measure() -> ThroughputEstimate, measured Evaluator.
#include <cstdio>
#include <stdexcept>

#include "trainplan/train.hpp"

using namespace trainplan;

int main() {
  ModelSpec m{2, 256, 4, 1024, 128};
  ClusterSpec cl = b200_preset(1, 1);
  ParallelConfig cfg;
  cfg.tp = 1, cfg.pp = 1, cfg.dp = 0, cfg.mbs = 2, cfg.gbs = 4, cfg.zero_stage = 1;
  cfg.precision = Precision::BF16, cfg.grad_accum_dtype = GradAccumDtype::FP32, cfg.flash_attention = true;
  MeasureOptions mo;
  mo.warmup = 2, mo.steps = 3;
  ThroughputEstimate est = measure(m, cfg, cl, mo);
  const auto& b = est.breakdown;
  std::printf("{\"iter_time\": %.9g, \"flops_per_gpu\": %.9g, \"peak_fraction\": %.9g, \"oom\": %d, "
              "\"compute\": %.9g, \"tp\": %.9g, \"pp\": %.9g, \"dp\": %.9g, \"bubble\": %.9g,\n",
              est.iter_time, est.flops_per_gpu, est.peak_fraction, est.oom ? 1 : 0, b.compute, b.tp_comm, b.pp_comm,
              b.dp_comm, b.bubble);
  int invalid = 0;
  try {
    ParallelConfig bad = cfg;
    bad.tp = 3;
    measure(m, bad, cl, mo);
  } catch (const std::invalid_argument&) {
    invalid = 1;
  }
  Evaluator ev = make_measured_evaluator(m, cl, mo);
  TrialRecord ok = ev(SearchPoint{1, 1, 2, 2, true, 1});
  TrialRecord inv = ev(SearchPoint{1, 3, 1, 1, false, 1});
  TrainSession s(m, cfg);
  s.init_params();
  std::vector<int32_t> toks(4 * 129);
  for (size_t i = 0; i < toks.size(); ++i) toks[i] = static_cast<int32_t>((i * 7919) % 1024);
  float l0 = s.train_step(toks), l1 = 0;
  for (int i = 0; i < 5; ++i) l1 = s.train_step(toks);
  std::printf("\"invalid_throws\": %d, \"eval_ok_tflops\": %.6g, \"eval_ok_failed\": %d, \"eval_invalid_kind\": %d, "
              "\"loss0\": %.6f, \"loss5\": %.6f, \"log\": \"%s\"}\n",
              invalid, ok.objective, ok.failed() ? 1 : 0, static_cast<int>(inv.failure_kind), l0, l1,
              megatron_log_line(6, 10, est, 1e-4, l1, cfg.gbs).c_str());
  return 0;
}
