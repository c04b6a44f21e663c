// Structural oracle driver — TEST INFRASTRUCTURE ONLY. Feeds stdin to the reference's own
// parse_training_log / aggregate_model_flops (proj/src/metrics.cpp:119-162) and prints the result.
#include <cstdio>
#include <iostream>

#include "trainplan/metrics.hpp"

int main() {
  auto log = trainplan::parse_training_log(std::cin);
  std::printf("{\"entries\": %zu, \"aggregate_tflops\": %.9g, \"first_iter_time\": %.9g, \"first_iteration\": %ld}\n",
              log.size(), trainplan::aggregate_model_flops(log), log.empty() ? 0.0 : log[0].iter_time,
              log.empty() ? -1L : log[0].iteration);
  return 0;
}
