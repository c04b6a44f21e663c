// Prints one megatron_log_line for a synthetic ThroughputEstimate (CPU; no GPU needed).
#include <cstdio>
#include <cstdlib>

#include "trainplan/train.hpp"

int main(int argc, char** argv) {
  trainplan::ThroughputEstimate est;
  est.iter_time = std::atof(argv[1]);
  est.flops_per_gpu = std::atof(argv[2]);
  for (long it = 1; it <= 3; ++it)
    std::printf("%s\n", trainplan::megatron_log_line(it, 3, est, 1e-4, 2.5f, 64).c_str());
  return 0;
}
