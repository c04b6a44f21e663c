// Test driver: the record format of oracle/ref_metrics.cpp answered by THIS library's restated
// diagnose_mbs_mismatch / roofline / weak_scaling / strong_scaling (include/trainplan/metrics.hpp);
// tests/test_metrics.py compares the two outputs byte for byte. Records on stdin:
//   D model_tflops hw_tflops cfg_mbs ds_mbs
//   R flops bytes peak hbm
//   W|S n g0 v0 g1 v1 ...
#include <cstdio>
#include <iostream>
#include <string>
#include <vector>

#include "trainplan/b200_metrics.hpp"

int main() {
  std::string tag;
  while (std::cin >> tag) {
    if (tag == "D") {
      double m, h;
      int c, d;
      std::cin >> m >> h >> c >> d;
      auto r = trainplan::diagnose_mbs_mismatch(m, h, c, d);
      std::printf("{\"kind\": %d, \"flops_ratio\": %.17g, \"message\": \"%s\"}\n", static_cast<int>(r.kind),
                  r.flops_ratio, r.message.c_str());
    } else if (tag == "R") {
      double f, b;
      trainplan::ClusterSpec cl;
      std::cin >> f >> b >> cl.peak_flops_per_gpu >> cl.hbm_bandwidth;
      auto r = trainplan::roofline(f, b, cl);
      std::printf("{\"ai\": %.17g, \"ridge\": %.17g, \"bound\": %d}\n", r.arithmetic_intensity, r.ridge_intensity,
                  static_cast<int>(r.bound));
    } else {
      int n;
      std::cin >> n;
      std::vector<trainplan::ScalingPoint> s(n);
      for (auto& p : s) std::cin >> p.gpus >> p.value;
      auto e = tag == "W" ? trainplan::weak_scaling(s) : trainplan::strong_scaling(s);
      std::printf("{\"eff\": [");
      for (size_t i = 0; i < e.size(); ++i) std::printf("%s%.17g", i ? ", " : "", e[i]);
      std::printf("]}\n");
    }
  }
  return 0;
}
