// Structural oracle driver — TEST INFRASTRUCTURE ONLY.
//
// Links the reference library compiled from /root/reference/proj/src (oracle/Makefile, output in
// oracle/_ref/) and prints, as JSON, the reference's own answers for the structural half of the
// hot path: param_count (proj/src/arch.cpp:48-62), model_flops_per_iteration (arch.cpp:64-92),
// validate (proj/src/search.cpp:23-84) and the per-device 1F1B / interleaved order exposed by
// simulate (proj/src/pipesim.cpp:41-91,113-210). tests/golden/make_ref_structural.py runs it and
// commits the JSON as tests/golden/ref_structural.json; the product's C++ plan layer must match it.
#include <cstdio>
#include <sstream>
#include <string>
#include <vector>

#include "trainplan/arch.hpp"
#include "trainplan/cluster.hpp"
#include "trainplan/memory.hpp"
#include "trainplan/pipesim.hpp"
#include "trainplan/search.hpp"

using namespace trainplan;

static std::string spec_json(const ModelSpec& m) {
  std::ostringstream o;
  o << "[" << m.num_layers << "," << m.hidden_size << "," << m.num_heads << "," << m.vocab_size
    << "," << m.seq_length << "]";
  return o.str();
}

int main() {
  std::vector<ModelSpec> specs = {
      {2, 256, 4, 51200, 128},   {2, 256, 4, 1024, 128},     {24, 2048, 16, 51200, 2048},
      {48, 6144, 48, 51200, 2048}, {96, 12288, 96, 51200, 2048}, {8, 12288, 96, 51200, 2048},
      {128, 25600, 160, 51200, 2048}, {4, 25600, 160, 51200, 2048}, {1, 1, 1, 1, 1}};
  std::printf("{\n\"param_count\": [\n");
  for (size_t i = 0; i < specs.size(); ++i) {
    auto p = param_count(specs[i]);
    std::printf("  {\"spec\": %s, \"attention\": %llu, \"ffn\": %llu, \"embedding\": %llu, "
                "\"total_exact\": %llu, \"total_approx\": %llu}%s\n",
                spec_json(specs[i]).c_str(), (unsigned long long)p.attention_params,
                (unsigned long long)p.ffn_params, (unsigned long long)p.embedding_params,
                (unsigned long long)p.total_exact, (unsigned long long)p.total_approx,
                i + 1 < specs.size() ? "," : "");
  }
  std::printf("],\n\"model_flops\": [\n");
  bool first = true;
  for (auto& s : specs)
    for (long long B : {0LL, 1LL, 8LL, 64LL, 640LL})
      for (int ck : {0, 1}) {
        double f = model_flops_per_iteration(s, B, ck != 0);
        std::printf("%s  {\"spec\": %s, \"batch\": %lld, \"ckpt\": %d, \"flops\": %.17g}",
                    first ? "" : ",\n", spec_json(s).c_str(), B, ck, f);
        first = false;
      }
  std::printf("\n],\n\"validate\": [\n");
  struct Case {
    ModelSpec m;
    int tp, pp, dp, mbs, gbs, zero, world;
  };
  std::vector<Case> cases = {
      {{2, 256, 4, 51200, 128}, 2, 2, 2, 1, 8, 1, 8},
      {{2, 256, 4, 51200, 128}, 2, 2, 0, 1, 8, 1, 8},
      {{24, 2048, 16, 51200, 2048}, 1, 1, 1, 8, 8, 1, 1},
      {{24, 2048, 16, 51200, 2048}, 1, 1, 0, 8, 64, 1, 8},
      {{48, 6144, 48, 51200, 2048}, 2, 1, 0, 1, 32, 1, 8},
      {{48, 6144, 48, 51200, 2048}, 8, 1, 0, 1, 8, 1, 8},
      {{8, 12288, 96, 51200, 2048}, 4, 2, 0, 1, 16, 1, 8},
      {{4, 25600, 160, 51200, 2048}, 8, 1, 0, 1, 8, 1, 8},
      {{4, 25600, 160, 51200, 2048}, 4, 2, 0, 1, 8, 1, 8},
      {{24, 2048, 16, 51200, 2048}, 3, 1, 0, 1, 8, 1, 8},
      {{24, 2048, 16, 51200, 2048}, 1, 5, 0, 1, 8, 1, 5},
      {{24, 2048, 16, 51200, 2048}, 1, 2, 0, 1, 8, 3, 8},
      {{24, 2048, 16, 51200, 2048}, 1, 1, 0, 3, 8, 1, 8},
      {{24, 2048, 16, 51200, 2048}, 2, 2, 3, 1, 24, 1, 8},
      {{24, 2048, 16, 51200, 2048}, 16, 1, 0, 1, 16, 1, 16},
      {{24, 2048, 16, 51200, 2048}, 0, 1, 0, 1, 8, 1, 8},
  };
  for (size_t i = 0; i < cases.size(); ++i) {
    const Case& c = cases[i];
    ParallelConfig cfg;
    cfg.tp = c.tp;
    cfg.pp = c.pp;
    cfg.dp = c.dp;
    cfg.mbs = c.mbs;
    cfg.gbs = c.gbs;
    cfg.zero_stage = c.zero;
    ClusterSpec cl;
    cl.num_nodes = 1;
    cl.gpus_per_node = c.world > 8 ? 8 : c.world;
    if (c.world > 8) cl.num_nodes = c.world / 8;
    auto r = validate(c.m, cfg, cl);
    std::printf("  {\"spec\": %s, \"cfg\": [%d,%d,%d,%d,%d,%d], \"nodes\": %d, \"gpn\": %d, "
                "\"ok\": %d, \"dp\": %d, \"m\": %d, \"fields\": [",
                spec_json(c.m).c_str(), c.tp, c.pp, c.dp, c.mbs, c.gbs, c.zero, cl.num_nodes,
                cl.gpus_per_node, r.ok ? 1 : 0, r.resolved.dp, r.num_microbatches);
    for (size_t j = 0; j < r.violations.size(); ++j)
      std::printf("%s[\"%s\", %d]", j ? ", " : "", r.violations[j].field.c_str(),
                  r.violations[j].hard ? 1 : 0);
    std::printf("]}%s\n", i + 1 < cases.size() ? "," : "");
  }
  std::printf("],\n\"schedules\": [\n");
  first = true;
  struct Sch {
    int p, m, v;
  };
  std::vector<Sch> sch = {{1, 4, 1}, {2, 4, 1},  {2, 16, 1}, {4, 8, 1}, {4, 3, 1}, {8, 8, 1},
                          {8, 32, 1}, {3, 7, 1}, {2, 4, 2},  {4, 8, 2}, {2, 6, 3}};
  for (auto& s : sch) {
    StageTiming t{1.0, 2.0, 0.0};
    auto tl = simulate(s.v > 1 ? ScheduleKind::Interleaved1F1B : ScheduleKind::OneF1B, s.p, s.m,
                       s.v, t);
    std::printf("%s  {\"p\": %d, \"m\": %d, \"v\": %d, \"bubble_ratio\": %.17g, \"order\": [",
                first ? "" : ",\n", s.p, s.m, s.v, tl.bubble_ratio);
    first = false;
    for (int d = 0; d < s.p; ++d) {
      std::printf("%s[", d ? ", " : "");
      bool f2 = true;
      for (auto& ev : tl.events)
        if (ev.device == d && (ev.kind == EventKind::Fwd || ev.kind == EventKind::Bwd)) {
          std::printf("%s[%d,%d,%d]", f2 ? "" : ",", ev.kind == EventKind::Bwd ? 1 : 0,
                      ev.microbatch, ev.chunk);
          f2 = false;
        }
      std::printf("]");
    }
    std::printf("]}");
  }
  std::printf("\n]\n}\n");
  return 0;
}
