#include <algorithm>
// C-ABI wrappers of the structural plan layer (include/trainplan/capi.h "plan" section).
#include <cstring>
#include <exception>
#include <stdexcept>

#include "runtime/pipe_exec.h"
#include "runtime/status.h"
#include "trainplan/capi.h"
#include "trainplan/core.hpp"
#include "trainplan/b200_metrics.hpp"
#include <sstream>

using namespace trainplan;

namespace gptb200 {

ModelSpec to_spec(const tp_model_spec& m) {
  ModelSpec s;
  s.num_layers = m.num_layers;
  s.hidden_size = m.hidden_size;
  s.num_heads = m.num_heads;
  s.vocab_size = m.vocab_size;
  s.seq_length = m.seq_length;
  return s;
}

ParallelConfig to_cfg(const tp_parallel_config& c) {
  ParallelConfig p;
  p.tp = c.tp;
  p.pp = c.pp;
  p.dp = c.dp;
  p.mbs = c.mbs;
  p.gbs = c.gbs;
  p.zero_stage = c.zero_stage;
  p.interleave_v = c.interleave_v;
  p.precision = c.precision == 1 ? Precision::BF16 : (c.precision == 2 ? Precision::FP32 : Precision::FP16);
  p.grad_accum_dtype = c.grad_accum_fp32 ? GradAccumDtype::FP32 : GradAccumDtype::FP16;
  p.checkpoint_activations = c.checkpoint_activations != 0;
  p.flash_attention = c.flash_attention != 0;
  return p;
}

template <class F>
int guarded(const char* where, F&& f) {
  try {
    f();
    return clear_error();
  } catch (const std::invalid_argument& e) {
    return set_error(TP_ERR_INVALID, std::string(where) + ": " + e.what());
  } catch (const std::exception& e) {
    return set_error(TP_ERR_INTERNAL, std::string(where) + ": " + e.what());
  }
}

}  // namespace gptb200

using namespace gptb200;

extern "C" {

int tp_param_count(const tp_model_spec* m, uint64_t out[6]) {
  return guarded("tp_param_count", [&] {
    auto s = to_spec(*m);
    auto b = param_count(s);
    out[0] = b.attention_params;
    out[1] = b.ffn_params;
    out[2] = b.embedding_params;
    out[3] = b.total_exact;
    out[4] = b.total_approx;
    out[5] = executed_param_count(s);
  });
}

int tp_model_flops(const tp_model_spec* m, int64_t batch, int ckpt, int factor, double* out) {
  return guarded("tp_model_flops",
                 [&] { *out = model_flops_per_iteration(to_spec(*m), batch, ckpt != 0, factor); });
}

int tp_validate(const tp_model_spec* m, const tp_parallel_config* c, int num_nodes,
                int gpus_per_node, int kernel_checks, tp_validation* out) {
  return guarded("tp_validate", [&] {
    ClusterSpec cl = b200_preset(num_nodes, gpus_per_node);
    auto r = validate(to_spec(*m), to_cfg(*c), cl);
    if (kernel_checks) validate_kernels(to_spec(*m), r.resolved, r);
    std::memset(out, 0, sizeof(*out));
    out->ok = r.ok ? 1 : 0;
    out->dp = r.resolved.dp;
    out->num_microbatches = r.num_microbatches;
    out->num_violations = static_cast<int>(r.violations.size());
    for (size_t i = 0; i < r.violations.size() && i < 16; ++i) {
      std::strncpy(out->fields[i], r.violations[i].field.c_str(), 23);
      out->hard[i] = r.violations[i].hard ? 1 : 0;
    }
    if (!r.violations.empty()) std::strncpy(out->first_message, r.violations[0].message.c_str(), 255);
  });
}

int tp_pipeline_order(int kind, int p, int m, int v, int device, int* ops, int cap, int* n) {
  return guarded("tp_pipeline_order", [&] {
    auto k = kind == 0 ? ScheduleKind::GPipe : (kind == 1 ? ScheduleKind::OneF1B : ScheduleKind::Interleaved1F1B);
    auto order = pipeline_order(k, p, m, v, device);
    *n = static_cast<int>(order.size());
    for (int i = 0; i < *n && i < cap; ++i) {
      ops[3 * i] = order[i].backward ? 1 : 0;
      ops[3 * i + 1] = order[i].microbatch;
      ops[3 * i + 2] = order[i].chunk;
    }
  });
}

int tp_pipeline_actions(int p, int m, int v, int device, int dh_ring, int forward_only, int* out, int cap, int* n) {
  return guarded("tp_pipeline_actions", [&] {
    auto acts = gptb200::pipeline_actions(p, m, v, device, dh_ring, forward_only != 0);
    *n = static_cast<int>(acts.size());
    for (int i = 0; i < *n && i < cap; ++i) {
      const auto& a = acts[i];
      int* o = out + 6 * i;
      o[0] = a.kind, o[1] = a.microbatch, o[2] = a.chunk, o[3] = a.slot, o[4] = a.dh, o[5] = a.flags;
    }
  });
}

int tp_rank_coords(int rank, int tp, int pp, int dp, int out[3]) {
  return guarded("tp_rank_coords", [&] {
    if (tp < 1 || pp < 1 || dp < 1 || rank < 0 || rank >= tp * pp * dp)
      throw std::invalid_argument("rank out of range");
    ParallelConfig c;
    c.tp = tp;
    c.pp = pp;
    c.dp = dp;
    auto r = rank_coords(rank, c);
    out[0] = r.t;
    out[1] = r.p;
    out[2] = r.d;
  });
}

int tp_ncu_parse_csv(const char* text, size_t len, const char* kernel_filter, tp_hw_counters* out) {
  return guarded("tp_ncu_parse_csv", [&] {
    if (!text || !out) throw std::invalid_argument("null argument");
    std::istringstream in(std::string(text, len));
    NcuParseResult r = parse_ncu_csv(in);
    NcuCounterRecord t;
    if (!kernel_filter || !*kernel_filter) {
      t = r.totals;
    } else {
      for (const auto& [name, rec] : r.per_kernel)
        if (name.find(kernel_filter) != std::string::npos) t += rec;
    }
    out->launches = t.launches;
    out->tensor_utc_bf16 = t.tensor_utc_bf16;
    out->tensor_utc_f16 = t.tensor_utc_f16;
    out->tensor_hmma_bf16 = t.tensor_hmma_bf16;
    out->tensor_hmma_f16 = t.tensor_hmma_f16;
    out->dram_read_bytes = t.dram_read_bytes;
    out->dram_write_bytes = t.dram_write_bytes;
    out->duration_ns = t.duration_ns;
    out->tensor_flops = hw_tensor_flops(t);
    out->simt_flops = hw_simt_flops(t);
    out->hw_flops = hw_flops(t);
    out->num_warnings = static_cast<int>(r.warnings.size());
  });
}

int tp_ncu_metric_list(char* buf, size_t cap) {
  return guarded("tp_ncu_metric_list", [&] {
    const std::string s = ncu_metric_list();
    if (!buf || cap < s.size() + 1) throw std::invalid_argument("buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

int tp_diagnose_mbs_mismatch(double model_tflops, double hw_tflops, int cfg_mbs, int ds_mbs, int* kind,
                             double* ratio, char* msg, size_t cap) {
  return guarded("tp_diagnose_mbs_mismatch", [&] {
    MbsDiagnosis d = diagnose_mbs_mismatch(model_tflops, hw_tflops, cfg_mbs, ds_mbs);
    if (kind) *kind = static_cast<int>(d.kind);
    if (ratio) *ratio = d.flops_ratio;
    if (msg && cap) {
      const size_t n = std::min(cap - 1, d.message.size());
      std::memcpy(msg, d.message.data(), n);
      msg[n] = 0;
    }
  });
}

}  // extern "C"
