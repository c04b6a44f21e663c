// C-ABI of the train-step session (include/trainplan/capi.h "train-step session").
#include <nccl.h>

#include <cstring>
#include <exception>
#include <memory>

#include "kernels/tma_host.h"
#include "runtime/stage.h"
#include "runtime/status.h"
#include "trainplan/capi.h"
#include "trainplan/core.hpp"

namespace gptb200 {
trainplan::ModelSpec to_spec(const tp_model_spec& m);
trainplan::ParallelConfig to_cfg(const tp_parallel_config& c);
}  // namespace gptb200

using namespace gptb200;

struct tp_session {
  std::unique_ptr<Stage> stage;
  int rank = 0, world = 1;
};

namespace {

template <class F>
int run(const char* where, F&& f) {
  try {
    f();
    return clear_error();
  } catch (const StepError& e) {
    return set_error(e.code, std::string(where) + ": " + e.msg);
  } catch (const CommError& e) {
    return set_error(e.code, std::string(where) + ": " + e.msg);
  } catch (const std::invalid_argument& e) {
    return set_error(TP_ERR_INVALID, std::string(where) + ": " + e.what());
  } catch (const std::exception& e) {
    return set_error(TP_ERR_INTERNAL, std::string(where) + ": " + e.what());
  }
}

}  // namespace

extern "C" {

int tp_nccl_unique_id(unsigned char out[128]) {
  return run("tp_nccl_unique_id", [&] {
    ncclUniqueId id;
    nccl_check(ncclGetUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(id) == 128, "ncclUniqueId size");
    std::memcpy(out, &id, 128);
  });
}

int tp_session_create(const tp_model_spec* model, const tp_parallel_config* cfg, const tp_train_options* opts,
                      int rank, int world, int device, const unsigned char* nccl_id, tp_session** out) {
  return run("tp_session_create", [&] {
    *out = nullptr;
    const auto spec = to_spec(*model);
    auto pc = to_cfg(*cfg);
    trainplan::ClusterSpec cl = trainplan::b200_preset(1, world);
    auto v = trainplan::validate(spec, pc, cl);
    trainplan::validate_kernels(spec, v.resolved, v);
    if (!v.ok) {
      auto hv = v.hard_violations();
      throw StepError{TP_ERR_INVALID, "invalid configuration: " + hv.front().field + ": " + hv.front().message};
    }
    if (world > 1 && nccl_id == nullptr) throw StepError{TP_ERR_INVALID, "nccl_id required when world > 1"};
    TrainOptions o;
    if (opts) {
      o.seed = opts->seed;
      o.dropout = opts->dropout;
      o.lr = opts->lr;
      o.beta1 = opts->beta1;
      o.beta2 = opts->beta2;
      o.eps = opts->eps;
      o.weight_decay = opts->weight_decay;
    }
    auto s = std::make_unique<tp_session>();
    s->rank = rank;
    s->world = world;
    s->stage = std::make_unique<Stage>(spec, v.resolved, o, rank, world, device, nccl_id);
    *out = s.release();
  });
}

int tp_session_destroy(tp_session* s) {
  return run("tp_session_destroy", [&] { delete s; });
}

int tp_session_init_params(tp_session* s) {
  return run("tp_session_init_params", [&] { s->stage->init_params(); });
}

int tp_session_upload_tokens(tp_session* s, const int32_t* tokens, int64_t n, int on_device) {
  return run("tp_session_upload_tokens", [&] { s->stage->upload_tokens(tokens, n, on_device != 0); });
}

int tp_session_step(tp_session* s) {
  return run("tp_session_step", [&] { s->stage->step(); });
}

int tp_session_train_step(tp_session* s, const int32_t* host_tokens, int64_t n, float* loss_out) {
  return run("tp_session_train_step", [&] {
    s->stage->upload_tokens(host_tokens, n, false);
    s->stage->step();
    float l = s->stage->read_loss();
    if (loss_out) *loss_out = l;
  });
}

int tp_session_read_loss(tp_session* s, float* loss_out) {
  return run("tp_session_read_loss", [&] { *loss_out = s->stage->read_loss(); });
}

int tp_session_eval_loss(tp_session* s, float* loss_out) {
  return run("tp_session_eval_loss", [&] { *loss_out = s->stage->eval_loss(); });
}

int tp_session_sync(tp_session* s) {
  return run("tp_session_sync", [&] { s->stage->sync(); });
}

int tp_session_barrier(tp_session* s) {
  return run("tp_session_barrier", [&] { s->stage->barrier(); });
}

int tp_session_tensor_info(tp_session* s, int tensor_id, int64_t info[9]) {
  return run("tp_session_tensor_info", [&] {
    std::memset(info, 0, 9 * sizeof(int64_t));
    const ParamSlot* p = s->stage->slot(tensor_id);
    if (!p) return;
    info[0] = 1;
    info[1] = p->rows;
    info[2] = p->cols;
    info[3] = p->offset;
    info[4] = p->rseg;
    info[5] = p->rstride;
    info[6] = p->roff;
    info[7] = p->coff;
    info[8] = p->gcols;
  });
}

int tp_session_read_tensor(tp_session* s, int which, int tensor_id, float* host_out) {
  return run("tp_session_read_tensor", [&] { s->stage->read_tensor(which, tensor_id, host_out); });
}

int tp_session_read_flat(tp_session* s, int which, int64_t offset, int64_t n, float* host_out) {
  return run("tp_session_read_flat", [&] { s->stage->read_flat(which, offset, n, host_out); });
}

int tp_session_buckets(tp_session* s, int64_t* out, int cap, int* n) {
  return run("tp_session_buckets", [&] {
    const auto& b = s->stage->buckets();
    *n = static_cast<int>(b.size());
    for (int i = 0; i < *n && i < cap; ++i) {
      out[3 * i] = b[i].off;
      out[3 * i + 1] = b[i].len;
      out[3 * i + 2] = b[i].master_off;
    }
  });
}

int tp_session_info(tp_session* s, int64_t out[8]) {
  return run("tp_session_info", [&] {
    out[0] = s->stage->flat_params();
    out[1] = s->stage->shard_params();
    out[2] = static_cast<int64_t>(s->stage->device_bytes());
    out[3] = s->stage->microbatches();
    out[4] = s->stage->kernel_launches_per_step();
    out[5] = s->rank;
    out[6] = s->world;
    out[7] = s->stage->tp_mode();
  });
}

int tp_session_step_times(tp_session* s, float* out, int n) {
  return run("tp_session_step_times", [&] {
    const std::vector<float>& t = s->stage->step_times();
    for (int i = 0; i < n && i < static_cast<int>(t.size()); ++i) out[i] = t[i];
  });
}

int tp_session_time_steps(tp_session* s, int steps, int profile, float* ms, tp_kernel_times* kt) {
  return run("tp_session_time_steps", [&] {
    KernelTimes k;
    *ms = s->stage->time_steps(steps, profile != 0, &k);
    if (kt) {
      static_assert(K_NUM == TP_KERNEL_CLASSES, "kernel class count");
      for (int i = 0; i < K_NUM; ++i) {
        kt->ms[i] = k.ms[i];
        kt->launches[i] = k.launches[i];
        kt->flops[i] = k.flops[i];
        kt->bytes[i] = k.bytes[i];
      }
    }
  });
}

int tp_session_set_timeout(tp_session* s, double seconds) {
  return run("tp_session_set_timeout", [&] { s->stage->set_timeout(seconds); });
}

int tp_session_memory(tp_session* s, tp_memory_report* out) {
  return run("tp_session_memory", [&] {
    const Stage& st = *s->stage;
    out->params_bytes = st.category_bytes(MEM_PARAMS);
    out->gradient_bytes = st.category_bytes(MEM_GRADS);
    out->optimizer_bytes = st.category_bytes(MEM_OPTIMIZER);
    out->activation_bytes = st.category_bytes(MEM_ACTIVATIONS);
    out->workspace_bytes = st.category_bytes(MEM_WORKSPACE);
    out->window_bytes = st.window_bytes();
    out->total_bytes = st.device_bytes() + st.window_bytes();
    out->zero_stage = st.zero_stage();
  });
}

int tp_variant_counts(int64_t out[TP_KERNEL_VARIANTS]) {
  static_assert(KV_NUM == TP_KERNEL_VARIANTS, "variant count");
  return run("tp_variant_counts", [&] { read_variants(out, TP_KERNEL_VARIANTS); });
}

int tp_variant_counts_reset(void) {
  return run("tp_variant_counts_reset", [&] { reset_variants(); });
}

int tp_session_allreduce_max(tp_session* s, float* v) {
  return run("tp_session_allreduce_max", [&] { *v = s->stage->allreduce_max(*v); });
}

int tp_session_debug_tp_allreduce(tp_session* s, const uint16_t* in, uint16_t* out, int mode) {
  return run("tp_session_debug_tp_allreduce", [&] { s->stage->debug_tp_allreduce(in, out, mode); });
}

int tp_session_bench_sp(tp_session* s, int iters, int mode, float* ms) {
  return run("tp_session_bench_sp", [&] { *ms = s->stage->bench_sp(iters, mode); });
}

int tp_session_bench_tp_allreduce(tp_session* s, int iters, int mode, int ctas, float* ms, int* nvls) {
  return run("tp_session_bench_tp_allreduce", [&] {
    *ms = s->stage->bench_tp_allreduce(iters, mode, ctas);
    *nvls = s->stage->tp_uses_nvls() ? 1 : 0;
  });
}

}  // extern "C"
