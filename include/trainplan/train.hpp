// The executed GPT train step behind the reference's API.
//
// `estimate()` (/root/reference/proj/include/trainplan/perf.hpp:42-44) PREDICTS a train step;
// `measure()` below RUNS it on B200s and returns the same ThroughputEstimate, so callers of the
// reference switch by changing one call. `make_measured_evaluator()` is the plug-in for the
// reference's search loop (Evaluator, search.hpp:77), the seam where the paper launched real
// training jobs. All of it sits on the C-ABI in trainplan/capi.h.
#pragma once

#include <array>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "trainplan/b200.hpp"
#include "trainplan/capi.h"
#include "trainplan/memory.hpp"
#include "trainplan/perf.hpp"
#include "trainplan/search.hpp"

namespace trainplan {

struct TrainOptions {
  std::uint64_t seed = 1234;  // counter-based init + dropout key
  float dropout = 0.1f;       // hidden dropout (embedding, attention-out, MLP-out)
  float lr = 1e-4f, beta1 = 0.9f, beta2 = 0.95f, eps = 1e-8f, weight_decay = 0.0f;
};

// This process's place in the job (one process per GPU). world > 1 needs the NCCL id that
// rank 0 obtained from nccl_unique_id().
struct DistributedContext {
  int rank = 0, world = 1, device = 0;
  std::optional<std::array<unsigned char, 128>> nccl_id;
};

std::array<unsigned char, 128> nccl_unique_id();

// A host wait of the session exceeded its watchdog timeout (TP_ERR_TIMEOUT): the NCCL
// communicators were aborted and the session is unusable; the process should exit. Maps to
// FailureKind::Timeout (search.hpp:59) in the measured evaluator.
class StepTimeout : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

// RAII owner of one rank's train-step session. Throws std::invalid_argument for an invalid
// configuration, std::bad_alloc when the configuration does not fit in HBM, StepTimeout when the
// watchdog fires and std::runtime_error for other CUDA/NCCL failures.
class TrainSession {
 public:
  TrainSession(const ModelSpec& model, const ParallelConfig& cfg, const TrainOptions& opts = {},
               const DistributedContext& dist = {});
  ~TrainSession();
  TrainSession(TrainSession&& o) noexcept;
  TrainSession& operator=(TrainSession&&) = delete;
  TrainSession(const TrainSession&) = delete;

  void init_params();
  // tokens: global batch [gbs][s+1] int32 (inputs = [:, :s], labels = [:, 1:]).
  float train_step(const std::vector<std::int32_t>& tokens);  // H2D + step + D2H loss
  void upload(const std::int32_t* tokens, std::size_t n);
  void step();        // on the uploaded tokens, asynchronous
  float loss();       // mean CE of the last step (blocking)
  // Device time (ms) of `steps` iterations; per-kernel-class timing when kt != nullptr.
  float time_steps(int steps, tp_kernel_times* kt = nullptr);
  float allreduce_max(float v);
  // Watchdog for host waits (seconds <= 0: none); see tp_session_set_timeout.
  void set_timeout(double seconds);
  // MEASURED per-GPU footprint in the categories of the reference's MemoryReport (memory.hpp):
  // params = bf16 working copy + fp32 master (ZeRO shard), gradients = fp32 main grads, optimizer
  // = Adam m + v (ZeRO shard), activations = stored / recomputed per-microbatch tensors,
  // overhead = per-op workspace + the unused part of the NVLS window; fits vs mem_per_gpu.
  MemoryReport memory_report(std::uint64_t mem_per_gpu = 0);
  tp_session* handle() { return s_; }

 private:
  tp_session* s_ = nullptr;
};

struct MeasureOptions {
  int warmup = 3;
  int steps = 5;
  double timeout_s = 0.0;  // watchdog for every host wait (0: none)
  TrainOptions train;
  DistributedContext dist;
};

// Measured counterpart of estimate(): validates like estimate() (std::invalid_argument on an
// invalid configuration; OOM anywhere — allocation, init, steps — is a reported state, est.oom =
// true; StepTimeout when the watchdog fires), runs warmup + timed steps on
// synthetic tokens (std::mt19937_64(seed), uniform over the vocabulary) and fills
//   iter_time      device seconds per iteration (max over ranks)
//   flops_per_gpu  model_flops_per_iteration(model, gbs, ckpt) / (iter_time * world)
//   peak_fraction  flops_per_gpu / cluster.peak_flops_per_gpu
//   breakdown      compute / tp_comm / pp_comm from CUDA events around every launch on the step
//                  stream; dp_comm = the EXPOSED data-parallel tail (the step waiting for the
//                  comm-stream reduce-scatter / Adam / allgather pipeline after the last
//                  backward op; the DP collectives themselves overlap the backward, so the
//                  reference's serial dp_time, perf.cpp:88-102, is an upper bound of this);
//                  bubble = iter_time - the rest (pipeline idle + launch gaps)
// Multi-GPU: every rank calls measure() with its DistributedContext.
ThroughputEstimate measure(const ModelSpec& model, const ParallelConfig& cfg, const ClusterSpec& cluster,
                           const MeasureOptions& opts = {});

// Allocates the session for (model, cfg) on this process's GPU without running a step and
// returns its measured footprint (TrainSession::memory_report); fits = false and all-zero bytes
// when it does not fit (the allocation failed). Compare with memory_per_gpu (the model).
MemoryReport measured_memory_per_gpu(const ModelSpec& model, const ParallelConfig& cfg, const ClusterSpec& cluster,
                                     const DistributedContext& dist = {});

// The configuration a search point denotes (reference semantics, perf.cpp:161-181: gbs = mbs *
// gas * dp, activation checkpointing and flash attention on) computed in bf16.
std::optional<ParallelConfig> measured_config_from_point(const SearchPoint& point, const ClusterSpec& cluster);

// Evaluator that runs the point on this process's GPU(s) instead of modelling it: Invalid for
// configurations that do not factor or validate (including the kernels' constraints) or fail to
// run, Oom when they do not fit, Timeout when the watchdog (opts.timeout_s) fires; objective =
// measured model TFLOPS/GPU; wall_time = host seconds spent on the point. zero1 = false runs
// replicated data parallelism (ZeRO-0: gradient allreduce, full optimizer state per rank).
// Not thread-safe: use run_search(..., workers = 1).
Evaluator make_measured_evaluator(const ModelSpec& model, const ClusterSpec& cluster,
                                  const MeasureOptions& opts = {});

// One Megatron-style iteration log line ("iteration N/ M | ... elapsed time per iteration (ms):
// T | ... TFLOPs: F |"), parseable by the reference's parse_training_log (metrics.cpp:119-147).
std::string megatron_log_line(long iteration, long total, const ThroughputEstimate& est, double lr, float loss,
                              long global_batch);

}  // namespace trainplan
