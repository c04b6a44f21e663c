// Structural half of the hot path: shape accounting, the config gate, rank layout and the
// pipeline order. Semantics follow the reference (citations per function); tests compare every
// result with the reference library compiled from its own sources (oracle/_ref).
#include <algorithm>
#include <stdexcept>
#include <string>

#include "trainplan/core.hpp"

namespace trainplan {

namespace {

using u128 = unsigned __int128;

u128 checked_mul(u128 a, u128 b) {
  if (a != 0 && b > ~u128{0} / a) throw std::overflow_error("model FLOPs overflow 128 bits");
  return a * b;
}

u128 checked_add(u128 a, u128 b) {
  if (b > ~u128{0} - a) throw std::overflow_error("model FLOPs overflow 128 bits");
  return a + b;
}

void require_positive_shape(const ModelSpec& s) {
  if (s.num_layers < 1 || s.hidden_size < 1 || s.num_heads < 1 || s.vocab_size < 1 ||
      s.seq_length < 1)
    throw std::invalid_argument("ModelSpec fields must be strictly positive");
}

}  // namespace

// arch.cpp:35-46
std::vector<std::string> ModelSpec::validate() const {
  std::vector<std::string> out;
  const std::pair<int, const char*> fields[] = {{num_layers, "num_layers"},
                                                {hidden_size, "hidden_size"},
                                                {num_heads, "num_heads"},
                                                {vocab_size, "vocab_size"},
                                                {seq_length, "seq_length"}};
  for (const auto& [v, name] : fields)
    if (v < 1) out.push_back(std::string(name) + " must be >= 1");
  if (num_heads >= 1 && hidden_size >= 1 && hidden_size % num_heads != 0)
    out.push_back("hidden_size must be divisible by num_heads");
  return out;
}

// arch.cpp:48-62
ParamBreakdown param_count(const ModelSpec& spec) {
  require_positive_shape(spec);
  const std::uint64_t L = spec.num_layers, d = spec.hidden_size, V = spec.vocab_size,
                      s = spec.seq_length;
  ParamBreakdown b;
  b.attention_params = 3 * L * d * d;
  b.ffn_params = 8 * L * d * d;
  b.embedding_params = (V + s) * d;
  b.total_exact = b.attention_params + b.ffn_params + b.embedding_params;
  b.total_approx = 12 * L * d * d;
  return b;
}

std::uint64_t executed_param_count(const ModelSpec& spec) {
  require_positive_shape(spec);
  const std::uint64_t L = spec.num_layers, d = spec.hidden_size, V = spec.vocab_size,
                      s = spec.seq_length;
  return L * (12 * d * d + 13 * d) + (V + s) * d + 2 * d;
}

// arch.cpp:64-92: c/2 * B*s*d*(48*L*d + 8*L*s + 3*V), the bracket exact in u128.
double model_flops_per_iteration(const ModelSpec& spec, std::int64_t batch_size,
                                 bool checkpoint_activations, int checkpoint_factor) {
  require_positive_shape(spec);
  if (batch_size < 0) throw std::invalid_argument("batch_size must be non-negative");
  if (checkpoint_factor != 3 && checkpoint_factor != 4)
    throw std::invalid_argument("checkpoint_factor must be 3 or 4");
  if (batch_size == 0) return 0.0;
  const u128 L = static_cast<u128>(spec.num_layers), d = static_cast<u128>(spec.hidden_size),
             V = static_cast<u128>(spec.vocab_size), s = static_cast<u128>(spec.seq_length),
             B = static_cast<u128>(static_cast<std::uint64_t>(batch_size));
  const u128 bracket = checked_add(checked_add(checked_mul(checked_mul(48, L), d),
                                               checked_mul(checked_mul(8, L), s)),
                                   checked_mul(3, V));
  const u128 tokens_width = checked_mul(checked_mul(B, s), d);
  const u128 base = checked_mul(tokens_width, bracket);
  const double c = checkpoint_activations ? static_cast<double>(checkpoint_factor) : 3.0;
  return c * (static_cast<double>(base) * 0.5);
}

// memory.cpp:20-28
int ParallelConfig::num_microbatches() const {
  if (dp < 1) throw std::invalid_argument("dp not bound; run validate first");
  if (mbs < 1) throw std::invalid_argument("mbs must be >= 1");
  return gbs / (mbs * dp);
}

ClusterSpec b200_preset(int num_nodes, int gpus_per_node) {
  ClusterSpec c;
  c.num_nodes = num_nodes;
  c.gpus_per_node = gpus_per_node;
  c.mem_per_gpu = 180ull * 1000 * 1000 * 1000;
  c.peak_flops_per_gpu = 2.25e15;
  c.bw_same_card = 900e9;
  c.bw_intra_node = 900e9;
  c.bw_inter_node = 50e9;
  c.link_latency_intra = 2e-6;
  c.link_latency_inter = 5e-6;
  c.hbm_bandwidth = 8e12;
  return c;
}

std::vector<Violation> ValidationResult::hard_violations() const {
  std::vector<Violation> out;
  std::copy_if(violations.begin(), violations.end(), std::back_inserter(out),
               [](const Violation& v) { return v.hard; });
  return out;
}

// search.cpp:23-84
ValidationResult validate(const ModelSpec& model, const ParallelConfig& cfg,
                          const ClusterSpec& cluster) {
  ValidationResult r;
  r.resolved = cfg;
  auto hard = [&](const char* f, std::string msg) { r.violations.push_back({f, std::move(msg), true}); };

  if (cfg.tp < 1) hard("tp", "tp must be >= 1");
  if (cfg.pp < 1) hard("pp", "pp must be >= 1");
  if (cfg.mbs < 1) hard("mbs", "mbs must be >= 1");
  if (cfg.gbs < 1) hard("gbs", "gbs must be >= 1");
  if (cfg.interleave_v < 1) hard("interleave_v", "interleave_v must be >= 1");
  if (cfg.zero_stage < 0 || cfg.zero_stage > 3) hard("zero_stage", "zero_stage must be 0..3");
  if (!r.violations.empty()) return r;  // ok stays false

  const long long world = cluster.world_size();
  const long long shards = static_cast<long long>(cfg.tp) * cfg.pp;
  if (cfg.dp == 0) {
    if (world % shards == 0)
      r.resolved.dp = static_cast<int>(world / shards);
    else
      hard("dp", "world size " + std::to_string(world) + " not divisible by tp*pp");
  } else if (shards * cfg.dp != world) {
    hard("dp", "tp*pp*dp != num_nodes*gpus_per_node (" + std::to_string(world) + " GPUs)");
  }
  if (model.num_layers % cfg.pp != 0)
    hard("pp", "num_layers " + std::to_string(model.num_layers) + " not divisible by pp " +
                   std::to_string(cfg.pp));
  if (model.hidden_size % cfg.tp != 0) hard("tp", "hidden_size not divisible by tp");
  if (model.num_heads % cfg.tp != 0) hard("tp", "num_heads not divisible by tp");
  if (cfg.zero_stage == 3 && cfg.pp > 1)
    hard("zero_stage", "ZeRO-3 cannot be combined with pipeline parallelism");
  if (cfg.tp > cluster.gpus_per_node)
    r.violations.push_back({"tp", "tp " + std::to_string(cfg.tp) +
                                      " spans nodes; keep TP within one node", false});
  if (r.resolved.dp >= 1) {
    const long long per_step = static_cast<long long>(cfg.mbs) * r.resolved.dp;
    if (cfg.gbs % per_step != 0) {
      hard("gbs", "gbs not divisible by mbs*dp (" + std::to_string(per_step) + ")");
    } else {
      r.num_microbatches = static_cast<int>(cfg.gbs / per_step);
      if (r.num_microbatches < 1) hard("gbs", "configuration yields no microbatches");
    }
  }
  r.ok = r.hard_violations().empty();
  return r;
}

void validate_kernels(const ModelSpec& model, const ParallelConfig& cfg, ValidationResult& res) {
  auto hard = [&](const char* f, std::string msg) {
    res.violations.push_back({f, std::move(msg), true});
    res.ok = false;
  };
  const int tp = std::max(cfg.tp, 1);
  if (model.num_heads < 1 || model.hidden_size % std::max(model.num_heads, 1) != 0) {
    hard("num_heads", "hidden_size must be divisible by num_heads");
    return;
  }
  const int hd = model.hidden_size / model.num_heads;
  if (hd != 64 && hd != 128 && hd != 160)
    hard("num_heads", "head dim " + std::to_string(hd) + " unsupported (64, 128, 160)");
  if (model.vocab_size % (128 * tp) != 0)
    hard("vocab_size", "vocab_size must be a multiple of 128*tp for the vocab-parallel head");
  if ((model.hidden_size / tp) % 64 != 0 || model.hidden_size % 128 != 0)
    hard("hidden_size", "hidden_size/tp must be a multiple of 64 (GEMM tile)");
  if (model.seq_length % 128 != 0)
    hard("seq_length", "seq_length must be a multiple of 128 (attention/GEMM tile)");
  if (cfg.precision != Precision::BF16)
    hard("precision", "the B200 step computes in bf16 (fp32 master weights and grads)");
  if (cfg.zero_stage > 1) hard("zero_stage", "ZeRO stages 2/3 are out of scope (north_star: ZeRO-1)");
  if (cfg.interleave_v > 1 && cfg.pp < 2) hard("interleave_v", "interleave_v > 1 needs pipeline parallelism (pp >= 2)");
  if (cfg.interleave_v > 1 && cfg.pp >= 1 && model.num_layers % (cfg.pp * cfg.interleave_v) != 0)
    hard("interleave_v", "num_layers must be divisible by pp*interleave_v (equal model chunks)");
}

RankCoords rank_coords(int rank, const ParallelConfig& c) {
  RankCoords r;
  r.t = rank % c.tp;
  r.p = (rank / c.tp) % c.pp;
  r.d = rank / (c.tp * c.pp);
  return r;
}

int rank_of(const RankCoords& r, const ParallelConfig& c) { return r.t + c.tp * (r.p + c.pp * r.d); }

// pipesim.cpp:31-91
std::vector<PipeOp> pipeline_order(ScheduleKind kind, int p, int m, int v, int device) {
  if (p < 1 || m < 1 || v < 1 || device < 0 || device >= p)
    throw std::invalid_argument("pipeline_order: bad (p, m, v, device)");
  if (v > 1 && kind != ScheduleKind::Interleaved1F1B)
    throw std::invalid_argument("v > 1 requires the interleaved schedule");
  std::vector<PipeOp> ops;
  ops.reserve(2 * static_cast<size_t>(m) * v);
  if (kind == ScheduleKind::GPipe) {
    for (int i = 0; i < m; ++i) ops.push_back({false, i, 0});
    for (int i = 0; i < m; ++i) ops.push_back({true, i, 0});
    return ops;
  }
  if (kind == ScheduleKind::OneF1B || v == 1) {
    const int warm = std::min(p - 1 - device, m);
    int f = 0, b = 0;
    while (f < warm) ops.push_back({false, f++, 0});
    while (f < m) {
      ops.push_back({false, f++, 0});
      ops.push_back({true, b++, 0});
    }
    while (b < m) ops.push_back({true, b++, 0});
    return ops;
  }
  // Interleaved: microbatches advance in rounds of up to p over the v chunks; backwards visit
  // chunks in reverse order.
  std::vector<PipeOp> fwd, bwd;
  for (int r0 = 0; r0 < m; r0 += p) {
    const int n = std::min(p, m - r0);
    for (int c = 0; c < v; ++c)
      for (int i = 0; i < n; ++i) fwd.push_back({false, r0 + i, c});
    for (int c = v - 1; c >= 0; --c)
      for (int i = 0; i < n; ++i) bwd.push_back({true, r0 + i, c});
  }
  const int total = m * v;
  const int warm = (m % p != 0 || m == p) ? total
                                          : std::min((p - 1 - device) * 2 + (v - 1) * p, total);
  for (int i = 0; i < warm; ++i) ops.push_back(fwd[i]);
  for (int i = 0; i < total - warm; ++i) {
    ops.push_back(fwd[warm + i]);
    ops.push_back(bwd[i]);
  }
  for (int i = total - warm; i < total; ++i) ops.push_back(bwd[i]);
  return ops;
}

}  // namespace trainplan
