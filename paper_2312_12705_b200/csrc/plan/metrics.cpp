// B200 hardware-counter accounting (include/trainplan/metrics.hpp). Host-only C++.
//
// Reference roles: CounterRecord / hw_flops / parse_counter_csv (proj/src/metrics.cpp:67-117,
// AMD SQ_INSTS_VALU_*), diagnose_mbs_mismatch / roofline / weak_scaling / strong_scaling
// (proj/src/metrics.cpp:164-240).
#include "trainplan/b200_metrics.hpp"

#include <array>
#include <charconv>
#include <cmath>
#include <istream>
#include <set>
#include <sstream>
#include <stdexcept>

namespace trainplan {

namespace {

using Field = std::uint64_t NcuCounterRecord::*;

struct MetricField {
  const char* name;  // without the .sum rollup suffix
  Field field;
};

constexpr std::array<MetricField, 19> kMetrics = {{
    {"sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32", &NcuCounterRecord::tensor_utc_bf16},
    {"sm__ops_path_tensor_op_utchmma_src_fp16_dst_fp32", &NcuCounterRecord::tensor_utc_f16},
    {"sm__ops_path_tensor_op_hmma_src_bf16_dst_fp32", &NcuCounterRecord::tensor_hmma_bf16},
    {"sm__ops_path_tensor_op_hmma_src_fp16_dst_fp32", &NcuCounterRecord::tensor_hmma_f16},
    {"smsp__sass_thread_inst_executed_op_fadd_pred_on", &NcuCounterRecord::fadd},
    {"smsp__sass_thread_inst_executed_op_fmul_pred_on", &NcuCounterRecord::fmul},
    {"smsp__sass_thread_inst_executed_op_ffma_pred_on", &NcuCounterRecord::ffma},
    {"smsp__sass_thread_inst_executed_op_fadd2_pred_on", &NcuCounterRecord::fadd2},
    {"smsp__sass_thread_inst_executed_op_fmul2_pred_on", &NcuCounterRecord::fmul2},
    {"smsp__sass_thread_inst_executed_op_ffma2_pred_on", &NcuCounterRecord::ffma2},
    {"smsp__sass_thread_inst_executed_op_hadd_pred_on", &NcuCounterRecord::hadd},
    {"smsp__sass_thread_inst_executed_op_hmul_pred_on", &NcuCounterRecord::hmul},
    {"smsp__sass_thread_inst_executed_op_hfma_pred_on", &NcuCounterRecord::hfma},
    {"smsp__sass_thread_inst_executed_op_dadd_pred_on", &NcuCounterRecord::dadd},
    {"smsp__sass_thread_inst_executed_op_dmul_pred_on", &NcuCounterRecord::dmul},
    {"smsp__sass_thread_inst_executed_op_dfma_pred_on", &NcuCounterRecord::dfma},
    {"dram__bytes_read", &NcuCounterRecord::dram_read_bytes},
    {"dram__bytes_write", &NcuCounterRecord::dram_write_bytes},
    {"gpu__time_duration", &NcuCounterRecord::duration_ns},
}};

std::string trim(const std::string& s) {
  const auto b = s.find_first_not_of(" \t\r\n");
  if (b == std::string::npos) return {};
  return s.substr(b, s.find_last_not_of(" \t\r\n") - b + 1);
}

// RFC-4180-style split: quoted fields may contain commas and doubled quotes.
std::vector<std::string> split_csv(const std::string& line) {
  std::vector<std::string> out;
  std::string cur;
  bool quoted = false;
  for (std::size_t i = 0; i < line.size(); ++i) {
    const char c = line[i];
    if (quoted) {
      if (c == '"' && i + 1 < line.size() && line[i + 1] == '"') {
        cur.push_back('"');
        ++i;
      } else if (c == '"') {
        quoted = false;
      } else {
        cur.push_back(c);
      }
    } else if (c == '"') {
      quoted = true;
    } else if (c == ',') {
      out.push_back(cur);
      cur.clear();
    } else {
      cur.push_back(c);
    }
  }
  out.push_back(cur);
  for (auto& f : out) f = trim(f);
  return out;
}

Field field_for(std::string name) {
  // "smsp__x.sum" / "sm__x.sum" rollups; SIMT op counters are accepted at sm__ or smsp__ scope
  if (name.size() > 4 && name.compare(name.size() - 4, 4, ".sum") == 0) name.resize(name.size() - 4);
  if (name.rfind("sm__sass_thread_inst_executed_op_", 0) == 0) name.insert(2, "sp");
  for (const auto& m : kMetrics)
    if (name == m.name) return m.field;
  return nullptr;
}

bool is_metric_name(const std::string& name) { return name.find("__") != std::string::npos; }

// Scale of an ncu unit to the record's base unit (bytes, nanoseconds, counts).
double unit_scale(const std::string& unit_raw) {
  const std::string u = trim(unit_raw);
  if (u.empty() || u == "inst" || u == "warp" || u == "thread" || u == "cycle") return 1.0;
  auto prefixed = [&](const std::string& base, double unit) -> double {
    if (u == base) return unit;
    if (u.size() == base.size() + 1 && u.compare(1, base.size(), base) == 0) {
      switch (u[0]) {
        case 'K': case 'k': return unit * 1e3;
        case 'M': return unit * 1e6;
        case 'G': return unit * 1e9;
        case 'T': return unit * 1e12;
        case 'n': return unit * 1e-9;
        case 'u': return unit * 1e-6;
        case 'm': return unit * 1e-3;
        default: break;
      }
    }
    return 0.0;
  };
  if (double s = prefixed("byte", 1.0); s > 0) return s;
  if (double s = prefixed("second", 1e9); s > 0) return s;  // base: nanoseconds
  if (u == "ns") return 1.0;
  if (u == "us") return 1e3;
  if (u == "ms") return 1e6;
  if (u == "s") return 1e9;
  throw std::invalid_argument("unsupported ncu metric unit: " + u);
}

std::uint64_t parse_value(const std::string& raw, const std::string& unit) {
  std::string text;
  for (char c : trim(raw))
    if (c != ',') text.push_back(c);  // thousands separators
  if (text.empty()) return 0;
  const double scale = unit_scale(unit);
  if (scale == 1.0 && text.find_first_not_of("0123456789") == std::string::npos) return std::stoull(text);
  std::size_t used = 0;
  double v = 0.0;
  try {
    v = std::stod(text, &used);
  } catch (const std::exception&) {
    throw std::invalid_argument("unparsable counter value: " + raw);
  }
  if (used != text.size()) throw std::invalid_argument("unparsable counter value: " + raw);
  if (v < 0) throw std::invalid_argument("negative counter value: " + raw);
  return static_cast<std::uint64_t>(std::llround(v * scale));
}

int column(const std::vector<std::string>& header, const char* name) {
  for (std::size_t i = 0; i < header.size(); ++i)
    if (header[i] == name) return static_cast<int>(i);
  return -1;
}

bool is_ncu_banner(const std::string& line) { return line.rfind("==", 0) == 0; }

}  // namespace

NcuCounterRecord& NcuCounterRecord::operator+=(const NcuCounterRecord& other) {
  for (const auto& m : kMetrics) this->*m.field += other.*m.field;
  launches += other.launches;
  return *this;
}

double hw_tensor_flops(const NcuCounterRecord& r, double flops_per_utc_op, double flops_per_hmma_op) {
  return flops_per_utc_op * (static_cast<double>(r.tensor_utc_bf16) + static_cast<double>(r.tensor_utc_f16)) +
         flops_per_hmma_op * (static_cast<double>(r.tensor_hmma_bf16) + static_cast<double>(r.tensor_hmma_f16));
}

double hw_simt_flops(const NcuCounterRecord& r) {
  using u128 = unsigned __int128;
  const u128 f32 = u128{r.fadd} + r.fmul + u128{2} * r.ffma + u128{2} * (u128{r.fadd2} + r.fmul2) + u128{4} * r.ffma2;
  const u128 f16 = u128{2} * (u128{r.hadd} + r.hmul) + u128{4} * r.hfma;
  const u128 f64 = u128{r.dadd} + r.dmul + u128{2} * r.dfma;
  return static_cast<double>(f32 + f16 + f64);
}

double hw_flops(const NcuCounterRecord& r, double flops_per_utc_op, double flops_per_hmma_op) {
  return hw_tensor_flops(r, flops_per_utc_op, flops_per_hmma_op) + hw_simt_flops(r);
}

std::string ncu_metric_list() {
  std::string s;
  for (const auto& m : kMetrics) {
    if (!s.empty()) s += ',';
    s += m.name;
    s += ".sum";
  }
  return s;
}

NcuParseResult parse_ncu_csv(std::istream& in) {
  std::string line;
  std::vector<std::string> header;
  while (std::getline(in, line)) {  // skip ncu's "==PROF==" banner lines and blank lines
    if (trim(line).empty() || is_ncu_banner(line)) continue;
    header = split_csv(line);
    break;
  }
  if (header.empty()) throw std::invalid_argument("ncu CSV is empty");

  NcuParseResult res;
  std::set<std::string> unknown;
  auto warn = [&](const std::string& name) {
    if (unknown.insert(name).second) res.warnings.push_back("ignoring unknown metric: " + name);
  };
  const int c_id = column(header, "ID");
  const int c_kernel = column(header, "Kernel Name");
  const int c_metric = column(header, "Metric Name");
  const int c_unit = column(header, "Metric Unit");
  const int c_value = column(header, "Metric Value");

  if (c_metric >= 0) {
    // long form: rows of (launch ID, kernel, metric, unit, value)
    if (c_id < 0 || c_value < 0) throw std::invalid_argument("ncu CSV lacks the ID / Metric Value columns");
    std::map<std::string, std::pair<std::string, NcuCounterRecord>> launches;  // by ID
    std::vector<std::string> order;
    while (std::getline(in, line)) {
      if (trim(line).empty() || is_ncu_banner(line)) continue;
      const auto f = split_csv(line);
      if (f.size() != header.size())
        throw std::invalid_argument("ncu CSV row has " + std::to_string(f.size()) + " fields, expected " +
                                    std::to_string(header.size()));
      const std::string& name = f[c_metric];
      Field field = field_for(name);
      auto it = launches.find(f[c_id]);
      if (it == launches.end()) {
        it = launches.emplace(f[c_id], std::make_pair(c_kernel >= 0 ? f[c_kernel] : std::string(), NcuCounterRecord{}))
                 .first;
        it->second.second.launches = 1;
        order.push_back(f[c_id]);
      }
      if (!field) {
        warn(name);
        continue;
      }
      it->second.second.*field += parse_value(f[c_value], c_unit >= 0 ? f[c_unit] : std::string());
    }
    for (const auto& id : order) {
      const auto& [kernel, rec] = launches[id];
      res.totals += rec;
      res.per_kernel[kernel] += rec;
      ++res.rows;
    }
    return res;
  }

  // wide form: header of metric names, optional units row, one row per launch
  std::vector<Field> fields(header.size(), nullptr);
  for (std::size_t i = 0; i < header.size(); ++i) {
    if (!is_metric_name(header[i])) continue;
    fields[i] = field_for(header[i]);
    if (!fields[i]) warn(header[i]);
  }
  std::vector<std::string> units(header.size());
  bool first = true;
  while (std::getline(in, line)) {
    if (trim(line).empty() || is_ncu_banner(line)) continue;
    const auto f = split_csv(line);
    if (f.size() != header.size())
      throw std::invalid_argument("ncu CSV row has " + std::to_string(f.size()) + " fields, expected " +
                                  std::to_string(header.size()));
    if (first) {
      first = false;
      // the units row has an empty ID (and unit names where the values would be)
      if (c_id >= 0 && f[c_id].empty()) {
        units = f;
        continue;
      }
    }
    NcuCounterRecord rec;
    rec.launches = 1;
    for (std::size_t i = 0; i < f.size(); ++i)
      if (fields[i]) rec.*fields[i] += parse_value(f[i], units[i]);
    res.totals += rec;
    res.per_kernel[c_kernel >= 0 ? f[c_kernel] : std::string()] += rec;
    ++res.rows;
  }
  return res;
}

// ------------------------------------------------------- restated reference semantics

namespace {
// shortest round-trip form, as the reference's format_double (util.cpp:8-13)
std::string fmt(double v) {
  char buf[64];
  auto [ptr, ec] = std::to_chars(buf, buf + sizeof(buf), v);
  (void)ec;
  return std::string(buf, ptr);
}
}  // namespace

MbsDiagnosis diagnose_mbs_mismatch(double model_tflops, double hw_tflops, int cfg_mbs, int ds_mbs) {
  if (hw_tflops <= 0) throw std::invalid_argument("hardware FLOPS rate must be positive");
  if (cfg_mbs < 1 || ds_mbs < 1) throw std::invalid_argument("micro-batch sizes must be >= 1");
  MbsDiagnosis d;
  d.flops_ratio = model_tflops / hw_tflops;
  d.mbs_ratio = static_cast<double>(ds_mbs) / cfg_mbs;
  if (ds_mbs != cfg_mbs && std::abs(d.flops_ratio / d.mbs_ratio - 1.0) <= 0.10) {
    d.kind = MbsDiagnosisKind::MbsMismatch;
    d.message = "model FLOPS over-reported by factor " + fmt(d.mbs_ratio) +
                " due to micro-batch-size mismatch (train_micro_batch_size_per_gpu=" + std::to_string(ds_mbs) +
                " vs micro_batch_size=" + std::to_string(cfg_mbs) + ")";
  } else if (std::abs(d.flops_ratio - 1.0) <= 0.10) {
    d.kind = MbsDiagnosisKind::Consistent;
    d.message = "model and hardware FLOPS agree";
  } else {
    d.kind = MbsDiagnosisKind::UnexplainedDivergence;
    d.message = "model/hardware FLOPS ratio " + fmt(d.flops_ratio) + " not explained by the micro-batch settings";
  }
  return d;
}

RooflineReport roofline(double flops, double bytes, const ClusterSpec& cluster) {
  if (bytes <= 0) throw std::invalid_argument("bytes must be positive");
  if (flops < 0) throw std::invalid_argument("flops must be non-negative");
  if (cluster.hbm_bandwidth <= 0 || cluster.peak_flops_per_gpu <= 0)
    throw std::invalid_argument("cluster needs positive peak and hbm_bandwidth");
  RooflineReport r;
  r.total_flops = flops;
  r.total_bytes = bytes;
  r.arithmetic_intensity = flops / bytes;
  r.ridge_intensity = cluster.peak_flops_per_gpu / cluster.hbm_bandwidth;
  r.bound = r.arithmetic_intensity >= r.ridge_intensity ? RooflineBound::ComputeBound : RooflineBound::MemoryBound;
  return r;
}

RooflineReport roofline(const NcuCounterRecord& rec, const ClusterSpec& cluster) {
  return roofline(hw_flops(rec), static_cast<double>(rec.dram_read_bytes + rec.dram_write_bytes), cluster);
}

namespace {
void require_series(const std::vector<ScalingPoint>& s) {
  if (s.empty()) throw std::invalid_argument("empty scaling series");
  for (std::size_t i = 0; i < s.size(); ++i) {
    if (s[i].gpus <= 0 || s[i].value <= 0) throw std::invalid_argument("scaling points must be positive");
    if (i > 0 && s[i].gpus < s[i - 1].gpus)
      throw std::invalid_argument("series must be sorted by GPU count with the baseline first");
  }
}
}  // namespace

std::vector<double> weak_scaling(const std::vector<ScalingPoint>& s) {
  require_series(s);
  std::vector<double> e;
  for (const auto& p : s) e.push_back(p.value / s.front().value);
  return e;
}

std::vector<double> strong_scaling(const std::vector<ScalingPoint>& s) {
  require_series(s);
  std::vector<double> e;
  for (const auto& p : s) e.push_back((s.front().value / p.value) / (p.gpus / s.front().gpus));
  return e;
}

}  // namespace trainplan
