// Hardware-counter accounting on B200.
//
// The reference measures hardware FLOPs on MI250X from summed rocprof SQ_INSTS_VALU_* counters
// (/root/reference/proj/include/trainplan/metrics.hpp:13-35, proj/src/metrics.cpp:67-117) and
// checks them against the model FLOPs of the iteration log (PAPER.md:1031-1033,
// metrics.cpp:164-185). On B200 the same roles are played by Nsight Compute metrics:
//   tensor pipe  sm__ops_path_tensor_op_utchmma_src_{bf16,fp16}_dst_fp32 (tcgen05.mma, kind::f16)
//                sm__ops_path_tensor_op_hmma_src_{bf16,fp16}_dst_fp32    (legacy mma.sync)
//   SIMT         smsp__sass_thread_inst_executed_op_{fadd,fmul,ffma,fadd2,fmul2,ffma2,
//                hadd,hmul,hfma,dadd,dmul,dfma}_pred_on (thread-level instruction counts)
//   memory       dram__bytes_read / dram__bytes_write, gpu__time_duration
// NcuCounterRecord / parse_ncu_csv / hw_flops replace CounterRecord / parse_counter_csv /
// hw_flops; the agreement check, roofline and scaling helpers keep the reference's declarations
// (trainplan/metrics.hpp) and semantics (metrics.cpp:164-240).
#pragma once

#include <cstdint>
#include <iosfwd>
#include <map>
#include <string>
#include <vector>

#include "trainplan/cluster.hpp"
#include "trainplan/metrics.hpp"

namespace trainplan {

// Summed Nsight Compute counters of one or more kernel launches.
struct NcuCounterRecord {
  // tensor pipe, in ncu "math ops" (hw_flops converts with the measured coefficient)
  std::uint64_t tensor_utc_bf16 = 0, tensor_utc_f16 = 0;    // tcgen05.mma (UTCHMMA)
  std::uint64_t tensor_hmma_bf16 = 0, tensor_hmma_f16 = 0;  // mma.sync (HMMA)
  // SIMT floating-point thread instructions (predicated-on)
  std::uint64_t fadd = 0, fmul = 0, ffma = 0, fadd2 = 0, fmul2 = 0, ffma2 = 0;
  std::uint64_t hadd = 0, hmul = 0, hfma = 0;
  std::uint64_t dadd = 0, dmul = 0, dfma = 0;
  // DRAM traffic and device time
  std::uint64_t dram_read_bytes = 0, dram_write_bytes = 0;
  std::uint64_t duration_ns = 0;
  std::uint64_t launches = 0;

  NcuCounterRecord& operator+=(const NcuCounterRecord& other);
  friend NcuCounterRecord operator+(NcuCounterRecord a, const NcuCounterRecord& b) { return a += b; }
};

// FLOPs per ncu tensor "math op" — the analogue of the reference's MfmaCoeffMode::Measured512.
// UTCHMMA: measured on B200, one tcgen05 GEMM 4096^3 counts exactly 2*M*N*K = 137438953472 ops
// (profiles/r01_hwc_gemm_4096.csv, profiles/r01_hw_counters.json), so the counter is in FLOPs.
// HMMA (the mma.sync hd-160 attention fallback): same counter family, assumed 1 (uncalibrated).
constexpr double kB200FlopsPerUtcOp = 1.0;
constexpr double kB200FlopsPerHmmaOp = 1.0;

// Tensor FLOPs = coefficient * ops; SIMT FLOPs = add + mul + 2 fma, x2 for the paired fp32
// forms (FADD2/FMUL2/FFMA2) and for packed half2 (HADD2/HMUL2/HFMA2).
double hw_tensor_flops(const NcuCounterRecord& rec, double flops_per_utc_op = kB200FlopsPerUtcOp,
                       double flops_per_hmma_op = kB200FlopsPerHmmaOp);
double hw_simt_flops(const NcuCounterRecord& rec);
double hw_flops(const NcuCounterRecord& rec, double flops_per_utc_op = kB200FlopsPerUtcOp,
                double flops_per_hmma_op = kB200FlopsPerHmmaOp);

struct NcuParseResult {
  NcuCounterRecord totals;
  std::map<std::string, NcuCounterRecord> per_kernel;  // keyed by kernel name (demangled, as printed)
  std::size_t rows = 0;                                 // launches
  std::vector<std::string> warnings;                    // one per unknown metric name
};

// Parses `ncu --csv` output: the long form (one row per launch and metric, columns "ID",
// "Kernel Name", "Metric Name", "Metric Unit", "Metric Value") or the wide `--page raw --csv`
// form (a header of metric names, a units row, one row per launch). Thousands separators and
// SI unit prefixes (byte/Kbyte/Mbyte/Gbyte, nsecond/usecond/msecond/second) are normalised;
// metric names may carry a .sum suffix. Unknown metrics warn and are skipped; a negative or
// unparsable count throws std::invalid_argument, as parse_counter_csv does.
NcuParseResult parse_ncu_csv(std::istream& in);

// The metric list the parser understands (for `ncu --metrics`).
std::string ncu_metric_list();

// Roofline of counter totals: hw_flops over DRAM bytes (RooflineReport / roofline of metrics.hpp).
RooflineReport roofline(const NcuCounterRecord& rec, const ClusterSpec& cluster);

}  // namespace trainplan
