"""Hardware-counter accounting: trainplan::parse_ncu_csv / hw_flops (the B200
replacement of the reference's parse_counter_csv / hw_flops over AMD SQ_* counters,
proj/src/metrics.cpp:67-117) and the restated diagnose_mbs_mismatch / roofline / scaling helpers,
checked against the reference's own functions (oracle/_ref/ref_metrics, built from
/root/reference sources)."""
import subprocess
from pathlib import Path

import pytest

from paper_2312_12705_b200 import _lib as T

ROOT = Path(__file__).resolve().parents[1]
LIBDIR = ROOT / "paper_2312_12705_b200" / "lib"

HDR = '"ID","Process ID","Process Name","Host Name","Kernel Name","Context","Stream","Block Size","Grid Size",' \
      '"Device","CC","Section Name","Metric Name","Metric Unit","Metric Value"'


def _row(i, kernel, metric, unit, value):
    return f'"{i}","11","python","box","{kernel}","1","7","(128, 1, 1)","(148, 1, 1)","0","10.0","Command line profiler metrics","{metric}","{unit}","{value}"'


LONG = "\n".join([
    "==PROF== Connected to process 11",
    HDR,
    _row(0, "gemm_sm100_kernel<2, 0>", "dram__bytes_read.sum", "Mbyte", "1,234.5"),
    _row(0, "gemm_sm100_kernel<2, 0>", "dram__bytes_write.sum", "byte", "1000"),
    _row(0, "gemm_sm100_kernel<2, 0>", "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum", "", "68,719,476,736"),
    _row(0, "gemm_sm100_kernel<2, 0>", "gpu__time_duration.sum", "usecond", "110.5"),
    _row(0, "gemm_sm100_kernel<2, 0>", "l1tex__t_bytes.sum", "byte", "7"),
    _row(1, "ln_fwd_kernel", "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "inst", "100"),
    _row(1, "ln_fwd_kernel", "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum", "inst", "10"),
    _row(1, "ln_fwd_kernel", "smsp__sass_thread_inst_executed_op_ffma2_pred_on.sum", "inst", "5"),
    _row(1, "ln_fwd_kernel", "smsp__sass_thread_inst_executed_op_hfma_pred_on.sum", "inst", "3"),
    _row(1, "ln_fwd_kernel", "gpu__time_duration.sum", "nsecond", "2500"),
    _row(2, "gemm_sm100_kernel<2, 0>", "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum", "", "1000"),
    _row(2, "gemm_sm100_kernel<2, 0>", "sm__ops_path_tensor_op_hmma_src_bf16_dst_fp32.sum", "", "10"),
    "==PROF== Disconnected from process 11",
])


def test_parse_long_form(native_lib):
    t = T.ncu_parse_csv(LONG)
    assert t["launches"] == 3
    assert t["dram_read_bytes"] == 1_234_500_000 and t["dram_write_bytes"] == 1000
    assert t["tensor_utc_bf16"] == 68_719_476_736 + 1000 and t["tensor_hmma_bf16"] == 10
    assert t["duration_ns"] == 110_500 + 2500
    assert t["tensor_flops"] == pytest.approx(1.0 * (68_719_476_736 + 1000 + 10))
    # FFMA 2, FADD 1, FFMA2 4, HFMA2 4 FLOPs per thread instruction
    assert t["simt_flops"] == 2 * 100 + 10 + 4 * 5 + 4 * 3
    assert t["hw_flops"] == pytest.approx(t["tensor_flops"] + t["simt_flops"])
    assert t["num_warnings"] == 1  # l1tex__t_bytes: unknown metric, skipped once
    g = T.ncu_parse_csv(LONG, "gemm_sm100")
    assert g["launches"] == 2 and g["simt_flops"] == 0 and g["duration_ns"] == 110_500
    ln = T.ncu_parse_csv(LONG, "ln_fwd")
    assert ln["launches"] == 1 and ln["tensor_flops"] == 0


def test_parse_wide_raw_form(native_lib):
    text = "\n".join([
        '"ID","Kernel Name","dram__bytes_read.sum","gpu__time_duration.sum",'
        '"sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum","sm__sass_thread_inst_executed_op_fmul_pred_on.sum",'
        '"launch__grid_size"',
        '"","","Kbyte","msecond","","inst",""',
        '"0","gemm_sm100_kernel","2","0.5","100","0","148"',
        '"1","fa_fwd_tc_kernel","1.5","0.25","50","7","296"',
    ])
    t = T.ncu_parse_csv(text)
    assert t["launches"] == 2
    assert t["dram_read_bytes"] == 3500 and t["duration_ns"] == 750_000
    assert t["tensor_utc_bf16"] == 150 and t["simt_flops"] == 7
    assert t["num_warnings"] == 1  # launch__grid_size
    assert T.ncu_parse_csv(text, "fa_fwd")["tensor_utc_bf16"] == 50


@pytest.mark.parametrize("bad", ["-5", "12abc", "n/a"])
def test_parse_rejects_bad_counts(native_lib, bad):
    text = HDR + "\n" + _row(0, "k", "dram__bytes_read.sum", "byte", bad)
    with pytest.raises(T.TrainplanError) as e:
        T.ncu_parse_csv(text)
    assert e.value.code == 1  # std::invalid_argument, as the reference's parse_counter_csv


def test_parse_rejects_empty_and_ragged(native_lib):
    with pytest.raises(T.TrainplanError):
        T.ncu_parse_csv("")
    with pytest.raises(T.TrainplanError):
        T.ncu_parse_csv(HDR + '\n"0","k"')


def test_metric_list_roundtrips(native_lib):
    names = T.ncu_metric_list().split(",")
    assert "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum" in names
    text = HDR + "\n" + "\n".join(_row(0, "k", n, "", "1") for n in names)
    t = T.ncu_parse_csv(text)
    assert t["num_warnings"] == 0 and t["launches"] == 1


RECORDS = """D 200 100 1 2
D 100 97 1 1
D 150.5 100 1 1
D 95 100 4 4
D 190 100 2 4
D 1109.2 1095.7 16 16
R 1e15 1e11 2.25e15 8e12
R 1e12 1e11 2.25e15 6.4568e12
W 4 1 1109.2 2 1088.4 4 1079 8 1050
S 3 1 10 2 5.2 4 2.9
"""


def test_restated_semantics_match_reference(tmp_path, native_lib):
    ref = ROOT / "oracle" / "_ref" / "ref_metrics"
    if not ref.exists():
        pytest.skip("reference library not built (needs /root/reference: make -C oracle ref)")
    exe = tmp_path / "metrics_cli"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{ROOT / 'include'}", str(ROOT / "tests" / "cpp" / "metrics_cli.cpp"),
                    "-o", str(exe), f"-L{LIBDIR}", "-ltrainplan_b200", f"-Wl,-rpath,{LIBDIR}"],
                   check=True, capture_output=True)
    ours = subprocess.run([str(exe)], input=RECORDS, check=True, capture_output=True, text=True).stdout
    theirs = subprocess.run([str(ref)], input=RECORDS, check=True, capture_output=True, text=True).stdout
    assert ours == theirs


def test_diagnose_through_c_abi(native_lib):
    d = T.diagnose_mbs_mismatch(200.0, 100.0, 1, 2)
    assert d["kind"] == 1 and d["flops_ratio"] == 2.0 and "micro-batch-size mismatch" in d["message"]
    assert T.diagnose_mbs_mismatch(100.0, 97.0, 1, 1)["kind"] == 0
    assert T.diagnose_mbs_mismatch(150.0, 100.0, 1, 1)["kind"] == 2
    with pytest.raises(T.TrainplanError):
        T.diagnose_mbs_mismatch(1.0, 0.0, 1, 1)


def test_executed_flops_model():
    """The executed-tensor-FLOP model of tools/hw_counters.py: causal tiling ~ half the dense
    attention, GEMMs exact."""
    import sys
    sys.path.insert(0, str(ROOT / "tools"))
    import hw_counters as H
    e = H.executed_tensor_flops(24, 2048, 16, 51200, 2048, 16, False)
    M = 16 * 2048
    assert e["gemm"] == 3 * 2 * M * 2048 * 12 * 2048 * 24 + 6 * M * 51200 * 2048
    assert e["attention_causal_fraction_fwd"] == pytest.approx(136 / 256)
    dense_fwd = 16 * 16 * 24 * 4 * 2048 * 2048 * 128
    assert e["attention_fwd"] == pytest.approx(dense_fwd * 136 / 256)
    assert e["attention_bwd"] == pytest.approx(2.5 * dense_fwd * 272 / 512)


def test_measured_step_counters_match_executed_flops(native_lib):
    """The ncu capture of one GPT-1.4B MBS-16 train step on a B200 (profiles/, application replay,
    cuProfilerStart/Stop around exactly one step): the tcgen05 tensor FLOPs the hardware counted
    equal, to the FLOP, every GEMM's 2*M*N*K plus the causal attention tiles the kernels visit;
    the model FLOPs of the reference formula agree with the hardware FLOPs (diagnose: consistent)."""
    import gzip
    import sys
    sys.path.insert(0, str(ROOT / "tools"))
    import hw_counters as H
    gemm = T.ncu_parse_csv((ROOT / "profiles" / "r01_hwc_gemm_4096.csv").read_text())
    assert gemm["launches"] == 1 and gemm["tensor_utc_bf16"] == 2 * 4096 ** 3
    text = gzip.open(ROOT / "profiles" / "r01_hwc_step_gpt1.4b.csv.gz", "rt").read()
    step = T.ncu_parse_csv(text)
    exp = H.executed_tensor_flops(24, 2048, 16, 51200, 2048, 16, False)
    assert step["tensor_flops"] == exp["total"]
    assert T.ncu_parse_csv(text, "gemm_sm100")["tensor_flops"] == exp["gemm"]
    assert T.ncu_parse_csv(text, "fa_fwd")["tensor_flops"] == exp["attention_fwd"]
    assert T.ncu_parse_csv(text, "fa_bwd")["tensor_flops"] == exp["attention_bwd"]
    model = T.model_flops(T.ModelSpec(24, 2048, 16, 51200, 2048), 16, False)
    d = T.diagnose_mbs_mismatch(model, step["hw_flops"], 16, 16)
    assert d["kind"] == 0, d
