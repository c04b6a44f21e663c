"""The C++ drop-in layer (include/trainplan/train.hpp): compiled against the product library.

CPU: our Megatron-style iteration log line is parsed by the REFERENCE's own parse_training_log /
aggregate_model_flops (oracle/_ref/ref_parse_log, built from /root/reference sources).
GPU: TrainSession, measure() -> ThroughputEstimate and the measured Evaluator on a tiny model."""
import json
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
LIBDIR = ROOT / "paper_2312_12705_b200" / "lib"


def _build(src: Path, out: Path):
    cmd = ["g++", "-std=c++20", "-O1", f"-I{ROOT / 'include'}", str(src), "-o", str(out), f"-L{LIBDIR}",
           "-ltrainplan_b200", f"-Wl,-rpath,{LIBDIR}"]
    subprocess.run(cmd, check=True, capture_output=True)


def test_log_line_is_parsed_by_reference_parser(tmp_path, native_lib):
    ref = ROOT / "oracle" / "_ref" / "ref_parse_log"
    if not ref.exists():
        pytest.skip("reference library not built (needs /root/reference: make -C oracle ref)")
    exe = tmp_path / "log_line"
    _build(ROOT / "tests" / "cpp" / "log_line.cpp", exe)
    lines = subprocess.run([str(exe), "0.1625", "9.026e14"], check=True, capture_output=True, text=True).stdout
    parsed = json.loads(subprocess.run([str(ref)], input=lines, check=True, capture_output=True, text=True).stdout)
    assert parsed["entries"] == 3
    assert parsed["first_iteration"] == 1
    assert abs(parsed["first_iter_time"] - 0.1625) < 1e-4
    assert abs(parsed["aggregate_tflops"] - 902.6) < 0.01


@pytest.mark.gpu
def test_train_api_measure_and_evaluator(tmp_path, native_lib):
    exe = tmp_path / "train_api_smoke"
    _build(ROOT / "tests" / "cpp" / "train_api_smoke.cpp", exe)
    r = json.loads(subprocess.run([str(exe)], check=True, capture_output=True, text=True, timeout=300).stdout)
    assert r["oom"] == 0 and r["iter_time"] > 0 and r["flops_per_gpu"] > 0
    assert r["peak_fraction"] == pytest.approx(r["flops_per_gpu"] / 2.25e15)
    parts = r["compute"] + r["tp"] + r["pp"] + r["dp"] + r["bubble"]
    assert parts == pytest.approx(r["iter_time"], rel=0.05)
    assert r["invalid_throws"] == 1
    assert r["eval_ok_failed"] == 0 and r["eval_ok_tflops"] > 0
    assert r["eval_invalid_kind"] == 2  # FailureKind::Invalid
    assert r["loss5"] < r["loss0"]
    assert "elapsed time per iteration (ms):" in r["log"] and "TFLOPs:" in r["log"]
