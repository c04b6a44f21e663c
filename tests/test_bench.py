"""bench.py contract pieces that run on CPU: the metric numerator and the reference arm.

The reference arm (--impl reference) must time the CPU implementation of the path without loading
anything from this repo's product library; its FLOP count is computed in Python integers."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

import bench
from paper_2312_12705_b200 import _lib as T

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("cfg", [(48, 6144, 48, 51200, 2048, 1, True), (24, 2048, 16, 51200, 2048, 32, False),
                                 (4, 25600, 160, 51200, 2048, 8, True), (2, 256, 4, 51200, 128, 8, False),
                                 (8, 12288, 96, 51200, 2048, 16, True)])
def test_python_model_flops_matches_library(native_lib, cfg):
    L, d, a, V, s, B, ck = cfg
    assert bench.model_flops(L, d, a, V, s, B, ck) == T.model_flops(T.ModelSpec(L, d, a, V, s), B, ck)


def test_python_model_flops_reference_golden():
    # proj/tests/test_arch.cpp:95-101: 22B, B = 1, checkpointing
    assert bench.model_flops(48, 6144, 48, 51200, 2048, 1, True) == 379898447265792.0


def test_reference_arm_loads_no_product_library(tmp_path):
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--workload", "gpt-tiny",
                        "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert not any("libtrainplan_b200" in p for p in line["native_libs"]), line["native_libs"]
    assert any("libgpt_oracle" in p for p in line["native_libs"])
    assert line["cpu_baseline"]["extrapolated"] is True
    c1 = line["cpu_baseline"]["config1_full_step"]
    assert c1["seconds"] > 0 and c1["tokens_per_s"] > 0 and c1["extrapolated"] is False
    assert line["e2e"]["value"] == line["value"]
