"""The drop-in boundary: reference-side C++ compiles and links unchanged against this library.

* The footprint model and perf helpers defined by libtrainplan_b200.so (memory_per_gpu,
  activation_bytes, bytes_per_param, saturation_check, config_from_point, make_point_validator,
  training_budget) print byte-identical answers to the reference library compiled from its own
  sources (tests/golden/ref_memory.json, `make -C oracle golden`).
* tests/cpp/dropin_search.cpp — reference-style code calling run_search / estimate / calibrate /
  simulate / cluster costs / util next to train.hpp — compiles against this repo's restated headers
  AND with the reference's own include directory first (reference headers + only train.hpp /
  b200.hpp / capi.h from here), links libtrainplan_b200.so + the reference library, and both builds
  give identical planner results.
* Every ```c / ```cpp snippet of INTEGRATION.md compiles and links.
* GPU: the reference's run_search driven by make_measured_evaluator, calibrate() fed the measured
  observations, an OOM point, and the measured footprint beside memory_per_gpu.
"""
import json
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
LIBDIR = ROOT / "paper_2312_12705_b200" / "lib"
REF_LIB = ROOT / "oracle" / "_ref" / "libtrainplan_ref.a"
REF_INC = Path("/root/reference/proj/include")


def _link(src: Path, out: Path, incs=(ROOT / "include",), ref_lib=True, lang="c++"):
    cc = ["g++", "-std=c++20"] if lang == "c++" else ["gcc", "-std=c11"]
    cmd = [*cc, "-O1", *[f"-I{i}" for i in incs], str(src), "-o", str(out), f"-L{LIBDIR}", "-ltrainplan_b200",
           f"-Wl,-rpath,{LIBDIR}"]
    if ref_lib:
        cmd.append(str(REF_LIB))
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]


def _need_ref_lib():
    if not REF_LIB.exists():
        pytest.skip("reference library not built (make -C oracle ref needs /root/reference)")


def test_memory_model_matches_reference(tmp_path, native_lib):
    exe = tmp_path / "plan_dump"
    _link(ROOT / "tests" / "cpp" / "plan_dump.cpp", exe, ref_lib=False)
    ours = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout
    ref = (ROOT / "tests" / "golden" / "ref_memory.json").read_text()
    assert json.loads(ours) == json.loads(ref)
    assert ours == ref  # byte-identical, including the order of every field


def test_reference_code_compiles_against_restated_headers(tmp_path, native_lib):
    _need_ref_lib()
    exe = tmp_path / "dropin"
    _link(ROOT / "tests" / "cpp" / "dropin_search.cpp", exe)
    out = json.loads(subprocess.run([str(exe), "cpu"], check=True, capture_output=True, text=True).stdout)
    assert len(out["history"]) == 12 and out["best_objective"] > 0
    assert out["sim_events"] == 16
    assert out["calibrated_synthetic"] == pytest.approx(0.42)
    assert out["saturation"].startswith("pipeline unsaturated")
    if REF_INC.exists():  # the same translation unit with the reference's headers first
        exe2 = tmp_path / "dropin_refhdr"
        _link(ROOT / "tests" / "cpp" / "dropin_search.cpp", exe2, incs=(REF_INC, ROOT / "include"))
        out2 = json.loads(subprocess.run([str(exe2), "cpu"], check=True, capture_output=True, text=True).stdout)
        assert out2 == out


def _snippets():
    text = (ROOT / "INTEGRATION.md").read_text()
    return [(m.group(1), m.group(2)) for m in re.finditer(r"```(c|cpp)\n(.*?)```", text, re.S)]


def test_integration_snippets_compile(tmp_path, native_lib):
    _need_ref_lib()
    snips = _snippets()
    assert len(snips) >= 2
    for i, (lang, code) in enumerate(snips):
        src = tmp_path / f"snip{i}.{'c' if lang == 'c' else 'cpp'}"
        src.write_text(code)
        _link(src, tmp_path / f"snip{i}", lang="c" if lang == "c" else "c++", ref_lib=lang == "cpp")


@pytest.mark.gpu
def test_measured_evaluator_drives_reference_search(tmp_path, native_lib):
    _need_ref_lib()
    exe = tmp_path / "dropin"
    _link(ROOT / "tests" / "cpp" / "dropin_search.cpp", exe)
    r = subprocess.run([str(exe), "gpu"], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    out = json.loads(r.stdout)
    hist = out["history"]
    assert len(hist) == 6
    ok = [h for h in hist if h["failure"] == "none"]
    assert ok and all(h["objective"] > 0 and h["wall_time"] > 0 for h in ok)
    assert out["best_objective"] == max(h["objective"] for h in ok)
    # the reference's calibrate fitted to measured B200 points
    assert out["observations"] == len(ok)
    assert 0.2 <= out["calibrated_kernel_efficiency"] <= 1.0
    assert out["oom_failure"] == "oom"
    P = out["executed_params"]
    meas = out["measured_mem"]
    # fp32 main grads for every (padded) parameter, bf16 working copy + fp32 master, Adam m + v
    assert 4 * P <= meas["gradients"] <= 4 * P * 1.01
    assert 6 * P <= meas["params"] <= 6 * P * 1.01
    assert 8 * P <= meas["optimizer"] <= 8 * P * 1.01
    assert meas["fits"] == 1 and out["model_mem"]["fits"] == 1
    print(json.dumps({"model_mem": out["model_mem"], "measured_mem": meas, "calibrated_kernel_efficiency":
                      out["calibrated_kernel_efficiency"], "history": hist}))
