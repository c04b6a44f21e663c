"""The product's structural plan layer (C++, via the C-ABI) against the reference library's own
answers (tests/golden/ref_structural.json, produced by oracle/_ref/ref_dump linked against the
reference sources: `make -C oracle golden`)."""
import json

import pytest

from paper_2312_12705_b200 import _lib as T

REF = json.loads((T.PKG.parent / "tests" / "golden" / "ref_structural.json").read_text())


def spec(a):
    return T.ModelSpec(*a)


def test_library_exports_every_header_symbol(native_lib):
    for name in T.header_symbols():
        assert hasattr(native_lib, name), name


@pytest.mark.parametrize("case", REF["param_count"], ids=lambda c: str(c["spec"]))
def test_param_count_matches_reference(native_lib, case):
    got = T.param_count(spec(case["spec"]))
    for k in ["attention", "ffn", "embedding", "total_exact", "total_approx"]:
        assert got[k] == case[k], k
    L, d, a, V, s = case["spec"]
    assert got["executed_total"] == L * (12 * d * d + 13 * d) + (V + s) * d + 2 * d


def test_param_count_reference_goldens(native_lib):
    # proj/tests/test_arch.cpp:19-33 (22B / 175B / 1T presets of the reference)
    assert T.param_count(spec([48, 6144, 48, 51200, 2048]))["total_approx"] == 21743271936
    assert T.param_count(spec([96, 12288, 96, 51200, 2048]))["total_approx"] == 173946175488
    assert T.param_count(spec([128, 25600, 128, 51200, 2048]))["total_approx"] == 1006632960000


def test_model_flops_matches_reference(native_lib):
    for case in REF["model_flops"]:
        got = T.model_flops(spec(case["spec"]), case["batch"], bool(case["ckpt"]))
        assert got == case["flops"], case
    # proj/tests/test_arch.cpp:95-101
    assert T.model_flops(spec([48, 6144, 48, 51200, 2048]), 1, True) == 379898447265792.0


@pytest.mark.parametrize("case", REF["validate"], ids=lambda c: str(c["cfg"]))
def test_validate_matches_reference(native_lib, case):
    tp, pp, dp, mbs, gbs, zero = case["cfg"]
    v = T.validate(spec(case["spec"]), T.ParallelConfig(tp, pp, dp, mbs, gbs, zero), case["nodes"], case["gpn"])
    assert v.ok == case["ok"]
    assert v.dp == case["dp"]
    assert v.num_microbatches == case["m"]
    assert [list(x) for x in v.violations()] == case["fields"]


@pytest.mark.parametrize("case", REF["schedules"], ids=lambda c: f"p{c['p']}m{c['m']}v{c['v']}")
def test_pipeline_order_matches_reference_simulate(native_lib, case):
    kind = 2 if case["v"] > 1 else 1
    for dev in range(case["p"]):
        got = [list(x) for x in T.pipeline_order(kind, case["p"], case["m"], case["v"], dev)]
        assert got == case["order"][dev]


def test_1f1b_reference_kat(native_lib):
    # SURVEY.md §8 a7 / proj/tests/test_pipesim.cpp:73-89: p=2, m=4
    fmt = lambda ops: " ".join(("B" if b else "F") + str(mb) for b, mb, _ in ops)
    assert fmt(T.pipeline_order(1, 2, 4, 1, 0)) == "F0 F1 B0 F2 B1 F3 B2 B3"
    assert fmt(T.pipeline_order(1, 2, 4, 1, 1)) == "F0 B0 F1 B1 F2 B2 F3 B3"


def test_rank_layout(native_lib):
    # perf.cpp:15-20 convention; config 1 (TP2 PP2 DP2): TP {0,1}, PP {0,2}, DP {0,4}
    seen = set()
    for r in range(8):
        t, p, d = T.rank_coords(r, 2, 2, 2)
        assert r == t + 2 * (p + 2 * d)
        seen.add((t, p, d))
    assert len(seen) == 8
    assert T.rank_coords(2, 2, 2, 2) == (0, 1, 0)
    assert T.rank_coords(4, 2, 2, 2) == (0, 0, 1)
    with pytest.raises(T.TrainplanError):
        T.rank_coords(8, 2, 2, 2)


def test_invalid_shapes_raise(native_lib):
    with pytest.raises(T.TrainplanError) as e:
        T.param_count(spec([0, 1, 1, 1, 1]))
    assert e.value.code == 1


def test_kernel_constraints(native_lib):
    v = T.validate(spec([24, 2048, 16, 51200, 2048]), T.ParallelConfig(1, 1, 1, 8, 8, 1), 1, 1, kernel_checks=True)
    assert v.ok
    v = T.validate(spec([2, 256, 4, 1000, 128]), T.ParallelConfig(2, 1, 1, 1, 8, 1), 1, 2, kernel_checks=True)
    assert not v.ok and "vocab_size" in [f for f, _ in v.violations()]
