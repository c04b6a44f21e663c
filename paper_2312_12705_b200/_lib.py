"""ctypes binding of ``libtrainplan_b200.so`` (the C-ABI in include/trainplan/capi.h).

The library is the product: there is no Python or CPU fallback. ``load()`` raises if the
shared object is missing or does not export every symbol the header declares.
"""
from __future__ import annotations

import ctypes as C
import re
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "lib" / "libtrainplan_b200.so"
HEADER = PKG.parent / "include" / "trainplan" / "capi.h"

_vp, _i, _f, _u64 = C.c_void_p, C.c_int, C.c_float, C.c_uint64


class ModelSpec(C.Structure):
    """tp_model_spec (trainplan::ModelSpec)."""
    _fields_ = [("num_layers", _i), ("hidden_size", _i), ("num_heads", _i), ("vocab_size", _i),
                ("seq_length", _i)]


class ParallelConfig(C.Structure):
    """tp_parallel_config (trainplan::ParallelConfig)."""
    _fields_ = [("tp", _i), ("pp", _i), ("dp", _i), ("mbs", _i), ("gbs", _i), ("zero_stage", _i),
                ("interleave_v", _i), ("precision", _i), ("grad_accum_fp32", _i),
                ("checkpoint_activations", _i), ("flash_attention", _i)]

    def __init__(self, tp=1, pp=1, dp=0, mbs=1, gbs=1, zero_stage=0, interleave_v=1, precision=1,
                 grad_accum_fp32=1, checkpoint_activations=0, flash_attention=1):
        super().__init__(tp, pp, dp, mbs, gbs, zero_stage, interleave_v, precision, grad_accum_fp32,
                         checkpoint_activations, flash_attention)


class Validation(C.Structure):
    _fields_ = [("ok", _i), ("dp", _i), ("num_microbatches", _i), ("num_violations", _i),
                ("fields", (C.c_char * 24) * 16), ("hard", _i * 16), ("first_message", C.c_char * 256)]

    def violations(self):
        return [(self.fields[i].value.decode(), self.hard[i]) for i in range(min(self.num_violations, 16))]

# name -> (restype, argtypes)
SIGNATURES: dict[str, tuple] = {
    "tp_last_error": (C.c_char_p, []),
    "tp_abi_version": (_i, []),
    "tp_param_count": (_i, [C.POINTER(ModelSpec), C.POINTER(_u64)]),
    "tp_model_flops": (_i, [C.POINTER(ModelSpec), C.c_int64, _i, _i, C.POINTER(C.c_double)]),
    "tp_validate": (_i, [C.POINTER(ModelSpec), C.POINTER(ParallelConfig), _i, _i, _i, C.POINTER(Validation)]),
    "tp_pipeline_order": (_i, [_i, _i, _i, _i, _i, C.POINTER(_i), _i, C.POINTER(_i)]),
    "tp_rank_coords": (_i, [_i, _i, _i, _i, C.POINTER(_i)]),
    "tp_gemm_bf16": (_i, [_i, _i, _i, _vp, _i, _i, _vp, _i, _i, _vp, _i, _i, _vp, _vp, _vp, _i, _i, _vp]),
}

_lib = None


class TrainplanError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def header_symbols() -> list[str]:
    """Every function the C-ABI header declares."""
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(tp_[a-z0-9_]+)\s*\(", text)))


def load() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(f"{LIB_PATH} not built; run paper_2312_12705_b200/build.py")
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(code: int) -> None:
    if code != 0:
        raise TrainplanError(code, load().tp_last_error().decode())


def gemm_bf16(M, N, K, A, lda, a_mn, B, ldb, b_mn, Cm, ldc, epi=0, bias=None, C2=None, aux=None,
              ldaux=0, accumulate=0, stream=None) -> None:
    """Raw pointer GEMM (device addresses as ints)."""
    check(load().tp_gemm_bf16(M, N, K, A, lda, int(a_mn), B, ldb, int(b_mn), Cm, ldc, epi, bias, C2,
                              aux, ldaux, accumulate, stream))


# ---------------------------------------------------------------- plan layer
def param_count(spec: ModelSpec) -> dict:
    out = (_u64 * 6)()
    check(load().tp_param_count(C.byref(spec), out))
    keys = ["attention", "ffn", "embedding", "total_exact", "total_approx", "executed_total"]
    return dict(zip(keys, [int(x) for x in out]))


def model_flops(spec: ModelSpec, batch: int, ckpt: bool, factor: int = 4) -> float:
    out = C.c_double()
    check(load().tp_model_flops(C.byref(spec), batch, int(ckpt), factor, C.byref(out)))
    return out.value


def validate(spec: ModelSpec, cfg: ParallelConfig, num_nodes=1, gpus_per_node=8, kernel_checks=False) -> Validation:
    v = Validation()
    check(load().tp_validate(C.byref(spec), C.byref(cfg), num_nodes, gpus_per_node, int(kernel_checks), C.byref(v)))
    return v


def pipeline_order(kind: int, p: int, m: int, v: int, device: int) -> list[tuple[int, int, int]]:
    cap = 2 * m * v + 8
    buf = (_i * (3 * cap))()
    n = _i()
    check(load().tp_pipeline_order(kind, p, m, v, device, buf, cap, C.byref(n)))
    return [(buf[3 * i], buf[3 * i + 1], buf[3 * i + 2]) for i in range(n.value)]


def rank_coords(rank: int, tp: int, pp: int, dp: int) -> tuple[int, int, int]:
    out = (_i * 3)()
    check(load().tp_rank_coords(rank, tp, pp, dp, out))
    return out[0], out[1], out[2]
