"""ctypes binding of the CPU oracle (oracle/lib/libgpt_oracle.so) — test infrastructure only."""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
ORACLE_DIR = ROOT / "oracle"
LIB = ORACLE_DIR / "lib" / "libgpt_oracle.so"


class OrcModel(C.Structure):
    _fields_ = [("num_layers", C.c_int), ("hidden_size", C.c_int), ("num_heads", C.c_int),
                ("vocab_size", C.c_int), ("seq_length", C.c_int)]


class OrcOpts(C.Structure):
    _fields_ = [("dropout", C.c_float), ("seed", C.c_uint64), ("bf16_emulate", C.c_int),
                ("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float),
                ("weight_decay", C.c_float)]


_lib = None


def load():
    global _lib
    if _lib is None:
        if not LIB.exists():
            subprocess.run(["make", "-C", str(ORACLE_DIR)], check=True, capture_output=True)
        lib = C.CDLL(str(LIB))
        fp = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
        ip = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
        mp = C.POINTER(OrcModel)
        op = C.POINTER(OrcOpts)
        lib.orc_param_numel.restype = C.c_int64
        lib.orc_param_numel.argtypes = [mp]
        lib.orc_num_tensors.argtypes = [mp]
        lib.orc_tensor_info.argtypes = [mp, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        lib.orc_init_params.argtypes = [mp, C.c_uint64, fp]
        lib.orc_gen_tokens.argtypes = [C.c_uint64, C.c_int64, C.c_int, ip]
        lib.orc_fwd_bwd.restype = C.c_double
        lib.orc_fwd_bwd.argtypes = [mp, op, fp, ip, C.c_int, C.c_int64, C.c_int, C.c_double, fp, C.c_void_p]
        lib.orc_forward.restype = C.c_double
        lib.orc_forward.argtypes = [mp, op, fp, ip, C.c_int, C.c_int64, C.c_int, C.c_void_p]
        lib.orc_adam.argtypes = [C.c_int64, fp, fp, fp, fp, C.c_int, op]
        lib.orc_init_value.restype = C.c_float
        lib.orc_init_value.argtypes = [C.c_uint64, C.c_int, C.c_int64, C.c_float]
        lib.orc_dropout_keep.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int64, C.c_float]
        lib.orc_time_layer.restype = C.c_double
        lib.orc_time_layer.argtypes = [mp, C.c_int, C.c_int]
        lib.orc_bf16.restype = C.c_float
        lib.orc_bf16.argtypes = [C.c_float]
        _lib = lib
    return _lib


def model(L, d, heads, V, s) -> OrcModel:
    return OrcModel(L, d, heads, V, s)


def opts(dropout=0.0, seed=1234, bf16=0, lr=1e-3, b1=0.9, b2=0.95, eps=1e-8, wd=0.01) -> OrcOpts:
    return OrcOpts(dropout, seed, bf16, lr, b1, b2, eps, wd)


def tensor_info(m: OrcModel, tid: int):
    off, r, c = C.c_int64(), C.c_int64(), C.c_int64()
    load().orc_tensor_info(C.byref(m), tid, C.byref(off), C.byref(r), C.byref(c))
    return off.value, r.value, c.value


def init_params(m: OrcModel, seed: int) -> np.ndarray:
    lib = load()
    p = np.empty(lib.orc_param_numel(C.byref(m)), dtype=np.float32)
    lib.orc_init_params(C.byref(m), seed, p)
    return p


def gen_tokens(seed: int, n: int, vocab: int) -> np.ndarray:
    out = np.empty(n, dtype=np.int32)
    load().orc_gen_tokens(seed, n, vocab, out)
    return out


def fwd_bwd(m: OrcModel, o: OrcOpts, params: np.ndarray, tokens: np.ndarray, sample0=0, step=1,
            loss_scale=None, grads=None):
    lib = load()
    tokens = np.ascontiguousarray(tokens, dtype=np.int32)
    nseq = tokens.shape[0]
    if grads is None:
        grads = np.zeros_like(params)
    if loss_scale is None:
        loss_scale = 1.0 / (nseq * m.seq_length)
    loss = lib.orc_fwd_bwd(C.byref(m), C.byref(o), params, tokens, nseq, sample0, step, loss_scale, grads, None)
    return loss, grads


def tensor(m: OrcModel, flat: np.ndarray, tid: int) -> np.ndarray:
    off, r, c = tensor_info(m, tid)
    n = r * c
    return flat[off:off + n].reshape((r, c) if c > 1 else (r,))
