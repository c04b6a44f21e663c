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

# name -> (restype, argtypes)
SIGNATURES: dict[str, tuple] = {
    "tp_last_error": (C.c_char_p, []),
    "tp_abi_version": (_i, []),
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
