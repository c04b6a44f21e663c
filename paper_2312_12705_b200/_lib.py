"""ctypes binding of ``libtrainplan_b200.so`` (the C-ABI in include/trainplan/capi.h).

The library is the product: there is no Python or CPU fallback. ``load()`` raises if the
shared object is missing or does not export every symbol the header declares.
"""
from __future__ import annotations

import ctypes as C
import os
import re
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "lib" / "libtrainplan_b200.so"
if os.environ.get("GPTB200_LIB"):  # debugging aid: load an alternative build of the same library
    LIB_PATH = Path(os.environ["GPTB200_LIB"])
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

class TrainOptions(C.Structure):
    """tp_train_options."""
    _fields_ = [("seed", _u64), ("dropout", _f), ("lr", _f), ("beta1", _f), ("beta2", _f), ("eps", _f),
                ("weight_decay", _f)]

    def __init__(self, seed=1234, dropout=0.0, lr=1e-4, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.0):
        super().__init__(seed, dropout, lr, beta1, beta2, eps, weight_decay)


_i64, _sz = C.c_int64, C.c_size_t

KERNEL_CLASSES = ["gemm", "attn_fwd", "attn_bwd", "norm", "elementwise", "tp_comm", "pp_comm", "dp_comm", "adam"]


class KernelTimes(C.Structure):
    _fields_ = [("ms", C.c_double * 9), ("launches", C.c_int64 * 9), ("flops", C.c_double * 9),
                ("bytes", C.c_double * 9)]

    def as_dict(self):
        return {k: {"ms": self.ms[i], "launches": self.launches[i], "flops": self.flops[i], "bytes": self.bytes[i]}
                for i, k in enumerate(KERNEL_CLASSES)}
_ptr = C.c_void_p

# name -> (restype, argtypes)
SIGNATURES: dict[str, tuple] = {
    "tp_last_error": (C.c_char_p, []),
    "tp_abi_version": (_i, []),
    "tp_param_count": (_i, [C.POINTER(ModelSpec), C.POINTER(_u64)]),
    "tp_model_flops": (_i, [C.POINTER(ModelSpec), C.c_int64, _i, _i, C.POINTER(C.c_double)]),
    "tp_validate": (_i, [C.POINTER(ModelSpec), C.POINTER(ParallelConfig), _i, _i, _i, C.POINTER(Validation)]),
    "tp_pipeline_order": (_i, [_i, _i, _i, _i, _i, C.POINTER(_i), _i, C.POINTER(_i)]),
    "tp_pipeline_actions": (_i, [_i, _i, _i, _i, _i, _i, C.POINTER(_i), _i, C.POINTER(_i)]),
    "tp_rank_coords": (_i, [_i, _i, _i, _i, C.POINTER(_i)]),
    "tp_gemm_bf16": (_i, [_i, _i, _i, _vp, _i, _i, _vp, _i, _i, _vp, _i, _i, _vp, _vp, _vp, _i, _i, _vp]),
    "tp_gemm_force_cta_group": (_i, [_i]),
    "tp_flash_attn_fwd": (_i, [_i, _i, _i, _i, _vp, _vp, _vp, _vp]),
    "tp_flash_attn_bwd": (_i, [_i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "tp_resid_layernorm_fwd": (_i, [_i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _u64, _i, _i, _i, _f, _i64, _vp]),
    "tp_layernorm_bwd": (_i, [_i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _u64, _i, _i, _i, _f,
                              _i64, _vp, _vp]),
    "tp_layernorm_bwd_workspace_bytes": (_sz, [_i, _i]),
    "tp_cross_entropy": (_i, [_i, _i, _vp, _vp, _f, _vp, _vp, _vp]),
    "tp_adam_step": (_i, [_i64, _vp, _vp, _vp, _vp, _vp, _f, _f, _f, _f, _f, _i, _vp]),
    "tp_nccl_unique_id": (_i, [C.c_char_p]),
    "tp_session_create": (_i, [C.POINTER(ModelSpec), C.POINTER(ParallelConfig), C.POINTER(TrainOptions), _i, _i, _i,
                               C.c_char_p, C.POINTER(_vp)]),
    "tp_session_destroy": (_i, [_vp]),
    "tp_session_init_params": (_i, [_vp]),
    "tp_session_upload_tokens": (_i, [_vp, _vp, _i64, _i]),
    "tp_session_step": (_i, [_vp]),
    "tp_session_train_step": (_i, [_vp, _vp, _i64, C.POINTER(_f)]),
    "tp_session_read_loss": (_i, [_vp, C.POINTER(_f)]),
    "tp_session_eval_loss": (_i, [_vp, C.POINTER(_f)]),
    "tp_session_sync": (_i, [_vp]),
    "tp_session_barrier": (_i, [_vp]),
    "tp_session_tensor_info": (_i, [_vp, _i, C.POINTER(_i64)]),
    "tp_session_read_tensor": (_i, [_vp, _i, _i, _vp]),
    "tp_session_info": (_i, [_vp, C.POINTER(_i64)]),
    "tp_session_read_flat": (_i, [_vp, _i, _i64, _i64, _vp]),
    "tp_session_buckets": (_i, [_vp, C.POINTER(_i64), _i, C.POINTER(_i)]),
    "tp_session_time_steps": (_i, [_vp, _i, _i, C.POINTER(_f), C.POINTER(KernelTimes)]),
    "tp_session_step_times": (_i, [_vp, C.POINTER(_f), _i]),
    "tp_session_allreduce_max": (_i, [_vp, C.POINTER(_f)]),
    "tp_session_debug_tp_allreduce": (_i, [_vp, _vp, _vp, _i]),
    "tp_session_bench_tp_allreduce": (_i, [_vp, _i, _i, _i, C.POINTER(_f), C.POINTER(_i)]),
    "tp_session_bench_sp": (_i, [_vp, _i, _i, C.POINTER(_f)]),
    "tp_session_set_timeout": (_i, [_vp, C.c_double]),
    "tp_session_memory": (_i, [_vp, _vp]),
    "tp_variant_counts": (_i, [C.POINTER(_i64)]),
    "tp_variant_counts_reset": (_i, []),
    "tp_ncu_parse_csv": (_i, [C.c_char_p, C.c_size_t, C.c_char_p, _vp]),
    "tp_ncu_metric_list": (_i, [C.c_char_p, C.c_size_t]),
    "tp_diagnose_mbs_mismatch": (_i, [C.c_double, C.c_double, _i, _i, C.POINTER(_i), C.POINTER(C.c_double),
                                      C.c_char_p, C.c_size_t]),
}



class MemoryReport(C.Structure):
    """tp_memory_report (capi.h): measured per-category device bytes of a session."""
    _fields_ = [("params_bytes", _u64), ("gradient_bytes", _u64), ("optimizer_bytes", _u64),
                ("activation_bytes", _u64), ("workspace_bytes", _u64), ("window_bytes", _u64),
                ("total_bytes", _u64), ("zero_stage", _i)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


VARIANTS = ["gemm_single", "gemm_pair_256", "gemm_pair_512", "gemm_ksplit", "attn_fwd_persistent",
            "attn_fwd_per_block", "attn_bwd_per_block", "attn_bwd_persistent", "attn_bwd_hd64",
            "attn_bwd_hd160", "ln_bwd_stream", "ln_bwd_fused", "ln_bwd_two_pass", "attn_fwd_two_q"]


def variant_counts() -> dict:
    """Process-wide launch counts per kernel variant (tp_variant_counts)."""
    out = (_i64 * len(VARIANTS))()
    check(load().tp_variant_counts(out))
    return dict(zip(VARIANTS, list(out)))


def variant_counts_reset() -> None:
    check(load().tp_variant_counts_reset())


class HwCounters(C.Structure):
    """tp_hw_counters (capi.h): summed ncu counters of the selected launches."""
    _fields_ = [("launches", _u64), ("tensor_utc_bf16", _u64), ("tensor_utc_f16", _u64),
                ("tensor_hmma_bf16", _u64), ("tensor_hmma_f16", _u64), ("dram_read_bytes", _u64),
                ("dram_write_bytes", _u64), ("duration_ns", _u64), ("tensor_flops", C.c_double),
                ("simt_flops", C.c_double), ("hw_flops", C.c_double), ("num_warnings", _i)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


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


# ---------------------------------------------------------------- hardware counters
def ncu_parse_csv(text: str, kernel_filter: str | None = None) -> dict:
    """trainplan::parse_ncu_csv + hw_flops (metrics.hpp) over `ncu --csv` output."""
    raw = text.encode()
    out = HwCounters()
    check(load().tp_ncu_parse_csv(raw, len(raw), kernel_filter.encode() if kernel_filter else None,
                                  C.byref(out)))
    return out.as_dict()


def diagnose_mbs_mismatch(model_tflops: float, hw_tflops: float, cfg_mbs: int, ds_mbs: int) -> dict:
    """trainplan::diagnose_mbs_mismatch: kind 0 consistent / 1 MBS mismatch / 2 unexplained."""
    kind, ratio, msg = _i(), C.c_double(), C.create_string_buffer(512)
    check(load().tp_diagnose_mbs_mismatch(model_tflops, hw_tflops, cfg_mbs, ds_mbs, C.byref(kind),
                                          C.byref(ratio), msg, len(msg)))
    return {"kind": kind.value, "flops_ratio": ratio.value, "message": msg.value.decode()}


def ncu_metric_list() -> str:
    buf = C.create_string_buffer(4096)
    check(load().tp_ncu_metric_list(buf, len(buf)))
    return buf.value.decode()


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


PA_RECV, PA_SEND, PA_HEAD, PA_HEAD_LATE, PA_LAST_MB = 1, 2, 4, 8, 16


def pipeline_actions(p: int, m: int, v: int, device: int, dh_ring: int = 2, forward_only: bool = False) -> list[dict]:
    """The executable plan Stage::step() runs on `device` (runtime/pipe_exec.h)."""
    cap = 2 * m * v + 8
    buf = (_i * (6 * cap))()
    n = _i()
    check(load().tp_pipeline_actions(p, m, v, device, dh_ring, int(forward_only), buf, cap, C.byref(n)))
    keys = ("kind", "mb", "chunk", "slot", "dh", "flags")
    return [dict(zip(keys, buf[6 * i:6 * i + 6])) for i in range(n.value)]


def rank_coords(rank: int, tp: int, pp: int, dp: int) -> tuple[int, int, int]:
    out = (_i * 3)()
    check(load().tp_rank_coords(rank, tp, pp, dp, out))
    return out[0], out[1], out[2]


# ---------------------------------------------------------------- train-step session
def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(load().tp_nccl_unique_id(buf))
    return buf.raw


class Session:
    """One rank of the GPT train step (tp_session_* in capi.h)."""

    READ_PARAM, READ_GRAD, READ_MASTER, READ_ADAM_M, READ_ADAM_V = range(5)

    def __init__(self, spec: ModelSpec, cfg: ParallelConfig, opts: TrainOptions | None = None, rank: int = 0,
                 world: int = 1, device: int = 0, nccl_id: bytes | None = None):
        self._lib = load()
        self.spec, self.cfg = spec, cfg
        self.opts = opts or TrainOptions()
        h = _vp()
        check(self._lib.tp_session_create(C.byref(spec), C.byref(cfg), C.byref(self.opts), rank, world, device,
                                          nccl_id, C.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            check(self._lib.tp_session_destroy(self.h))
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def init_params(self):
        check(self._lib.tp_session_init_params(self.h))

    def upload_tokens(self, tokens, on_device: bool = False):
        """tokens: numpy int32 [gbs, s+1] (host) or a device address (int) with on_device."""
        if on_device:
            ptr, n = tokens
        else:
            import numpy as np
            arr = np.ascontiguousarray(tokens, dtype=np.int32)
            self._keep = arr
            ptr, n = arr.ctypes.data, arr.size
        check(self._lib.tp_session_upload_tokens(self.h, ptr, n, int(on_device)))

    def step(self):
        check(self._lib.tp_session_step(self.h))

    def train_step(self, tokens) -> float:
        import numpy as np
        arr = np.ascontiguousarray(tokens, dtype=np.int32)
        out = _f()
        check(self._lib.tp_session_train_step(self.h, arr.ctypes.data, arr.size, C.byref(out)))
        return out.value

    def read_loss(self) -> float:
        out = _f()
        check(self._lib.tp_session_read_loss(self.h, C.byref(out)))
        return out.value

    def eval_loss(self) -> float:
        out = _f()
        check(self._lib.tp_session_eval_loss(self.h, C.byref(out)))
        return out.value

    def sync(self):
        check(self._lib.tp_session_sync(self.h))

    def barrier(self):
        check(self._lib.tp_session_barrier(self.h))

    def tensor_info(self, tid: int) -> dict | None:
        info = (_i64 * 9)()
        check(self._lib.tp_session_tensor_info(self.h, tid, info))
        if not info[0]:
            return None
        keys = ["rows", "cols", "offset", "rseg", "rstride", "roff", "coff", "gcols"]
        return dict(zip(keys, list(info)[1:]))

    def read_tensor(self, which: int, tid: int):
        import numpy as np
        info = self.tensor_info(tid)
        if info is None:
            return None
        out = np.empty(info["rows"] * info["cols"], dtype=np.float32)
        check(self._lib.tp_session_read_tensor(self.h, which, tid, out.ctypes.data))
        return out.reshape(info["rows"], info["cols"]) if info["cols"] > 1 else out

    def time_steps(self, steps: int, profile: bool = False):
        ms = _f()
        kt = KernelTimes()
        check(self._lib.tp_session_time_steps(self.h, steps, int(profile), C.byref(ms), C.byref(kt)))
        return ms.value, (kt.as_dict() if profile else None)

    def step_times(self, steps: int) -> list:
        """Device ms of each step of the last time_steps call."""
        out = (_f * steps)()
        check(self._lib.tp_session_step_times(self.h, out, steps))
        return list(out)

    def allreduce_max(self, v: float) -> float:
        x = _f(v)
        check(self._lib.tp_session_allreduce_max(self.h, C.byref(x)))
        return x.value

    def debug_tp_allreduce(self, x, mode: int = 0):
        """x: uint16 bf16 bit patterns of one [mbs*s, d] buffer; returns the TP-summed buffer."""
        import numpy as np
        x = np.ascontiguousarray(x, dtype=np.uint16)
        out = np.empty_like(x)
        check(self._lib.tp_session_debug_tp_allreduce(self.h, x.ctypes.data, out.ctypes.data, mode))
        return out

    def bench_sp(self, iters: int = 20, mode: int = 0) -> float:
        ms = _f()
        check(self._lib.tp_session_bench_sp(self.h, iters, mode, C.byref(ms)))
        return ms.value

    def bench_tp_allreduce(self, iters: int = 20, mode: int = 0, ctas: int = 0):
        ms, nv = _f(), _i()
        check(self._lib.tp_session_bench_tp_allreduce(self.h, iters, mode, ctas, C.byref(ms), C.byref(nv)))
        return ms.value, bool(nv.value)

    def read_flat(self, which: int, offset: int, n: int):
        import numpy as np
        out = np.empty(n, dtype=np.float32)
        check(self._lib.tp_session_read_flat(self.h, which, offset, n, out.ctypes.data))
        return out

    def buckets(self) -> list[tuple[int, int, int]]:
        """ZeRO-1 buckets: (flat_offset, length, master_offset)."""
        buf = (_i64 * (3 * 4096))()
        n = _i()
        check(self._lib.tp_session_buckets(self.h, buf, 4096, C.byref(n)))
        return [(buf[3 * i], buf[3 * i + 1], buf[3 * i + 2]) for i in range(n.value)]

    def set_timeout(self, seconds: float) -> None:
        check(self._lib.tp_session_set_timeout(self.h, float(seconds)))

    def memory(self) -> dict:
        rep = MemoryReport()
        check(self._lib.tp_session_memory(self.h, C.byref(rep)))
        return rep.as_dict()

    def info(self) -> dict:
        out = (_i64 * 8)()
        check(self._lib.tp_session_info(self.h, out))
        keys = ["flat_params", "shard_params", "device_bytes", "microbatches", "launches", "rank", "world",
                "tp_mode"]
        return dict(zip(keys, list(out)))


def global_index_map(info: dict):
    """(global_rows, global_cols) index arrays of a local shard (mirrors the init kernel's map)."""
    import numpy as np
    r = np.arange(info["rows"])
    grow = (r // info["rseg"]) * info["rstride"] + info["roff"] + r % info["rseg"]
    gcol = info["coff"] + np.arange(info["cols"])
    return grow, gcol
