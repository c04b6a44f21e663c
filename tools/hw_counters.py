#!/usr/bin/env python
"""B200 hardware-counter accounting of the train step.

The paper checks the model FLOPs of its iteration log against hardware FLOPs summed from
rocprof SQ_* counters (reference: proj/src/metrics.cpp:67-117 parse_counter_csv / hw_flops,
:164-185 diagnose_mbs_mismatch). Here the counters are Nsight Compute metrics, parsed and
converted by the library's trainplan::parse_ncu_csv / hw_flops (include/trainplan/metrics.hpp,
C-ABI tp_ncu_parse_csv):

  # on the GPU box (one GPU; application replay re-runs the command once per metric pass)
  M=$(python tools/hw_counters.py metrics)
  ncu --replay-mode application --profile-from-start off --metrics $M --csv --print-units base \\
      --log-file gpurun_out/hwc_gemm.csv python tools/hw_counters.py run-gemm 4096 4096 4096
  ncu ... --log-file gpurun_out/hwc_step.csv python tools/hw_counters.py run-step --workload gpt-1.4b-mbs16
  # anywhere
  python tools/hw_counters.py analyze --gemm-csv gpurun_out/hwc_gemm.csv --gemm 4096 4096 4096 \\
      --step-csv gpurun_out/hwc_step.csv --workload gpt-1.4b-mbs16 > profiles/r01_hw_counters.json

`run-*` bracket exactly the measured work with cuProfilerStart/Stop (one GEMM launch; one full
train step after two warm-up steps), so the CSV holds nothing else.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2312_12705_b200 import _lib as T  # noqa: E402


def _profiler(on: bool) -> None:
    cuda = C.CDLL("libcuda.so.1")
    rc = (cuda.cuProfilerStart if on else cuda.cuProfilerStop)()
    if rc != 0:
        raise RuntimeError(f"cuProfiler{'Start' if on else 'Stop'} failed: {rc}")


def run_gemm(M: int, N: int, K: int) -> None:
    import torch
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn(N, K, device="cuda").bfloat16()
    Cm = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    st = torch.cuda.current_stream().cuda_stream
    call = lambda: T.gemm_bf16(M, N, K, A.data_ptr(), K, 0, B.data_ptr(), K, 0, Cm.data_ptr(), N, stream=st)  # noqa: E731
    call()
    torch.cuda.synchronize()
    _profiler(True)
    call()
    torch.cuda.synchronize()
    _profiler(False)
    print("ok")


def _workload(name: str):
    import bench
    L, d, a, V, s, mbs, tp, pp, ckpt, drop, nmb = bench.WORKLOADS[name]
    if tp * pp != 1:
        raise SystemExit("run-step profiles a single-GPU workload")
    return L, d, a, V, s, mbs, ckpt, drop, nmb


def run_step(name: str) -> None:
    L, d, a, V, s, mbs, ckpt, drop, nmb = _workload(name)
    gbs = mbs * nmb
    spec = T.ModelSpec(L, d, a, V, s)
    cfg = T.ParallelConfig(tp=1, pp=1, dp=1, mbs=mbs, gbs=gbs, zero_stage=1, checkpoint_activations=int(ckpt))
    with T.Session(spec, cfg, T.TrainOptions(seed=1234, dropout=drop, lr=1e-4)) as sess:
        sess.init_params()
        sess.upload_tokens(np.random.default_rng(1234).integers(0, V, size=(gbs, s + 1), dtype=np.int32))
        sess.time_steps(2)
        sess.sync()
        _profiler(True)
        sess.step()
        sess.sync()
        _profiler(False)
        print("loss", sess.read_loss())


def executed_tensor_flops(L, d, a, V, s, B, ckpt, q_fwd=128, kv=128, q_bwd=64) -> dict:
    """FLOPs the step's tensor-core kernels execute: every GEMM exactly (2*M*N*K), attention by
    the causal tiles the kernels visit (diagonal tiles computed whole; fwd q tile q_fwd x kv tile
    kv, bwd q tile q_bwd x kv block kv; fwd 2 MMAs, bwd 5 per tile pair)."""
    M, hd = B * s, d // a
    layer_gemm = 2 * M * d * 12 * d  # QKV 3d, W_o d, fc1 4d, fc2 4d (x d)
    gemm = 3 * layer_gemm * L + (layer_gemm * L if ckpt else 0) + 3 * 2 * M * V * d
    nq, nk = s // q_fwd, s // kv
    fwd_pairs = sum(min(nk, ((i + 1) * q_fwd + kv - 1) // kv) for i in range(nq))
    nqb = s // q_bwd
    bwd_pairs = sum(nqb - (j * kv) // q_bwd for j in range(nk))
    heads = B * a * L
    attn_fwd = heads * fwd_pairs * 2 * (2 * q_fwd * kv * hd)
    attn_bwd = heads * bwd_pairs * 5 * (2 * q_bwd * kv * hd)
    attn = attn_fwd * (2 if ckpt else 1) + attn_bwd
    return {"gemm": float(gemm), "attention_fwd": float(attn_fwd), "attention_bwd": float(attn_bwd),
            "attention_causal_fraction_fwd": fwd_pairs / (nq * nk), "total": float(gemm + attn)}


def analyze(args) -> dict:
    out: dict = {"metrics": T.ncu_metric_list().split(","),
                 "parser": "trainplan::parse_ncu_csv / hw_flops (include/trainplan/metrics.hpp) via tp_ncu_parse_csv"}
    if args.gemm_csv:
        M, N, K = args.gemm
        c = T.ncu_parse_csv(Path(args.gemm_csv).read_text())
        ops = c["tensor_utc_bf16"]
        out["calibration"] = {"gemm": [M, N, K], "launches": c["launches"], "utchmma_bf16_ops": ops,
                              "flops_2mnk": 2.0 * M * N * K,
                              "flops_per_utc_op": 2.0 * M * N * K / ops if ops else None,
                              "duration_ns": c["duration_ns"]}
    if args.step_csv:
        text = Path(args.step_csv).read_text()
        L, d, a, V, s, mbs, ckpt, drop, nmb = _workload(args.workload)
        B = mbs * nmb
        tot = T.ncu_parse_csv(text)
        classes = {}
        for key, pat in [("gemm", "gemm_sm100"), ("attn_fwd", "fa_fwd"), ("attn_bwd", "fa_bwd")]:
            classes[key] = T.ncu_parse_csv(text, pat)
        spec = T.ModelSpec(L, d, a, V, s)
        model = T.model_flops(spec, B, bool(ckpt))
        exp = executed_tensor_flops(L, d, a, V, s, B, bool(ckpt))
        t = tot["duration_ns"] * 1e-9
        diag = T.diagnose_mbs_mismatch(model / t / 1e12, tot["hw_flops"] / t / 1e12, mbs, mbs)
        out["step"] = {
            "workload": args.workload, "global_batch": B, "launches": tot["launches"],
            "serialised_kernel_time_s": t,
            "hw_flops": tot["hw_flops"], "hw_tensor_flops": tot["tensor_flops"], "hw_simt_flops": tot["simt_flops"],
            "tensor_ops": {k: tot[k] for k in ("tensor_utc_bf16", "tensor_utc_f16", "tensor_hmma_bf16", "tensor_hmma_f16")},
            "dram_bytes": tot["dram_read_bytes"] + tot["dram_write_bytes"],
            "model_flops": model,
            "expected_executed_tensor_flops": exp,
            "hw_tensor_over_expected": tot["tensor_flops"] / exp["total"],
            "model_over_hw": model / tot["hw_flops"],
            "diagnosis": diag,
            "per_class": {k: {"launches": v["launches"], "hw_tensor_flops": v["tensor_flops"],
                              "dram_bytes": v["dram_read_bytes"] + v["dram_write_bytes"],
                              "duration_ns": v["duration_ns"]} for k, v in classes.items()},
        }
        g = classes["gemm"]["tensor_flops"]
        out["step"]["gemm_hw_over_expected"] = g / exp["gemm"]
        out["step"]["attention_hw_over_expected"] = (
            (classes["attn_fwd"]["tensor_flops"] + classes["attn_bwd"]["tensor_flops"])
            / (exp["attention_fwd"] + exp["attention_bwd"]))
    return out


def main():
    ap = argparse.ArgumentParser()
    sub = ap.add_subparsers(dest="cmd", required=True)
    sub.add_parser("metrics")
    g = sub.add_parser("run-gemm")
    g.add_argument("M", type=int)
    g.add_argument("N", type=int)
    g.add_argument("K", type=int)
    r = sub.add_parser("run-step")
    r.add_argument("--workload", default="gpt-1.4b-mbs16")
    an = sub.add_parser("analyze")
    an.add_argument("--gemm-csv")
    an.add_argument("--gemm", type=int, nargs=3, default=[4096, 4096, 4096])
    an.add_argument("--step-csv")
    an.add_argument("--workload", default="gpt-1.4b-mbs16")
    args = ap.parse_args()
    if args.cmd == "metrics":
        print(T.ncu_metric_list())
    elif args.cmd == "run-gemm":
        run_gemm(args.M, args.N, args.K)
    elif args.cmd == "run-step":
        run_step(args.workload)
    else:
        print(json.dumps(analyze(args), indent=1))


if __name__ == "__main__":
    main()
