#!/usr/bin/env python
"""Benchmark of the B200-native GPT train step (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--impl b200|reference] [--workload gpt-1.4b]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N

One process per GPU. Default workload = BASELINE config 2: GPT 1.4B (24 layers, hidden 2048,
16 heads, seq 2048, V 51200), bf16 with fp32 master weights/grads, flash attention, MBS 32 per GPU,
data parallel with ZeRO-1 over N GPUs (weak scaling: GBS = 32*N), hidden dropout 0.1, no
activation checkpointing. A step = one full iteration: forward, backward, DP reduce-scatter,
ZeRO-1 Adam, parameter allgather.

`value` = whole-job tokens/s with the token batch already resident in HBM (device time, CUDA
events on the step stream, max over ranks). `e2e` = the same through the public API with host
tokens (H2D copy + step + D2H loss read each step). `--impl reference` times the reference-side
CPU implementation of the path (the oracle port: the reference `trainplan` only models the
step) on the host cores and prints the same metric.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "model TFLOPS/GPU (% of B200 bf16 peak) & tokens/s, GPT fwd+bwd at 1/2/4/8 GPUs"
NOMINAL_PEAK_TFLOPS = 2250.0
FALLBACK_PEAKS = {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "hbm_gbs": 6650.0}

WORKLOADS = {
    # name: (L, d, heads, V, s, mbs, tp, pp, ckpt, dropout, microbatches per DP replica)
    # BASELINE config 2 (headline): 1.4B on 1 GPU, DP = N with ZeRO-1 beyond. Micro-batch 32 is the
    # B200 choice from the sweep below (4: 927, 8: 1020, 16: 1062-1095, 32: 1085-1116 TFLOPS/GPU; the
    # final A/B on one box: 16 -> 1093 / 1096, 32 -> 1113 / 1116; 138 GB of the 180 GB HBM) — the
    # reference's own search tunes mbs the same way.
    "gpt-1.4b": (24, 2048, 16, 51200, 2048, 32, 1, 1, False, 0.1, 1),
    "gpt-1.4b-mbs16": (24, 2048, 16, 51200, 2048, 16, 1, 1, False, 0.1, 1),
    "gpt-1.4b-mbs4": (24, 2048, 16, 51200, 2048, 4, 1, 1, False, 0.1, 1),
    "gpt-1.4b-mbs8": (24, 2048, 16, 51200, 2048, 8, 1, 1, False, 0.1, 1),
    # BASELINE config 1 shape (tiny GPT) — smoke-sized.
    "gpt-tiny": (2, 256, 4, 51200, 128, 1, 1, 1, False, 0.0, 1),
    # BASELINE config 3: 22B shape with TP = 2/4/8 and activation checkpointing, GBS 8. The config does not
    # fix the micro-batch; MBS 4 (m = 2) is the B200 choice from the sweep on one 4-GPU box (TP4: MBS 1 / 2 /
    # 4 / 8 -> 1028 / 1100 / 1172 / 1127 TFLOPS/GPU; larger M per GEMM and per fused SP LayerNorm kernel).
    "gpt-22b-tp2": (48, 6144, 48, 51200, 2048, 4, 2, 1, True, 0.1, 2),
    "gpt-22b-tp4": (48, 6144, 48, 51200, 2048, 4, 4, 1, True, 0.1, 2),
    "gpt-22b-tp8": (48, 6144, 48, 51200, 2048, 4, 8, 1, True, 0.1, 2),
    "gpt-22b-tp4-mbs1": (48, 6144, 48, 51200, 2048, 1, 4, 1, True, 0.1, 8),
    "gpt-22b-tp4-mbs2": (48, 6144, 48, 51200, 2048, 2, 4, 1, True, 0.1, 4),
    "gpt-22b-tp4-mbs8": (48, 6144, 48, 51200, 2048, 8, 4, 1, True, 0.1, 1),
    # BASELINE config 4: 175B-shape layer slice (8 layers) TP4 x PP2 1F1B, m = 16, checkpointing.
    "gpt-175b-slice-tp4pp2": (8, 12288, 96, 51200, 2048, 1, 4, 2, True, 0.1, 16),
    "gpt-175b-slice-tp4": (4, 12288, 96, 51200, 2048, 1, 4, 1, True, 0.1, 8),
    # the same slice's pipeline on 4 GPUs (TP2 x PP2; --interleave 2 for the interleaved 1F1B).
    "gpt-175b-slice-tp2pp2": (8, 12288, 96, 51200, 2048, 1, 2, 2, True, 0.1, 16),
    # BASELINE config 5: 1T-shape layer slice (4 layers, 160 heads, hd 160) TP8 / TP4 x PP2.
    "gpt-1t-slice-tp8": (4, 25600, 160, 51200, 2048, 1, 8, 1, True, 0.1, 8),
    "gpt-1t-slice-tp4pp2": (4, 25600, 160, 51200, 2048, 1, 4, 2, True, 0.1, 8),
    # the same 4-layer 1T slice on 4 GPUs (TP4; ~140 GB/GPU) for single-box measurements
    "gpt-1t-slice-tp4": (4, 25600, 160, 51200, 2048, 1, 4, 1, True, 0.1, 8),
}


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {k: float(d[k]) for k in FALLBACK_PEAKS}, "measured (MEASURED_PEAKS.json)"
    return dict(FALLBACK_PEAKS), "fallback (B200_PROFILING.md)"


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def share_nccl_id(rank: int, world: int) -> bytes | None:
    if world == 1:
        return None
    from paper_2312_12705_b200 import _lib as T
    # Unique per launch: all ranks of one torchrun launch share the agent process as parent
    # (TORCHELASTIC_RUN_ID is constant under static rendezvous, so back-to-back launches on one
    # box would otherwise read a stale id).
    tag = f"{os.environ.get('MASTER_PORT', '0')}_{os.getppid()}_{os.environ.get('TORCHELASTIC_RESTART_COUNT', '0')}"
    path = Path(tempfile.gettempdir()) / f"gptb200_ncclid_{tag}"
    if rank == 0:
        nid = T.nccl_unique_id()
        tmp = path.with_suffix(".tmp")
        tmp.write_bytes(nid)
        os.replace(tmp, path)
        return nid
    t0 = time.time()
    while not path.exists() or path.stat().st_size != 128:
        if time.time() - t0 > 300:
            raise RuntimeError("timed out waiting for the NCCL id from rank 0")
        time.sleep(0.05)
    return path.read_bytes()


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, gpus: list[int]):
        self.file = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-i", ",".join(map(str, gpus)), "-lms", "200"],
                                         stdout=self.file, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.file.flush()
        rows = [r.split(",") for r in Path(self.file.name).read_text().strip().splitlines() if r.strip()]
        os.unlink(self.file.name)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                smax.append(float(r[2]))
                for n, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(n)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def model_flops(L, d, a, V, s, batch, ckpt) -> float:
    """trainplan::model_flops_per_iteration (proj/src/arch.cpp:64-92) in exact Python integers:
    24 c B s L d^2 (1 + s/6d + V/16Ld) = c B s d (48 L d + 8 L s + 3 V) / 2, c = 4 with activation
    checkpointing, else 3. (Pure Python so the reference arm loads nothing from this repo's
    library; tests/test_bench.py checks it against the C-ABI and the reference's golden.)"""
    c = 4 if ckpt else 3
    return float(c * batch * s * d * (48 * L * d + 8 * L * s + 3 * V)) / 2.0


def cpu_layer_sample(L, d, a, V, s, threads):
    """Times the CPU oracle (port of the step) on one decoder layer fwd+bwd over one sequence;
    returns (seconds, layer model-FLOPs, full-model tokens/s EXTRAPOLATED at the measured FLOP rate,
    model TFLOPS)."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib as O
    lib = O.load()
    m = O.model(1, d, a, V, s)
    import ctypes
    secs = lib.orc_time_layer(ctypes.byref(m), 1, threads)
    # one layer, one sequence, c = 3: 24*3*s*d^2*(1 + s/(6d))  (arch.cpp:64-92 restricted to a layer)
    layer_flops = 72.0 * s * d * d * (1 + s / (6.0 * d))
    rate = layer_flops / secs
    per_token_model = model_flops(L, d, a, V, s, 1, False) / s
    return secs, layer_flops, rate / per_token_model, rate / 1e12


def cpu_config1_step(threads):
    """One REAL full train step of BASELINE config 1 (tiny GPT: 2 layers, hidden 256, 4 heads,
    seq 128, V 51200, GBS 8) on the CPU oracle: 8 sequences fwd+bwd + Adam over every parameter —
    the unsharded arithmetic of the TP2 x PP2 x DP2 layout. Returns (seconds, tokens/s)."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib as O
    os.environ.setdefault("OMP_NUM_THREADS", str(threads))
    L, d, a, V, s, gbs = 2, 256, 4, 51200, 128, 8
    m, o = O.model(L, d, a, V, s), O.opts(seed=1234, lr=1e-4)
    params = O.init_params(m, 1234)
    tokens = O.gen_tokens(1234, gbs * (s + 1), V).reshape(gbs, s + 1)
    mom, var = np.zeros_like(params), np.zeros_like(params)
    t0 = time.perf_counter()
    grads = np.zeros_like(params)
    for i in range(gbs):
        O.fwd_bwd(m, o, params, tokens[i:i + 1], sample0=i, step=1, loss_scale=1.0 / (gbs * s), grads=grads)
    import ctypes
    O.load().orc_adam(params.size, params, mom, var, grads, 1, ctypes.byref(o))
    secs = time.perf_counter() - t0
    return secs, gbs * s / secs


def run_reference(args, rank, world):
    """--impl reference: the reference-side CPU implementation of the path on the host cores."""
    if rank != 0:
        return 0
    L, d, a, V, s, mbs, tp, pp, ckpt, drop, nmb = WORKLOADS[args.workload]
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_layer_sample(L, d, a, V, s, threads)
    vals, secs_all = [], []
    for _ in range(args.steps):
        secs, lf, tok_s, tflops = cpu_layer_sample(L, d, a, V, s, threads)
        vals.append(tok_s)
        secs_all.append(secs)
    v = statistics.median(vals)
    gbs = mbs * nmb * max(args.gpus // (tp * pp), 1)
    c1_secs, c1_tok = cpu_config1_step(threads)
    sample_ms = 1e3 * statistics.median(secs_all)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        # a reference-arm step is a bounded sample of the workload (one layer, one sequence): its
        # measured wall time is the step time; `value` is the workload's tokens/s extrapolated from it
        "ms_per_step": sample_ms, "value_extrapolated": True,
        "full_step_ms_extrapolated": 1e3 * gbs * s / v,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_config(args, world),
        "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": threads, "kind": "port", "extrapolated": True,
                         "sample": f"one decoder layer fwd+bwd (d={d}, s={s}, 1 sequence) of the CPU oracle port "
                                   f"(oracle/gpt_oracle.c; the reference trainplan only models the step), "
                                   f"{sample_ms / 1e3:.2f}s/sample, extrapolated to the full {L}-layer model at "
                                   f"the measured FLOP rate",
                         "config1_full_step": {"seconds": c1_secs, "tokens_per_s": c1_tok, "extrapolated": False,
                                               "what": "BASELINE config 1 (L2 d256 a4 V51200 s128, GBS 8): one "
                                                       "complete fwd+bwd+Adam step of the oracle"}},
        "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "native_libs": loaded_native_libs(),
    }
    print(json.dumps(line), flush=True)
    return 0


def loaded_native_libs():
    """Shared objects of this repo mapped into the process (the reference arm must show only the
    oracle's)."""
    try:
        maps = Path("/proc/self/maps").read_text().splitlines()
    except OSError:
        return None
    return sorted({ln.split()[-1] for ln in maps if str(ROOT) in ln and ln.endswith(".so")})


def workload_config(args, world):
    L, d, a, V, s, mbs, tp, pp, ckpt, drop, nmb = WORKLOADS[args.workload]
    dp = max(world // (tp * pp), 1)
    return {"workload": f"{args.workload}: GPT L{L} d{d} a{a} V{V} s{s}, fwd+bwd+ZeRO-1 Adam step",
            "global_batch": mbs * nmb * dp, "seq_len": s, "micro_batch": mbs, "microbatches": nmb,
            "parallelism": f"tp{tp}.pp{pp}.dp{dp}" + (f".v{args.interleave}" if args.interleave > 1 else ""),
            "zero_stage": 1, "activation_checkpointing": ckpt, "hidden_dropout": drop, "attention_dropout": 0.0,
            "flash_attention": True, "grad_accum_dtype": "fp32",
            "l2": "per-step working set (tens of GB) far larger than the 126 MB L2; no flush needed"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="gpt-1.4b", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-profile", action="store_true")
    ap.add_argument("--interleave", type=int, default=1, help="model chunks per pipeline stage (interleaved 1F1B)")
    args = ap.parse_args()
    rank, local, world = env_rank()
    if world != args.gpus:
        world = max(world, 1)
    if args.impl == "reference":
        return run_reference(args, rank, world)

    from paper_2312_12705_b200 import _lib as T
    from paper_2312_12705_b200.build import LIB, build
    if not LIB.exists():
        build()
    L, d, a, V, s, mbs, tp, pp, ckpt, drop, nmb = WORKLOADS[args.workload]
    if world % (tp * pp) != 0:
        raise SystemExit(f"{args.workload} needs a multiple of tp*pp = {tp * pp} GPUs, got {world}")
    dp = world // (tp * pp)
    gbs = mbs * nmb * dp
    spec = T.ModelSpec(L, d, a, V, s)
    cfg = T.ParallelConfig(tp=tp, pp=pp, dp=dp, mbs=mbs, gbs=gbs, zero_stage=1, checkpoint_activations=int(ckpt),
                           interleave_v=args.interleave)
    opts = T.TrainOptions(seed=1234, dropout=drop, lr=1e-4, weight_decay=0.0)
    nid = share_nccl_id(rank, world)
    sess = T.Session(spec, cfg, opts, rank=rank, world=world, device=local, nccl_id=nid)
    sess.barrier()  # every rank has joined the communicator: the id file is no longer needed
    if world > 1 and rank == 0:
        for f in Path(tempfile.gettempdir()).glob(f"gptb200_ncclid_{os.environ.get('MASTER_PORT', '0')}_{os.getppid()}_*"):
            f.unlink(missing_ok=True)
    sess.init_params()
    tokens = np.random.default_rng(1234).integers(0, V, size=(gbs, s + 1), dtype=np.int32)
    sess.upload_tokens(tokens)
    if args.warmup:
        sess.time_steps(args.warmup)
    sess.barrier()
    clocks = ClockSampler(list(range(world))) if rank == 0 else None
    ms, _ = sess.time_steps(args.steps, profile=False)
    ms_max = sess.allreduce_max(ms)
    # per-step device times of the same timed region (events between steps), max over ranks per step
    per_step = [sess.allreduce_max(t) for t in sess.step_times(args.steps)]
    sess.barrier()
    clk = clocks.stop() if clocks else None
    info = sess.info()
    # second timed region over the same K steps with every launch bracketed by CUDA events on the
    # step stream: per-kernel-class durations for the roofline (kept out of `value`)
    kt, ms_prof = None, None
    if not args.no_profile:
        ms_prof, kt = sess.time_steps(args.steps, profile=True)
        sess.barrier()
    # e2e through the public API with host tokens (H2D + step + D2H loss each step)
    sess.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        loss = sess.train_step(tokens)
    sess.barrier()
    e2e_s = sess.allreduce_max(time.perf_counter() - t0)
    step_s = ms_max / 1e3 / args.steps
    flops_iter = model_flops(L, d, a, V, s, gbs, ckpt)
    tflops_gpu = flops_iter / step_s / world / 1e12
    tok_s = gbs * s / step_s
    e2e_tok_s = gbs * s * args.steps / e2e_s
    peaks, peak_src = load_peaks()
    if rank != 0:
        sess.close()
        return 0
    line = {
        "metric": METRIC, "value": tok_s, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (uniform random tokens; counter-based N(0,0.02) init)",
        "config": workload_config(args, world),
        "model_tflops_per_gpu": tflops_gpu,
        "peak_fraction": {"of_nominal_2250": tflops_gpu / NOMINAL_PEAK_TFLOPS,
                          "of_measured_burst": tflops_gpu / peaks["bf16_tflops"],
                          "of_measured_sustained": tflops_gpu / peaks["bf16_tflops_sustained"],
                          "peaks_source": peak_src},
        "tokens_per_s_per_gpu": tok_s / world,
        # spread of the K timed steps: per-step device ms, max over ranks per step
        "step_ms": {"median": float(np.median(per_step)), "p10": float(np.percentile(per_step, 10)),
                    "p90": float(np.percentile(per_step, 90)), "min": min(per_step), "max": max(per_step)},
        "loss": loss,
        "e2e": {"value": e2e_tok_s, "unit": "tokens/s", "h2d_bytes_per_step": int(tokens.nbytes),
                "d2h_bytes_per_step": 4},
        "gpu_launches": int(info["launches"]) * args.steps,
        "clocks": clk,
    }
    if kt:
        g = kt["gemm"]
        gemm_tf = g["flops"] / (g["ms"] / 1e3) / 1e12 if g["ms"] else 0.0
        line["roofline"] = {"kernel": "tcgen05 GEMM (all GEMM launches of the step)", "bound": "tensor",
                            "achieved": gemm_tf, "peak": peaks["bf16_tflops_sustained"], "unit": "TFLOP/s",
                            "frac": gemm_tf / peaks["bf16_tflops_sustained"],
                            "traffic": gemm_traffic(args.workload),
                            "traffic_algorithmic": gemm_traffic(args.workload, "algorithmic_bytes"),
                            "traffic_kernel": gemm_traffic(args.workload, "kernel"),
                            "peak_source": peak_src + ", sustained bf16 (kernel timed inside a long step)",
                            "gemm_share_of_step": g["ms"] / ms_prof if ms_prof else None,
                            "algorithmic_flops_per_launch": g["flops"] / max(g["launches"], 1)}
        # the other kernel families against their own roofline (tensor for attention, HBM for norms)
        classes = {"attn_fwd": ("tensor", "bf16_tflops_sustained", "TFLOP/s"),
                   "attn_bwd": ("tensor", "bf16_tflops_sustained", "TFLOP/s"),
                   "norm": ("hbm", "hbm_gbs", "GB/s")}
        line["roofline_by_class"] = {}
        for k, (bound, pk, unit) in classes.items():
            v = kt[k]
            if not v["ms"]:
                continue
            ach = (v["flops"] / (v["ms"] / 1e3) / 1e12) if bound == "tensor" else (v["bytes"] / (v["ms"] / 1e3) / 1e9)
            line["roofline_by_class"][k] = {"bound": bound, "achieved": ach, "peak": peaks[pk], "unit": unit,
                                            "frac": ach / peaks[pk], "share_of_step": v["ms"] / ms_prof}
        line["kernels"] = {k: {"ms_per_step": v["ms"] / args.steps, "share": v["ms"] / ms_prof if ms_prof else None,
                               "launches_per_step": v["launches"] / args.steps,
                               **({"tflops": v["flops"] / (v["ms"] / 1e3) / 1e12} if v["flops"] and v["ms"] else {}),
                               **({"gbs": v["bytes"] / (v["ms"] / 1e3) / 1e9} if v["bytes"] and v["ms"] else {})}
                           for k, v in kt.items()}
    if world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        secs, lf, cpu_tok, cpu_tf = cpu_layer_sample(L, d, a, V, s, threads)
        line["cpu_baseline"] = {"value": cpu_tok, "unit": "tokens/s", "cores": threads, "kind": "port",
                                "model_tflops": cpu_tf,
                                "sample": f"one decoder layer fwd+bwd (d={d}, s={s}, 1 sequence) of the CPU oracle "
                                          f"port in {secs:.2f}s; tokens/s extrapolated to the full {L}-layer model"}
    sess.close()
    print(json.dumps(line), flush=True)
    return 0


def gemm_traffic(workload, key="bytes_per_launch"):
    """Per-launch DRAM bytes (or the algorithmic bytes, key="algorithmic_bytes") of the representative
    GEMM launch of THIS workload in the committed ncu capture (profiles/gemm_traffic.json, one
    entry per workload), else None."""
    p = ROOT / "profiles" / "gemm_traffic.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
        except ValueError:
            return None
        entry = d.get("workloads", {}).get(workload)
        if entry is None and d.get("workload") == workload:
            entry = d
        return entry.get(key) if entry else None
    return None


if __name__ == "__main__":
    sys.exit(main())
