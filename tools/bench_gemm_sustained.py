"""Sustained (power-capped) GEMM throughput: ~3 s of back-to-back launches of one shape, ours vs
cuBLAS, with the SM clock / power sampled by nvidia-smi during each run."""
import subprocess
import sys
import threading
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2312_12705_b200 import _lib as T  # noqa: E402


def sample(stop, out):
    while not stop.is_set():
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits", "-i", "0"],
                           capture_output=True, text=True).stdout.strip().split(",")
        try:
            out.append((float(r[0]), float(r[1])))
        except (ValueError, IndexError):
            pass
        time.sleep(0.1)


def run(name, fn, flops, secs=3.0):
    fn()
    torch.cuda.synchronize()
    t0 = time.time()
    n = 0
    while time.time() - t0 < 0.5:  # warm to the power-capped steady state
        fn()
        n += 1
    torch.cuda.synchronize()
    stop, smp = threading.Event(), []
    th = threading.Thread(target=sample, args=(stop, smp))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = max(int(n * secs / 0.5), 10)
    th.start()
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = e0.elapsed_time(e1) / iters
    clk = sorted(c for c, _ in smp)[len(smp) // 2] if smp else 0
    pw = sorted(p for _, p in smp)[len(smp) // 2] if smp else 0
    tf = flops / ms / 1e9
    print(f"{name:40s} {ms*1e3:8.1f} us  {tf:7.1f} TF/s  sm {clk:6.0f} MHz  power {pw:6.1f} W  "
          f"TF/s per GHz {tf / (clk / 1e3) if clk else 0:7.1f}  TFLOP/J {tf / pw if pw else 0:.2f}", flush=True)


import os  # noqa: E402


def main():
    lib = T.load()
    force = int(os.environ.get("FORCE_CG", "0"))
    T.check(lib.tp_gemm_force_cta_group(force))
    st = torch.cuda.current_stream().cuda_stream
    shapes = [(8192, 8192, 8192, 0, 0, 0), (16384, 8192, 2048, 0, 0, 0), (16384, 8192, 2048, 0, 0, 1),
              (8192, 2048, 16384, 1, 1, 2)]
    if os.environ.get("SHAPES") == "square":
        shapes = shapes[:2]
    if os.environ.get("SHAPES") == "mbs16":  # 1.4B step shapes at M = 32768 tokens
        shapes = [(32768, 6144, 2048, 0, 0, 0), (32768, 8192, 2048, 0, 0, 1), (32768, 2048, 2048, 0, 1, 0),
                  (32768, 2048, 8192, 0, 1, 0), (32768, 8192, 2048, 0, 1, 3)]
    if os.environ.get("SHAPES") == "mbs32":  # 1.4B step shapes at M = 65536 tokens (the bench default)
        shapes = [(65536, 6144, 2048, 0, 0, 0), (65536, 8192, 2048, 0, 0, 1), (65536, 2048, 2048, 0, 1, 0),
                  (65536, 2048, 8192, 0, 1, 0), (2048, 8192, 65536, 1, 1, 2),
                  (8192, 2048, 65536, 1, 1, 2)]
    if os.environ.get("SHAPES") == "longk":
        shapes = [(8192, 8192, 8192, 0, 0, 0), (16384, 2048, 8192, 0, 1, 0), (8192, 2048, 16384, 1, 1, 2)]
    ldaux = int(os.environ.get("LDAUX", "0"))  # experiment hook (no effect in the product build)
    for (M, N, K, a_mn, b_mn, epi) in shapes:
        A = torch.randn((K, M) if a_mn else (M, K), device="cuda").bfloat16()
        B = torch.randn((K, N) if b_mn else (N, K), device="cuda").bfloat16()
        C = torch.empty(M, N, device="cuda", dtype=torch.float32 if epi == 2 else torch.bfloat16)
        C2 = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        bias = torch.zeros(N, device="cuda", dtype=torch.bfloat16)
        fl = 2.0 * M * N * K
        ours = lambda: T.gemm_bf16(M, N, K, A.data_ptr(), M if a_mn else K, a_mn, B.data_ptr(), N if b_mn else K, b_mn,
                                   C.data_ptr(), N, epi=epi, bias=bias.data_ptr() if epi == 1 else None,
                                   C2=C2.data_ptr() if epi == 1 else None, ldaux=ldaux,
                                   accumulate=1 if epi == 2 else 0, stream=st)
        At = A.t() if a_mn else A
        Bt = B if b_mn else B.t()
        out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        cub = lambda: torch.matmul(At, Bt, out=out)
        run(f"ours   M{M} N{N} K{K} mn{a_mn}{b_mn} epi{epi}", ours, fl)
        run(f"cublas M{M} N{N} K{K} mn{a_mn}{b_mn}", cub, fl)


if __name__ == "__main__":
    main()
