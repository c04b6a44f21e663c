"""Attention kernel microbenchmark: TFLOP/s of fwd and bwd (causal algorithmic FLOPs)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2312_12705_b200 import _lib as T  # noqa: E402


def run(b=8, s=2048, h=16, hd=128, iters=10, which=("fwd", "bwd")):
    lib = T.load()
    M, d = b * s, h * hd
    st = torch.cuda.current_stream().cuda_stream
    qkv = torch.randn(M, 3 * d, device="cuda").bfloat16()
    out = torch.empty(M, d, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(b * h * s, device="cuda")
    dout = torch.randn(M, d, device="cuda").bfloat16()
    dqkv = torch.empty_like(qkv)
    D = torch.empty(b * h * s, device="cuda")
    dq = torch.empty(M * d, device="cuda")
    fwd = lambda: T.check(lib.tp_flash_attn_fwd(b, s, h, hd, qkv.data_ptr(), out.data_ptr(), lse.data_ptr(), st))
    bwd = lambda: T.check(lib.tp_flash_attn_bwd(b, s, h, hd, qkv.data_ptr(), out.data_ptr(), dout.data_ptr(),
                                                lse.data_ptr(), D.data_ptr(), dq.data_ptr(), dqkv.data_ptr(), st))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for name, fn, fl in [("fwd", fwd, 2.0 * b * h * s * s * hd), ("bwd", bwd, 5.0 * b * h * s * s * hd)]:
        if name not in which:
            continue
        fn()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / iters
        print(f"attn {name} b={b} s={s} h={h} hd={hd}: {ms:.3f} ms  {fl / ms / 1e9:.0f} TFLOP/s", flush=True)


if __name__ == "__main__":
    which = tuple(sys.argv[1:]) or ("fwd", "bwd")
    run(which=which)
    run(b=4, s=2048, h=6, hd=128, which=which)
    run(b=2, s=2048, h=5, hd=160, which=which)
    run(b=1, s=2048, h=40, hd=160, which=which)  # GPT-1T shape, TP4: 40 heads per rank
    run(b=1, s=2048, h=20, hd=160, which=which)  # GPT-1T shape, TP8
    run(b=2, s=256, h=4, hd=64, which=which)
