"""Attention fwd/bwd of this repo vs cuDNN SDPA (torch) and FA2 (flash_attn) at the step shapes.

Same algorithmic causal FLOPs for every implementation (fwd 2·b·h·s²·hd, bwd 5·b·h·s²·hd); CUDA-event
timing after warm-up. cuDNN / FA2 are library baselines for the judgement of the kernel, not on the
product path.
"""
import sys
from pathlib import Path

import torch
import torch.nn.functional as F

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2312_12705_b200 import _lib as T  # noqa: E402


def timeit(fn, iters=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def ours(b, s, h, hd):
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
    fwd()
    return timeit(fwd), timeit(bwd)


def cudnn(b, s, h, hd):
    q, k, v = (torch.randn(b, h, s, hd, device="cuda", dtype=torch.bfloat16, requires_grad=True) for _ in range(3))
    do = torch.randn(b, h, s, hd, device="cuda", dtype=torch.bfloat16)
    from torch.nn.attention import SDPBackend, sdpa_kernel
    with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
        o = F.scaled_dot_product_attention(q, k, v, is_causal=True)
        tf = timeit(lambda: F.scaled_dot_product_attention(q, k, v, is_causal=True))
        tb = timeit(lambda: torch.autograd.grad(o, (q, k, v), do, retain_graph=True))
    return tf, tb


def fa2(b, s, h, hd):
    from flash_attn import flash_attn_func
    q, k, v = (torch.randn(b, s, h, hd, device="cuda", dtype=torch.bfloat16, requires_grad=True) for _ in range(3))
    do = torch.randn(b, s, h, hd, device="cuda", dtype=torch.bfloat16)
    o = flash_attn_func(q, k, v, causal=True)
    tf = timeit(lambda: flash_attn_func(q, k, v, causal=True))
    tb = timeit(lambda: torch.autograd.grad(o, (q, k, v), do, retain_graph=True))
    return tf, tb


if __name__ == "__main__":
    shapes = [(32, 2048, 16, 128), (8, 2048, 16, 128), (1, 2048, 12, 128), (1, 2048, 40, 160)]
    for (b, s, h, hd) in shapes:
        ff, fb = 2.0 * b * h * s * s * hd, 5.0 * b * h * s * s * hd
        for name, fn in [("ours", ours), ("cudnn", cudnn), ("fa2", fa2)]:
            try:
                tf, tb = fn(b, s, h, hd)
                print(f"{name:6s} b={b} s={s} h={h} hd={hd}: fwd {tf:.3f} ms {ff / tf / 1e9:.0f} TF/s | "
                      f"bwd {tb:.3f} ms {fb / tb / 1e9:.0f} TF/s", flush=True)
            except Exception as e:  # noqa: BLE001
                print(f"{name:6s} b={b} s={s} h={h} hd={hd}: unavailable ({type(e).__name__}: {str(e)[:120]})", flush=True)
            torch.cuda.empty_cache()
