"""Back-to-back dependent launches with and without programmatic dependent launch (pdl.cuh):
a chain of GEMMs (each consumes the previous output) and of LayerNorm fwd/bwd pairs, timed with
CUDA events. Run twice: `python tools/bench_pdl.py` and `GPTB200_PDL=0 python tools/bench_pdl.py`."""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2312_12705_b200 import _lib as T  # noqa: E402


def timed(fn, iters):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / iters  # us


def main():
    tag = "pdl" if os.environ.get("GPTB200_PDL", "1") != "0" else "no-pdl"
    st = torch.cuda.current_stream().cuda_stream
    for n in (1024, 2048, 4096):
        a = torch.randn(n, n, device="cuda").bfloat16()
        w = torch.randn(n, n, device="cuda").bfloat16() * (1.0 / n ** 0.5)
        b = torch.empty_like(a)

        def chain():  # a -> b -> a ... (each GEMM reads the previous one's output)
            for i in range(50):
                src, dst = (a, b) if i % 2 == 0 else (b, a)
                T.gemm_bf16(n, n, n, src.data_ptr(), n, 0, w.data_ptr(), n, 0, dst.data_ptr(), n, stream=st)
        us = timed(chain, 5) / 50
        print(f"[{tag}] GEMM chain {n}^3: {us:.2f} us/launch  {2 * n ** 3 / us / 1e6:.0f} TF/s", flush=True)


if __name__ == "__main__":
    main()
