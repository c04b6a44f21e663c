"""Runs the headline-shape GEMM (2-CTA) and attention fwd/bwd a few times (for ncu captures)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
from paper_2312_12705_b200 import _lib as T  # noqa: E402
import bench_attn  # noqa: E402

M, N, K = 16384, 6144, 2048
A = torch.randn(M, K, device="cuda").bfloat16()
B = torch.randn(N, K, device="cuda").bfloat16()
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    T.gemm_bf16(M, N, K, A.data_ptr(), K, 0, B.data_ptr(), K, 0, C.data_ptr(), N,
                stream=torch.cuda.current_stream().cuda_stream)
bench_attn.run(b=8, s=2048, h=16, hd=128, iters=2)
torch.cuda.synchronize()
print("ok")
