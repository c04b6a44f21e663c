"""Run one GEMM shape a few times (for ncu captures): python tools/run_gemm_shape.py M N K a_mn b_mn epi [iters]."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2312_12705_b200 import _lib as T  # noqa: E402

M, N, K, a_mn, b_mn, epi = (int(x) for x in sys.argv[1:7])
iters = int(sys.argv[7]) if len(sys.argv) > 7 else 3
A = torch.randn((K, M) if a_mn else (M, K), device="cuda").bfloat16()
B = torch.randn((K, N) if b_mn else (N, K), device="cuda").bfloat16()
C = torch.zeros(M, N, device="cuda", dtype=torch.float32 if epi == 2 else torch.bfloat16)
C2 = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16) if epi == 1 else None
bias = torch.zeros(N, device="cuda", dtype=torch.bfloat16) if epi == 1 else None
st = torch.cuda.current_stream().cuda_stream
for _ in range(iters):
    T.gemm_bf16(M, N, K, A.data_ptr(), M if a_mn else K, a_mn, B.data_ptr(), N if b_mn else K, b_mn, C.data_ptr(), N,
                epi=epi, accumulate=1 if epi == 2 else 0, stream=st,
                **({"C2": C2.data_ptr(), "bias": bias.data_ptr()} if epi == 1 else {}))
torch.cuda.synchronize()
print("ok")
