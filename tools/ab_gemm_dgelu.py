"""A/B timing of the dGeLU-epilogue dgrad GEMM (fc2 dgrad of the 1.4B MBS-32 step: M=65536 N=8192
K=2048, B MN-major, aux = pre-activation) for the library selected by GPTB200_LIB."""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2312_12705_b200 import _lib as T  # noqa: E402

M, N, K = 65536, 8192, 2048
A = torch.randn(M, K, device="cuda").bfloat16()
B = (torch.randn(K, N, device="cuda") * 0.02).bfloat16()  # W2 [d][4d]: B(n,k) = W[k][n]
U = torch.randn(M, N, device="cuda").bfloat16()
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
st = torch.cuda.current_stream().cuda_stream
f = lambda: T.gemm_bf16(M, N, K, A.data_ptr(), K, 0, B.data_ptr(), N, 1, C.data_ptr(), N, epi=3,  # noqa: E731
                        aux=U.data_ptr(), ldaux=N, stream=st)
for _ in range(3):
    f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    f()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
ref = (A[:256].float() @ B.float()) * 0  # shape check only
print(f"{os.environ.get('GPTB200_LIB', 'current')}: dgelu GEMM {ms * 1e3:.1f} us  {2 * M * N * K / ms / 1e9:.0f} TF/s "
      f"checksum {C[:64].float().abs().mean().item():.6f}", flush=True)
