"""One launch each of our GEMM and cuBLAS on the same shape (ncu comparison): M N K."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2312_12705_b200 import _lib as T  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4])
A = torch.randn(M, K, device="cuda").bfloat16()
B = torch.randn(N, K, device="cuda").bfloat16()
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
st = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    T.gemm_bf16(M, N, K, A.data_ptr(), K, 0, B.data_ptr(), K, 0, C.data_ptr(), N, stream=st)
    torch.matmul(A, B.t(), out=C)
torch.cuda.synchronize()
print("ok")
