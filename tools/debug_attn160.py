import ctypes, sys
from pathlib import Path
import torch
lib = ctypes.CDLL(sys.argv[1])
b, s, h, hd = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
M, d = b * s, h * hd
qkv = torch.randn(M, 3 * d, device="cuda").bfloat16()
out = torch.empty(M, d, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(b * h * s, device="cuda")
r = lib.tp_flash_attn_fwd(b, s, h, hd, ctypes.c_void_p(qkv.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                          ctypes.c_void_p(lse.data_ptr()), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
print("rc", r, "ok", out.float().abs().mean().item())
