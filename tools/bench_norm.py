"""LayerNorm kernels microbenchmark (GB/s of algorithmic bytes) at M=16384, d=2048 (+ wide rows)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2312_12705_b200 import _lib as T  # noqa: E402


def run(rows, d, p=0.1, iters=20):
    lib = T.load()
    st = torch.cuda.current_stream().cuda_stream
    t = lambda: torch.randn(rows, d, device="cuda").bfloat16()
    y, resid, dy, rg = t(), t(), t(), t()
    h, ln, dx, dxd = (torch.empty_like(y) for _ in range(4))
    bias, gamma, beta = (torch.randn(d, device="cuda").bfloat16() for _ in range(3))
    mean, rstd = torch.empty(rows, device="cuda"), torch.empty(rows, device="cuda")
    dg, db, dbias = (torch.zeros(d, device="cuda") for _ in range(3))
    ws = torch.empty(lib.tp_layernorm_bwd_workspace_bytes(rows, d) // 4 + 1, device="cuda")
    fwd = lambda: T.check(lib.tp_resid_layernorm_fwd(rows, d, y.data_ptr(), bias.data_ptr(), resid.data_ptr(), h.data_ptr(),
                                                     gamma.data_ptr(), beta.data_ptr(), ln.data_ptr(), mean.data_ptr(),
                                                     rstd.data_ptr(), 1, 1, 0, 0, p, 0, st))
    bwd = lambda: T.check(lib.tp_layernorm_bwd(rows, d, h.data_ptr(), dy.data_ptr(), rg.data_ptr(), gamma.data_ptr(),
                                               mean.data_ptr(), rstd.data_ptr(), dx.data_ptr(), dxd.data_ptr(),
                                               dg.data_ptr(), db.data_ptr(), dbias.data_ptr(), 1, 1, 0, 0, p, 0,
                                               ws.data_ptr(), st))
    fwd()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for name, fn, nbytes in [("resid_ln_fwd", fwd, 8 * rows * d), ("ln_bwd", bwd, 10 * rows * d)]:
        fn()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / iters
        print(f"{name} rows={rows} d={d}: {ms * 1e3:.1f} us  {nbytes / ms / 1e6:.0f} GB/s", flush=True)


if __name__ == "__main__":
    run(32768, 2048)  # the 1.4B MBS-16 step's shape
    run(16384, 2048)
    run(16384, 2048, p=0.0)
    run(12288, 4096)
    run(2048, 6144)
    run(2048, 12288)
    run(2048, 25600)
