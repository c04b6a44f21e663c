"""Probe: NCCL allreduce / reduce-scatter / allgather busbw on the TP group at the TP message sizes
(bf16 [mbs*s, d]); run under torchrun. Prints one line per (op, size)."""
import os
import torch
import torch.distributed as dist

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl")
for n_mb in (2048 * 2048 * 2 / 2**20, 2048 * 6144 * 2 / 2**20, 2048 * 12288 * 2 / 2**20):
    n = int(n_mb * 2**20 / 2)
    x = torch.randn(n, device="cuda", dtype=torch.bfloat16)
    out = torch.empty(n // world, device="cuda", dtype=torch.bfloat16)
    for op in ("allreduce", "reduce_scatter", "allgather"):
        def run():
            if op == "allreduce":
                dist.all_reduce(x)
            elif op == "reduce_scatter":
                dist.reduce_scatter_tensor(out, x)
            else:
                dist.all_gather_into_tensor(x, out)
        for _ in range(5):
            run()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            run()
        b.record()
        torch.cuda.synchronize()
        t = a.elapsed_time(b) / 20 / 1e3
        factor = 2 * (world - 1) / world if op == "allreduce" else (world - 1) / world
        if rank == 0:
            print(f"{op:15s} {n_mb:7.1f} MB  {t*1e6:8.1f} us  algbw {n*2/t/1e9:7.1f} GB/s  busbw {n*2*factor/t/1e9:7.1f} GB/s", flush=True)
dist.destroy_process_group()
