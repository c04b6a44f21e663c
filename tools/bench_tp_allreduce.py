"""TP allreduce microbenchmark through the session (run under torchrun, one rank per GPU):
NVLS in-switch kernel (grid sweep) vs ncclAllReduce on the [mbs*s, d] bf16 activation buffer,
plus a bit-level check of the NVLS result against an fp32 host sum."""
import argparse
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2312_12705_b200 import _lib as T  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--hidden", type=int, default=6144)
    ap.add_argument("--tokens", type=int, default=2048)
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    idf = Path(f"/tmp/tpar_id_{os.environ['MASTER_PORT']}")
    if rank == 0:
        idf.with_suffix(".tmp").write_bytes(T.nccl_unique_id())
        os.replace(idf.with_suffix(".tmp"), idf)
    while not idf.exists():
        time.sleep(0.05)
    nid = idf.read_bytes()
    spec = T.ModelSpec(world, a.hidden, a.hidden // 128, 128 * world * 8, a.tokens)
    cfg = T.ParallelConfig(tp=world, pp=1, dp=1, mbs=1, gbs=1, zero_stage=1)
    sess = T.Session(spec, cfg, T.TrainOptions(), rank=rank, world=world, device=rank, nccl_id=nid)
    n = a.tokens * a.hidden
    rng = np.random.default_rng(rank)
    x = rng.standard_normal(n, dtype=np.float32)
    xb = (x.view(np.uint32) >> 16).astype(np.uint16)  # truncate to bf16
    out = sess.debug_tp_allreduce(xb, 0)
    ref_parts = [(np.random.default_rng(r).standard_normal(n, dtype=np.float32).view(np.uint32) >> 16 << 16).view(np.float32)
                 for r in range(world)]
    ref = np.sum(ref_parts, axis=0, dtype=np.float64).astype(np.float32)
    got = (out.astype(np.uint32) << 16).view(np.float32)
    rel = np.abs(got - ref) / np.maximum(np.abs(ref), 1e-3)
    res = []
    for mode, ctas in [(1, 0), (0, 16), (0, 32), (0, 64), (0, 96), (0, 148)]:
        ms, nv = sess.bench_tp_allreduce(30, mode, ctas)
        res.append((mode, ctas, ms, nv))
    if rank == 0:
        print(f"tp{world} buffer {n*2/2**20:.1f} MB  nvls={res[-1][3]}  max rel err vs fp32 sum {rel.max():.2e}"
              f" (bf16 half-ulp 3.9e-3)")
        for mode, ctas, ms, nv in res:
            bus = 2 * (world - 1) / world * n * 2 / (ms * 1e-3) / 1e9
            print(f"  {'nccl' if mode else 'nvls'} ctas={ctas:3d}  {ms*1e3:8.1f} us  busbw {bus:7.1f} GB/s")
    sess.barrier()
    sess.close()


if __name__ == "__main__":
    main()
