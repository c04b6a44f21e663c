"""Sequence-parallel LayerNorm kernels (NVLS reduce-scatter + LN + allgather) in isolation, under
torchrun (one rank per GPU): python -m torch.distributed.run --nproc-per-node 4 tools/bench_sp.py --hidden 6144
Per kernel: device us, and the NVLink bytes per rank (in: this rank's reduced rows + the other
ranks' LN rows; out: serving the peers' reductions of this rank's partials + this rank's rows)."""
import argparse
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2312_12705_b200 import _lib as T  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--hidden", type=int, default=6144)
    ap.add_argument("--heads", type=int, default=48)
    ap.add_argument("--tokens", type=int, default=2048)
    ap.add_argument("--iters", type=int, default=50)
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    idf = Path(f"/tmp/bsp_id_{os.environ['MASTER_PORT']}")
    if rank == 0:
        idf.with_suffix(".tmp").write_bytes(T.nccl_unique_id())
        os.replace(idf.with_suffix(".tmp"), idf)
    while not idf.exists():
        time.sleep(0.05)
    spec = T.ModelSpec(1, a.hidden, a.heads, 128 * world * 4, a.tokens)
    cfg = T.ParallelConfig(tp=world, pp=1, dp=1, mbs=1, gbs=1, zero_stage=1)
    sess = T.Session(spec, cfg, T.TrainOptions(dropout=0.1), rank=rank, world=world, device=rank,
                     nccl_id=idf.read_bytes())
    sess.init_params()
    M, d = a.tokens, a.hidden
    rows = M // world
    for mode, name in ((0, "sp_ln_fwd"), (1, "sp_ln_bwd")):
        ms = sess.allreduce_max(sess.bench_sp(a.iters, mode))
        # NVLink in per rank: own reduced rows (rows*d*2) + peers' allgathered rows ((world-1)*rows*d*2)
        nv_in = rows * d * 2 * world
        if rank == 0:
            print(f"{name:10s} d={d} M={M} tp={world}: {ms * 1e3:8.1f} us   NVLink in/rank {nv_in / 1e6:6.1f} MB "
                  f"-> {nv_in / (ms / 1e3) / 1e9:6.0f} GB/s", flush=True)
    ms, nv = sess.bench_tp_allreduce(a.iters, 0, 0)
    ms = sess.allreduce_max(ms)
    if rank == 0:
        print(f"nvls_allreduce [M,d] bf16 ({M * d * 2 / 1e6:.1f} MB): {ms * 1e3:8.1f} us", flush=True)
    sess.barrier()
    sess.close()
    if rank == 0:
        idf.unlink(missing_ok=True)


if __name__ == "__main__":
    main()
