"""One rank of a multi-GPU parity run (spawned by tests/test_multigpu.py, one process per GPU).

Runs init + one train step through the C-ABI session and dumps, as .npz in the output directory:
the rank's coordinates, its flat-buffer layout (tensor_info of every global tensor), the fp32
master shard before and after the step, the flat fp32 grads after the step (this rank's ZeRO
shard region holds the DP-reduced values) and the loss.
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", required=True)  # json: L d a V s tp pp dp mbs gbs ckpt dropout
    ap.add_argument("--rank", type=int, required=True)
    ap.add_argument("--world", type=int, required=True)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    c = json.loads(a.cfg)
    import oracle_lib as O
    from paper_2312_12705_b200 import _lib as T

    out = Path(a.out)
    idf = out / "nccl_id"
    if a.rank == 0:
        tmp = out / "nccl_id.tmp"
        tmp.write_bytes(T.nccl_unique_id())
        os.replace(tmp, idf)
    t0 = time.time()
    while not idf.exists() or idf.stat().st_size != 128:
        if time.time() - t0 > 120:
            raise RuntimeError("no nccl id")
        time.sleep(0.02)
    nid = idf.read_bytes()
    spec = T.ModelSpec(c["L"], c["d"], c["a"], c["V"], c["s"])
    cfg = T.ParallelConfig(tp=c["tp"], pp=c["pp"], dp=c["dp"], mbs=c["mbs"], gbs=c["gbs"], zero_stage=c.get("zero", 1),
                           checkpoint_activations=c.get("ckpt", 0), interleave_v=c.get("v", 1))
    opts = T.TrainOptions(seed=1234, dropout=c.get("dropout", 0.0), lr=1e-3, weight_decay=0.01)
    if c.get("tp_env"):
        os.environ.update(c["tp_env"])
    sess = T.Session(spec, cfg, opts, rank=a.rank, world=a.world, device=a.rank, nccl_id=nid)
    sess.init_params()
    info = sess.info()
    P, shard = info["flat_params"], info["shard_params"]
    ntens = 2 + 16 * c["L"] + 2
    layout = {}
    for tid in range(ntens):
        ti = sess.tensor_info(tid)
        if ti is not None:
            layout[tid] = ti
    coords = T.rank_coords(a.rank, c["tp"], c["pp"], c["dp"])
    tokens = O.gen_tokens(1234, c["gbs"] * (c["s"] + 1), c["V"]).reshape(c["gbs"], c["s"] + 1)
    nsample = c.get("sample", 0)
    if nsample:
        # wide layouts (dp == 1): per tensor only `nsample` evenly spaced local rows of the fp32
        # master before / after the step and of the gradient (host memory stays small at 1T widths)
        assert c["dp"] == 1
        rows = {tid: np.unique(np.linspace(0, ti["rows"] - 1, min(ti["rows"], nsample)).astype(np.int64))
                for tid, ti in layout.items()}

        def sample(which):
            return {str(tid): np.stack([sess.read_flat(which, ti["offset"] + int(r) * ti["cols"], ti["cols"])
                                        for r in rows[tid]]) for tid, ti in layout.items()}
        m0 = sample(2)
        loss = sess.train_step(tokens)
        g, m1 = sample(1), sample(2)
        extra = {f"{k}_{tid}": v for k, d in (("g", g), ("m0", m0), ("m1", m1)) for tid, v in d.items()}
        extra.update({f"rows_{tid}": r for tid, r in rows.items()})
        np.savez(out / f"rank{a.rank}.npz", tp_mode=np.array(info["tp_mode"]), loss=np.array(loss),
                 coords=np.array(coords), P=np.array(P), shard=np.array(shard), layout=json.dumps(layout),
                 variants=json.dumps(T.variant_counts()), **extra)
    else:
        master0 = sess.read_flat(2, 0, shard)
        loss = sess.train_step(tokens)
        grads = sess.read_flat(1, 0, P)
        master1 = sess.read_flat(2, 0, shard)
        np.savez(out / f"rank{a.rank}.npz", tp_mode=np.array(info["tp_mode"]), grads=grads, master0=master0,
                 master1=master1, loss=np.array(loss), coords=np.array(coords), P=np.array(P),
                 shard=np.array(shard), layout=json.dumps(layout), variants=json.dumps(T.variant_counts()),
                 buckets=np.array(sess.buckets(), dtype=np.int64).reshape(-1, 3))
    sess.barrier()
    sess.close()


if __name__ == "__main__":
    main()
