"""Host-side logic of the multi-rank path, on CPU.

1. The 1F1B executor (Stage::step) pairs the send of op i's output with the receive of op i+1's
   input in one ncclGroup (Megatron's send_forward_recv_backward pattern). A rendezvous simulation
   over the reference-identical per-device orders proves every stage finishes (no deadlock) and that
   every activation / gradient message is received exactly once by the right stage.
2. world_size-2 gloo run: each process derives its rank coordinates, pipeline order and ZeRO-1
   shard range through the C-ABI; rank 0 checks the union is consistent.
"""
import os
import socket
import sys
from pathlib import Path

import pytest

from paper_2312_12705_b200 import _lib as T

ROOT = Path(__file__).resolve().parents[1]


def executor_groups(p, m, stage):
    """The communication groups Stage::step() issues on `stage`, in order."""
    ops = T.pipeline_order(1, p, m, 1, stage)
    groups, pending = [], None
    for bwd, mb, _ in ops:
        recv = None
        if not bwd and stage > 0:
            recv = ("recv", stage - 1, ("act", mb))
        elif bwd and stage < p - 1:
            recv = ("recv", stage + 1, ("grad", mb))
        g = [x for x in (pending, recv) if x]
        if g:
            groups.append(g)
        pending = None
        if not bwd and stage < p - 1:
            pending = ("send", stage + 1, ("act", mb))
        elif bwd and stage > 0:
            pending = ("send", stage - 1, ("grad", mb))
    if pending:
        groups.append([pending])
    return groups


def simulate(p, m, groups_fn=None):
    """NCCL semantics: a stage posts its current group; each send/recv in it completes once the
    peer has posted the matching op (ops of one group progress independently); the stage moves on
    when every op of its group has completed."""
    groups_fn = groups_fn or executor_groups
    seq = [groups_fn(p, m, s) for s in range(p)]
    pos = [0] * p
    done = [set() for _ in range(p)]  # completed op indices of the current group
    delivered = []
    while not all(pos[s] == len(seq[s]) for s in range(p)):
        progressed = False
        for s in range(p):
            if pos[s] == len(seq[s]):
                continue
            for i, (kind, peer, tag) in enumerate(seq[s][pos[s]]):
                if i in done[s] or pos[peer] == len(seq[peer]):
                    continue
                want = ("recv" if kind == "send" else "send", s, tag)
                cur = seq[peer][pos[peer]]
                if want in cur:
                    j = cur.index(want)
                    done[s].add(i)
                    done[peer].add(j)
                    if kind == "send":
                        delivered.append((s, peer, tag))
                    else:
                        delivered.append((peer, s, tag))
                    progressed = True
        for s in range(p):
            if pos[s] < len(seq[s]) and len(done[s]) == len(seq[s][pos[s]]):
                pos[s] += 1
                done[s] = set()
                progressed = True
        if not progressed:
            raise AssertionError(f"deadlock p={p} m={m} at {pos}")
    return delivered


def test_unpaired_sends_would_deadlock(native_lib):
    """Sanity check of the simulator: issuing every send/recv alone (no pairing) deadlocks 1F1B."""
    def unpaired(p, m, stage):
        return [[op] for grp in executor_groups(p, m, stage) for op in sorted(grp, key=lambda o: o[0] == "recv")]

    with pytest.raises(AssertionError):
        simulate(2, 4, unpaired)


@pytest.mark.parametrize("p", [2, 3, 4, 8])
@pytest.mark.parametrize("m", [1, 2, 3, 4, 7, 8, 16])
def test_1f1b_executor_pairing_is_deadlock_free(native_lib, p, m):
    delivered = simulate(p, m)
    acts = sorted((s, mb) for s, peer, (k, mb) in delivered if k == "act")
    grads = sorted((s, mb) for s, peer, (k, mb) in delivered if k == "grad")
    assert acts == sorted((s, mb) for s in range(p - 1) for mb in range(m))
    assert grads == sorted((s, mb) for s in range(1, p) for mb in range(m))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, result_path):
    sys.path.insert(0, str(ROOT))
    import torch.distributed as dist

    from paper_2312_12705_b200 import _lib as TL
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    tp, pp, dp = 1, 2, 1  # the two ranks are the two pipeline stages
    coords = TL.rank_coords(rank, tp, pp, dp)
    order = TL.pipeline_order(1, pp, 4, 1, coords[1])
    P = 1000 * 64
    shard = (rank * P // world, (rank + 1) * P // world)
    mine = {"rank": rank, "coords": coords, "order": order, "shard": shard,
            "groups": executor_groups(pp, 4, coords[1])}
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    if rank == 0:
        import json
        Path(result_path).write_text(json.dumps(gathered))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_layout(tmp_path, native_lib):
    pytest.importorskip("torch")
    import json

    import torch.multiprocessing as mp
    port = _free_port()
    out = tmp_path / "gathered.json"
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    mp.start_processes(_gloo_worker, args=(2, port, str(out)), nprocs=2, join=True, start_method="spawn")
    g = json.loads(out.read_text())
    assert sorted(tuple(x["coords"]) for x in g) == [(0, 0, 0), (0, 1, 0)]
    # every send posted by one stage is a receive posted by the other, same tag, same order
    sends0 = [op for grp in g[0]["groups"] for op in grp if op[0] == "send"]
    recvs1 = [op for grp in g[1]["groups"] for op in grp if op[0] == "recv"]
    assert [tuple(x[2]) for x in sends0] == [tuple(x[2]) for x in recvs1]
    sends1 = [op for grp in g[1]["groups"] for op in grp if op[0] == "send"]
    recvs0 = [op for grp in g[0]["groups"] for op in grp if op[0] == "recv"]
    assert [tuple(x[2]) for x in sends1] == [tuple(x[2]) for x in recvs0]
    # ZeRO shards tile the flat buffer
    shards = sorted(tuple(x["shard"]) for x in g)
    assert shards[0][0] == 0 and shards[-1][1] == 1000 * 64 and shards[0][1] == shards[1][0]
