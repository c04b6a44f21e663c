"""Host-side logic of the multi-rank path, on CPU.

1. Stage::step() executes tp_pipeline_actions (runtime/pipe_exec.h) for the reference-identical
   per-device orders (1F1B and interleaved 1F1B, pipesim.cpp:31-91): receives block the compute
   stream right before the consuming op, sends run on one side stream per direction (each ring
   link and direction its own 2-rank NCCL communicator), and an op reusing an activation slot or
   gradient buffer first waits for that buffer's previous send. `replay` runs every device's plan
   under NCCL rendezvous semantics and proves all devices finish (no deadlock), every activation /
   gradient reaches the right virtual stage in order, and buffers are never overwritten in flight.
2. world_size-2 gloo run: each process derives its rank coordinates, plan and ZeRO-1 shard range
   through the C-ABI; rank 0 checks the send/receive sequences of the two stages pair up.
"""
import os
import socket
import sys
from pathlib import Path

import pytest

from paper_2312_12705_b200 import _lib as T

ROOT = Path(__file__).resolve().parents[1]


def replay(p, m, v, ring=2, forward_only=False, plans=None):
    """Returns the delivered messages [(kind, mb, sender_vstage, receiver_device)]."""
    plans = plans or [T.pipeline_actions(p, m, v, d, ring, forward_only) for d in range(p)]
    pc, phase = [0] * p, [0] * p
    queue = {(d, k): [] for d in range(p) for k in ("act", "grad")}  # side-stream FIFO per direction
    busy = [set() for _ in range(p)]  # ("slot", i) / ("dh", i) with a send in flight
    delivered = []
    while not all(pc[d] == len(plans[d]) for d in range(p)):
        progressed = False
        for d in range(p):
            if pc[d] == len(plans[d]):
                continue
            a = plans[d][pc[d]]
            fwd = a["kind"] == 0
            vs = a["chunk"] * p + d
            buf = ("slot", a["slot"]) if fwd else ("dh", a["dh"])
            if phase[d] == 0:  # cudaStreamWaitEvent on the buffer's last send
                if buf in busy[d]:
                    continue
                phase[d] = 1 if a["flags"] & T.PA_RECV else 2
                progressed = True
            if phase[d] == 1:  # ncclRecv posted on the compute stream: rendezvous with the peer's send
                src = (d - 1) % p if fwd else (d + 1) % p
                kind = "act" if fwd else "grad"
                q = queue[(src, kind)]
                if not q:
                    continue
                tag, sbuf = q.pop(0)
                want = (kind, a["mb"], vs - 1 if fwd else vs + 1)
                assert tag == want, f"device {d} expected {want}, link delivered {tag}"
                busy[src].discard(sbuf)
                delivered.append(tag + (d,))
                phase[d] = 2
                progressed = True
            if phase[d] == 2:  # the op runs; its output send is queued on the side stream
                if a["flags"] & T.PA_SEND:
                    assert buf not in busy[d]
                    queue[(d, "act" if fwd else "grad")].append((("act" if fwd else "grad", a["mb"], vs), buf))
                    busy[d].add(buf)
                pc[d] += 1
                phase[d] = 0
                progressed = True
        if not progressed:
            raise AssertionError(f"deadlock p={p} m={m} v={v} at {pc}")
    assert all(not q for q in queue.values()), "unmatched sends"
    return delivered


def test_replay_detects_mismatched_links(native_lib):
    """Sanity check of the replay: a plan whose two devices disagree on the order deadlocks or
    mis-delivers."""
    plans = [T.pipeline_actions(2, 4, 1, d) for d in range(2)]
    plans[1] = plans[1][2:] + plans[1][:2]
    with pytest.raises(AssertionError):
        replay(2, 4, 1, plans=plans)


@pytest.mark.parametrize("p", [2, 3, 4, 8])
@pytest.mark.parametrize("m", [1, 2, 3, 4, 7, 8, 16])
def test_1f1b_plan_is_deadlock_free(native_lib, p, m):
    delivered = replay(p, m, 1)
    acts = sorted((vs, mb) for k, mb, vs, _ in delivered if k == "act")
    grads = sorted((vs, mb) for k, mb, vs, _ in delivered if k == "grad")
    assert acts == sorted((s, mb) for s in range(p - 1) for mb in range(m))
    assert grads == sorted((s, mb) for s in range(1, p) for mb in range(m))


@pytest.mark.parametrize("p", [2, 3, 4, 8])
@pytest.mark.parametrize("m", [2, 4, 6, 8, 16])
@pytest.mark.parametrize("v", [2, 3, 4])
def test_interleaved_plan_is_deadlock_free(native_lib, p, m, v):
    delivered = replay(p, m, v)
    nvs = p * v
    acts = sorted((vs, mb) for k, mb, vs, _ in delivered if k == "act")
    grads = sorted((vs, mb) for k, mb, vs, _ in delivered if k == "grad")
    assert acts == sorted((s, mb) for s in range(nvs - 1) for mb in range(m))
    assert grads == sorted((s, mb) for s in range(1, nvs) for mb in range(m))
    assert all(dev == (vs + 1) % p for k, mb, vs, dev in delivered if k == "act")


@pytest.mark.parametrize("p,v", [(2, 1), (2, 2), (4, 2), (3, 3)])
def test_forward_only_plan(native_lib, p, v):
    delivered = replay(p, 5, v, forward_only=True)
    assert len(delivered) == 5 * (p * v - 1)


@pytest.mark.parametrize("p,m,v", [(2, 4, 1), (4, 8, 1), (2, 4, 2), (2, 2, 2), (4, 8, 2), (3, 5, 2)])
def test_plan_buffers_and_head(native_lib, p, m, v):
    for d in range(p):
        plan = T.pipeline_actions(p, m, v, d)
        live = {}
        for i, a in enumerate(plan):
            key = (a["mb"], a["chunk"])
            if a["kind"] == 0:
                assert a["slot"] not in live.values(), "slot reused while its microbatch is alive"
                live[key] = a["slot"]
            else:
                assert live.pop(key) == a["slot"]
        assert not live
        if v == 1:  # 1F1B keeps at most p - d microbatches alive
            assert max(a["slot"] for a in plan) + 1 <= min(m, p - d)
        if d == p - 1:  # last virtual stage: the LM head runs exactly once per microbatch
            for mb in range(m):
                f = [a for a in plan if a["kind"] == 0 and a["mb"] == mb and a["chunk"] == v - 1][0]
                b = [a for a in plan if a["kind"] == 1 and a["mb"] == mb and a["chunk"] == v - 1][0]
                assert bool(f["flags"] & T.PA_HEAD) != bool(b["flags"] & T.PA_HEAD_LATE)
        for c in range(v):  # grads of a chunk are final after its flagged backward
            idx = [i for i, a in enumerate(plan) if a["chunk"] == c and a["kind"] == 1]
            last = [i for i in idx if plan[i]["flags"] & T.PA_LAST_MB]
            assert last == [idx[-1]]


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
    plan = TL.pipeline_actions(pp, 4, 1, coords[1])
    sends = [("act" if a["kind"] == 0 else "grad", a["mb"]) for a in plan if a["flags"] & TL.PA_SEND]
    recvs = [("act" if a["kind"] == 0 else "grad", a["mb"]) for a in plan if a["flags"] & TL.PA_RECV]
    mine = {"rank": rank, "coords": coords, "order": order, "shard": shard, "sends": sends, "recvs": recvs}
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
    assert g[0]["sends"] == g[1]["recvs"] and g[1]["sends"] == g[0]["recvs"]
    assert [k for k, _ in g[0]["sends"]] == ["act"] * 4 and [k for k, _ in g[1]["sends"]] == ["grad"] * 4
    # ZeRO shards tile the flat buffer
    shards = sorted(tuple(x["shard"]) for x in g)
    assert shards[0][0] == 0 and shards[-1][1] == 1000 * 64 and shards[0][1] == shards[1][0]
