"""Multi-GPU parity (one process per GPU, NCCL over NVLink): TP / PP (1F1B) / DP (ZeRO-1) and their
combinations against the CPU oracle on the same tokens and counter-based weights.

Checks per run: fp32 master shards bit-exact to the oracle's initial weights after the TP/PP/DP
index maps (shard indexing), identical loss on every rank ≈ oracle loss, DP-reduced gradients per
tensor (rel L2 <= 3e-2, cosine >= 0.999), and the ZeRO-1 Adam update of every shard (rtol 1e-5)
on the reduced gradients. Skipped when the box has fewer GPUs than the layout needs."""
import json
import subprocess
import sys
import tempfile
from pathlib import Path

import numpy as np
import pytest

import oracle_lib as O
from paper_2312_12705_b200 import _lib as T

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]
ROOT = Path(__file__).resolve().parents[1]


def _ngpus():
    try:
        out = subprocess.run(["nvidia-smi", "-L"], capture_output=True, text=True, timeout=30).stdout
        return sum(1 for l in out.splitlines() if l.startswith("GPU "))
    except (OSError, subprocess.SubprocessError):
        return 0


def _rel(a, b):
    a, b = a.ravel().astype(np.float64), b.ravel().astype(np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def _cos(a, b):
    a, b = a.ravel().astype(np.float64), b.ravel().astype(np.float64)
    return float(a @ b / max(np.linalg.norm(a) * np.linalg.norm(b), 1e-30))


def _slice(full, info):
    grow, gcol = T.global_index_map(info)
    return full[np.ix_(grow, gcol)] if info["cols"] > 1 else full[grow]


def _slice_rows(full, info, local_rows):
    grow, gcol = T.global_index_map(info)
    grow = grow[local_rows]
    return full[np.ix_(grow, gcol)] if info["cols"] > 1 else full[grow]


def run_layout(tp, pp, dp, L=2, d=256, a=4, V=1024, s=128, mbs=1, gbs=None, ckpt=0, dropout=0.0, v=1, tp_env=None,
               want_tp_mode=None, zero=1, sample=0, want_variants=()):
    """One train step on tp*pp*dp GPUs against the oracle. zero = ZeRO stage (1 sharded, 0
    replicated). sample > 0 (dp == 1 only): the ranks return `sample` evenly spaced local rows per
    tensor instead of their full flat buffers — the wide (22B / 175B / 1T) layouts."""
    world = tp * pp * dp
    if _ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    gbs = gbs or mbs * dp * 2
    c = dict(L=L, d=d, a=a, V=V, s=s, tp=tp, pp=pp, dp=dp, mbs=mbs, gbs=gbs, ckpt=ckpt, dropout=dropout, v=v,
             tp_env=tp_env or {}, zero=zero, sample=sample)
    (ROOT / ".mp_tmp").mkdir(exist_ok=True)  # not /tmp: the 1T-width dumps should not sit in a tmpfs
    with tempfile.TemporaryDirectory(dir=ROOT / ".mp_tmp") as td:
        procs = [subprocess.Popen([sys.executable, str(ROOT / "tests" / "mp_worker.py"), "--cfg", json.dumps(c),
                                   "--rank", str(r), "--world", str(world), "--out", td],
                                  stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
                 for r in range(world)]
        outs = []
        for p in procs:
            try:
                outs.append(p.communicate(timeout=600)[0])
            except subprocess.TimeoutExpired:
                for q in procs:
                    q.kill()
                raise
        for p, o in zip(procs, outs):
            assert p.returncode == 0, o[-3000:]
        ranks = [dict(np.load(Path(td) / f"rank{r}.npz")) for r in range(world)]
    # oracle on the global batch
    om = O.model(L, d, a, V, s)
    oo = O.opts(dropout=dropout, seed=1234, bf16=1, lr=1e-3, wd=0.01)
    params = O.init_params(om, 1234)
    tokens = O.gen_tokens(1234, gbs * (s + 1), V).reshape(gbs, s + 1)
    grads = np.zeros_like(params)
    oloss = 0.0
    for i in range(gbs // mbs):
        l, _ = O.fwd_bwd(om, oo, params, tokens[i * mbs:(i + 1) * mbs], sample0=i * mbs, step=1,
                         loss_scale=1.0 / (gbs * s), grads=grads)
        oloss += l
    oloss /= gbs * s
    if want_tp_mode is not None:
        assert {int(r["tp_mode"]) for r in ranks} == {want_tp_mode}, [int(r["tp_mode"]) for r in ranks]
    losses = [float(r["loss"]) for r in ranks]
    assert max(losses) - min(losses) < 1e-6, losses
    assert abs(losses[0] - oloss) <= 1e-2 * max(1.0, oloss), (losses[0], oloss)
    report = []
    b1, b2, lr, eps, wd = np.float32(0.9), np.float32(0.95), np.float32(1e-3), np.float32(1e-8), np.float32(0.01)

    def check_tensor(t, p, tid, w0, g, w1, init_ref, g_ref, info):
        np.testing.assert_array_equal(w0, init_ref, err_msg=f"init tid {tid}")
        if np.linalg.norm(g_ref) > 1e-6:
            e, cs = _rel(g, g_ref), _cos(g, g_ref)
            report.append((t, p, tid, e, cs))
            # vector parameters (LayerNorm gamma / beta, biases) are sums over every token of
            # bf16-rounded per-token terms that largely cancel: at 12k-25k widths their relative
            # error sits a little above the matrices' (same cosine bar)
            tol = 3e-2 if g.ndim == 2 and info["cols"] > 1 else 5e-2
            assert e < tol and cs > 0.999, (t, p, tid, e, cs)
        mh, vh = ((1 - b1) * g) / (1 - b1), ((1 - b2) * g * g) / (1 - b2)
        ref = w0 - lr * (mh / (np.sqrt(vh) + eps) + wd * w0)
        np.testing.assert_allclose(w1, ref, rtol=1e-5, atol=1e-7, err_msg=f"adam tid {tid}")

    for t in range(tp):
        for p in range(pp):
            members = [r for r in ranks if tuple(r["coords"][:2]) == (t, p)]
            members.sort(key=lambda r: int(r["coords"][2]))
            layout = {int(k): v for k, v in json.loads(str(members[0]["layout"])).items()}
            if sample:
                m = members[0]
                for tid, info in layout.items():
                    rows = m[f"rows_{tid}"]
                    shape = (len(rows), info["cols"]) if info["cols"] > 1 else (len(rows),)
                    check_tensor(t, p, tid, m[f"m0_{tid}"].reshape(shape), m[f"g_{tid}"].reshape(shape),
                                 m[f"m1_{tid}"].reshape(shape), _slice_rows(O.tensor(om, params, tid), info, rows),
                                 _slice_rows(O.tensor(om, grads, tid), info, rows), info)
                continue
            P = int(members[0]["P"])
            if zero == 0:  # replicated: every DP rank holds the reduced gradients and the full master
                red, m0, m1 = members[0]["grads"], members[0]["master0"], members[0]["master1"]
                for other in members[1:]:
                    np.testing.assert_array_equal(other["master1"], m1)
            else:
                red, m0, m1 = np.zeros(P, np.float32), np.zeros(P, np.float32), np.zeros(P, np.float32)
                for off, ln, moff in members[0]["buckets"]:  # DP rank k owns slice k of every bucket
                    per = ln // dp
                    for k, m in enumerate(members):
                        lo = off + k * per
                        red[lo:lo + per] = m["grads"][lo:lo + per]
                        m0[lo:lo + per] = m["master0"][moff:moff + per]
                        m1[lo:lo + per] = m["master1"][moff:moff + per]
            for tid, info in layout.items():
                n = info["rows"] * info["cols"]
                off = info["offset"]
                shape = (info["rows"], info["cols"]) if info["cols"] > 1 else (info["rows"],)
                check_tensor(t, p, tid, m0[off:off + n].reshape(shape), red[off:off + n].reshape(shape),
                             m1[off:off + n].reshape(shape), _slice(O.tensor(om, params, tid), info),
                             _slice(O.tensor(om, grads, tid), info), info)
    print(json.dumps({"layout": f"tp{tp}.pp{pp}.dp{dp}", "L": L, "d": d, "a": a, "s": s, "V": V, "loss": losses[0],
                      "oracle_loss": oloss, "worst_grad_rel": max((r[3] for r in report), default=0.0),
                      "min_cos": min((r[4] for r in report), default=1.0),
                      "per_tensor": [[int(x) for x in r[:3]] + [round(r[3], 5), round(r[4], 6)] for r in report],
                      "variants": json.loads(str(ranks[0]["variants"]))}))
    for name in want_variants:  # the kernel variants the production layouts rely on ran
        assert all(json.loads(str(r["variants"]))[name] > 0 for r in ranks), name
    return losses[0], oloss, report


def test_tp2():
    # NVSwitch boxes run sequence parallelism (LayerNorms fused with the NVLS reduce-scatter/allgather)
    run_layout(tp=2, pp=1, dp=1, dropout=0.1, want_tp_mode=3)


def test_tp2_nvls_allreduce_without_sp():
    run_layout(tp=2, pp=1, dp=1, dropout=0.1, tp_env={"GPTB200_TP_SP": "0"}, want_tp_mode=2)


def test_tp2_nccl_allreduce():
    run_layout(tp=2, pp=1, dp=1, tp_env={"GPTB200_TP_SP": "0", "GPTB200_TP_NVLS": "0"}, want_tp_mode=1)


def test_pp2_1f1b_four_microbatches():
    run_layout(tp=1, pp=2, dp=1, gbs=4)


def test_dp2_zero1():
    run_layout(tp=1, pp=1, dp=2)


def test_dp2_zero1_dropout():
    run_layout(tp=1, pp=1, dp=2, dropout=0.1)


def test_tp2_pp2():
    run_layout(tp=2, pp=2, dp=1, gbs=4)


def test_tp2_ckpt_four_layers_dropout():
    # sequence parallel + checkpointing: recompute of layer l-1 overlaps the backward of layer l
    run_layout(tp=2, pp=1, dp=1, L=4, gbs=2, ckpt=1, dropout=0.1, want_tp_mode=3)


def test_tp2_dp2_ckpt():
    run_layout(tp=2, pp=1, dp=2, ckpt=1)


def test_pp2_dp2():
    run_layout(tp=1, pp=2, dp=2, gbs=8)


def test_pp2_interleaved_v2():
    # 4 layers = 2 devices x 2 chunks: device 0 holds layers {0, 2}, device 1 {1, 3}
    run_layout(tp=1, pp=2, dp=1, L=4, gbs=4, v=2)


def test_pp2_interleaved_v2_dropout_late_head():
    # m == p: every forward runs before the first backward, so the LM head is deferred
    run_layout(tp=1, pp=2, dp=1, L=4, gbs=2, v=2, dropout=0.1)


def test_tp2_pp2_interleaved_v2_ckpt():
    run_layout(tp=2, pp=2, dp=1, L=4, gbs=4, v=2, ckpt=1)


def test_pp2_dp2_interleaved_v2():
    run_layout(tp=1, pp=2, dp=2, L=4, gbs=8, v=2)


def test_config1_tp2_pp2_dp2():
    # BASELINE config 1 layout (needs 8 GPUs)
    run_layout(tp=2, pp=2, dp=2, gbs=8)


def test_dp2_zero0_replicated():
    # zero_stage 0 (search point zero1 = false): gradient allreduce, every rank updates everything
    run_layout(tp=1, pp=1, dp=2, zero=0, dropout=0.1)


# ---- BASELINE widths (TP-rank-local shapes of configs 3-5; reduced depth / sequence / vocab)

def test_tp2_22b_width_ckpt():
    # config 3 width: d 6144, 48 heads (hd 128), TP2 -> 24 heads / 3072 columns per rank
    run_layout(tp=2, pp=1, dp=1, L=1, d=6144, a=48, V=1024, s=1024, gbs=2, ckpt=1, dropout=0.1, want_tp_mode=3,
               want_variants=("gemm_pair_256", "attn_fwd_persistent"))


def test_tp4_22b_width_ckpt():
    run_layout(tp=4, pp=1, dp=1, L=2, d=6144, a=48, V=1024, s=1024, gbs=2, ckpt=1, dropout=0.1, want_tp_mode=3,
               sample=48)


def test_tp2_pp2_175b_width_ckpt():
    # config 4 width: d 12288, 96 heads, TP2 x PP2 1F1B, 4 microbatches
    run_layout(tp=2, pp=2, dp=1, L=2, d=12288, a=96, V=1024, s=256, gbs=4, ckpt=1, want_tp_mode=3, sample=32)


def test_tp4_1t_width_hd160_ckpt():
    # config 5 width: d 25600, 160 heads (hd 160), TP4 -> 40 heads / 6400 columns per rank; the SP
    # LayerNorm kernels at their widest instantiation and the hd-160 attention kernels
    run_layout(tp=4, pp=1, dp=1, L=1, d=25600, a=160, V=512, s=256, gbs=1, ckpt=1, want_tp_mode=3, sample=24,
               want_variants=("attn_bwd_hd160",))
