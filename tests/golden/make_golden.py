"""Generates the numerical golden fixtures that pin the CPU oracle (oracle/gpt_oracle.c).

The reference (`trainplan`) has no numerical train step, so the oracle is
pinned against an INDEPENDENT restatement: this script re-implements the counter-based init and
dropout hashes in numpy and the GPT decoder train step with torch CPU autograd in float64, then
stores tokens, per-token losses, gradients and one Adam step as .npz fixtures.

    python tests/golden/make_golden.py          # rewrites tests/golden/*.npz

Model convention (same as the oracle / product): pre-LN GPT, learned positions, tied LM head,
QKV rows ordered (q heads | k heads | v heads), tanh GeLU, LN eps 1e-5, hidden dropout after
embedding, attention projection and MLP (Megatron-DeepSpeed GPT as run in PAPER.md:305-327).
"""
from __future__ import annotations

import math
from pathlib import Path

import numpy as np
import torch

HERE = Path(__file__).resolve().parent
M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
TPL = 16  # tensor ids per layer


def mix64(z: np.ndarray) -> np.ndarray:
    z = (z + np.uint64(0x9E3779B97F4A7C15))
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def init_values(seed: int, tid: int, n: int, std: float) -> np.ndarray:
    with np.errstate(over="ignore"):
        key = mix64(np.array([seed ^ (tid << 48)], dtype=np.uint64))[0]
        idx = np.arange(n, dtype=np.uint64) * np.uint64(4)
        s = np.zeros(n, dtype=np.int64)
        for i in range(4):
            s += (mix64(key + idx + np.uint64(i)) >> np.uint64(40)).astype(np.int64)
    c = (s - (2 << 24)).astype(np.int32)
    scale = np.float32(std * math.sqrt(3.0) / 16777216.0)
    return c.astype(np.float32) * scale


def dropout_keep(seed: int, step: int, layer: int, site: int, elems: np.ndarray, p: float) -> np.ndarray:
    """One 64-bit hash per 4 consecutive elements; element e keeps iff its 16-bit field >= p*2^16."""
    if p <= 0:
        return np.ones(elems.shape, dtype=bool)
    with np.errstate(over="ignore"):
        key = np.uint64(seed) ^ np.uint64(0xD6E8FEB86659FD93) ^ np.uint64(step << 40) ^ \
            np.uint64((layer & 0xFFFF) << 16) ^ np.uint64(site)
        key = mix64(np.array([key], dtype=np.uint64))[0]
        e = elems.astype(np.uint64)
        h = mix64(key + (e >> np.uint64(2)))
        r = ((h >> (np.uint64(16) * (e & np.uint64(3)))) & np.uint64(0xFFFF)).astype(np.uint32)
    return r >= np.uint32(int(p * 65536.0))


def mt19937_64_tokens(seed: int, n: int, vocab: int) -> np.ndarray:
    """std::mt19937_64 (pure python; small n only)."""
    mt = [0] * 312
    mt[0] = seed & 0xFFFFFFFFFFFFFFFF
    for i in range(1, 312):
        mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
    idx = 312
    out = np.empty(n, dtype=np.int32)
    for j in range(n):
        if idx >= 312:
            for k in range(312):
                x = (mt[k] & 0xFFFFFFFF80000000) | (mt[(k + 1) % 312] & 0x7FFFFFFF)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                mt[k] = mt[(k + 156) % 312] ^ xa
            idx = 0
        y = mt[idx]
        idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        out[j] = y % vocab
    return out


def tensor_shapes(L, d, V, s):
    shapes = [(V, d), (s, d)]
    for _ in range(L):
        shapes += [(d,), (d,), (3 * d, d), (3 * d,), (d, d), (d,), (d,), (d,), (4 * d, d), (4 * d,),
                   (d, 4 * d), (d,), (0,), (0,), (0,), (0,)]
    shapes += [(d,), (d,)]
    return shapes


def init_params(L, d, V, s, seed):
    params = []
    for tid, shp in enumerate(tensor_shapes(L, d, V, s)):
        n = int(np.prod(shp))
        j = (tid - 2) % TPL if 2 <= tid < 2 + TPL * L else -1
        if tid < 2 or j in (2, 8):
            std = 0.02
        elif j in (4, 10):
            std = 0.02 / math.sqrt(2.0 * L)
        else:
            std = 0.0
        if std > 0:
            v = init_values(seed, tid, n, std)
        else:
            const = 1.0 if (j in (0, 6) or tid == 2 + TPL * L) else 0.0
            v = np.full(n, const, dtype=np.float32)
        params.append(v.reshape(shp))
    return params


def gelu_t(x):
    return 0.5 * x * (1 + torch.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3)))


def forward(P, tokens, L, d, heads, V, s, p_drop, seed, step, sample0):
    nseq = tokens.shape[0]
    T = nseq * s
    hd = d // heads
    inp = torch.as_tensor(tokens[:, :s].astype(np.int64))
    lab = torch.as_tensor(tokens[:, 1:].astype(np.int64)).reshape(-1)
    base_elem = sample0 * s * d
    elems = np.arange(T * d, dtype=np.int64) + base_elem

    def drop(x, layer, site):
        if p_drop <= 0:
            return x
        keep = torch.as_tensor(dropout_keep(seed, step, layer, site, elems, p_drop).reshape(T, d))
        return torch.where(keep, x * (1.0 / (1.0 - p_drop)), torch.zeros_like(x))

    h = P[0][inp.reshape(-1)] + P[1][torch.arange(s).repeat(nseq)]
    h = drop(h, 0xFFFF, 2)
    mask = torch.triu(torch.ones(s, s, dtype=torch.bool), 1)
    for l in range(L):
        b = 2 + TPL * l
        a = torch.nn.functional.layer_norm(h, (d,), P[b], P[b + 1], eps=1e-5)
        qkv = a @ P[b + 2].t() + P[b + 3]
        q, k, v = qkv[:, :d], qkv[:, d:2 * d], qkv[:, 2 * d:]
        q = q.reshape(nseq, s, heads, hd).transpose(1, 2)
        k = k.reshape(nseq, s, heads, hd).transpose(1, 2)
        v = v.reshape(nseq, s, heads, hd).transpose(1, 2)
        sc = (q @ k.transpose(-1, -2)) / math.sqrt(hd)
        sc = sc.masked_fill(mask, float("-inf"))
        o = torch.softmax(sc, -1) @ v
        o = o.transpose(1, 2).reshape(T, d)
        y = o @ P[b + 4].t() + P[b + 5]
        h = h + drop(y, l, 0)
        m = torch.nn.functional.layer_norm(h, (d,), P[b + 6], P[b + 7], eps=1e-5)
        u = m @ P[b + 8].t() + P[b + 9]
        y = gelu_t(u) @ P[b + 10].t() + P[b + 11]
        h = h + drop(y, l, 1)
    f = 2 + TPL * L
    hf = torch.nn.functional.layer_norm(h, (d,), P[f], P[f + 1], eps=1e-5)
    logits = hf @ P[0].t()
    tok_loss = torch.nn.functional.cross_entropy(logits, lab, reduction="none")
    return tok_loss


def make_case(name, L, d, heads, V, s, nseq, p_drop, full_grads=True):
    seed, tok_seed, step, sample0 = 1234, 1234, 1, 0
    params = init_params(L, d, V, s, seed)
    tokens = mt19937_64_tokens(tok_seed, nseq * (s + 1), V).reshape(nseq, s + 1)
    P = [torch.tensor(p, dtype=torch.float64, requires_grad=True) for p in params]
    tok_loss = forward(P, tokens, L, d, heads, V, s, p_drop, seed, step, sample0)
    scale = 1.0 / (nseq * s)
    (tok_loss.sum() * scale).backward()
    out = {"cfg": np.array([L, d, heads, V, s, nseq]), "p_drop": np.array(p_drop),
           "tokens": tokens, "tok_loss": tok_loss.detach().numpy(),
           "init_checksum": np.array([float(np.abs(p.astype(np.float64)).sum()) for p in params])}
    grads = [p.grad.numpy() if p.grad is not None else np.zeros(p.shape) for p in P]
    if full_grads:
        for i, g in enumerate(grads):
            if g.size:
                out[f"grad_{i}"] = g.astype(np.float32)
        # one Adam step (lr 1e-3, betas 0.9/0.95, eps 1e-8, wd 0.01) on fp64
        lr, b1, b2, eps, wd = 1e-3, 0.9, 0.95, 1e-8, 0.01
        for i, (p, g) in enumerate(zip(params, grads)):
            if not g.size:
                continue
            m = (1 - b1) * g
            v = (1 - b2) * g * g
            mh, vh = m / (1 - b1), v / (1 - b2)
            out[f"adam_{i}"] = (p - lr * (mh / (np.sqrt(vh) + eps) + wd * p)).astype(np.float32)
    else:
        rng = np.random.default_rng(0)
        for i, g in enumerate(grads):
            if g.size:
                flat = g.reshape(-1)
                idx = np.unique(np.concatenate([np.arange(min(64, flat.size)),
                                                rng.integers(0, flat.size, 192)]))
                out[f"gidx_{i}"] = idx
                out[f"gval_{i}"] = flat[idx].astype(np.float32)
                out[f"gnorm_{i}"] = np.array(np.linalg.norm(flat))
    np.savez_compressed(HERE / f"{name}.npz", **out)
    print(name, "loss", float(tok_loss.mean()))


if __name__ == "__main__":
    torch.set_num_threads(8)
    make_case("gpt_small", L=2, d=64, heads=4, V=128, s=32, nseq=2, p_drop=0.0)
    make_case("gpt_small_dropout", L=2, d=64, heads=4, V=128, s=32, nseq=2, p_drop=0.1)
    # BASELINE config 1 shape (tiny GPT: 2 layers, hidden 256, 4 heads, seq 128), V reduced to
    # 1024 to keep the fixture small; sampled gradients.
    make_case("gpt_tiny_cfg1", L=2, d=256, heads=4, V=1024, s=128, nseq=2, p_drop=0.0, full_grads=False)
