"""Pins the CPU oracle (oracle/gpt_oracle.c) against the float64 torch-autograd golden fixtures
(tests/golden/make_golden.py) and the independent numpy restatement of its hashes."""
import math

import numpy as np
import pytest

import oracle_lib as O
from golden import make_golden as G

GOLD = O.ROOT / "tests" / "golden"


def _load(name):
    return dict(np.load(GOLD / f"{name}.npz"))


def test_init_hash_matches_independent_restatement():
    m = O.model(2, 64, 4, 128, 32)
    p = O.init_params(m, 1234)
    ref = G.init_params(2, 64, 128, 32, 1234)
    for tid, t in enumerate(ref):
        if t.size:
            np.testing.assert_array_equal(O.tensor(m, p, tid).reshape(t.shape), t)


def test_init_statistics():
    v = np.array([O.load().orc_init_value(7, 3, i, 0.02) for i in range(20000)], dtype=np.float64)
    assert abs(v.mean()) < 1e-3
    assert abs(v.std() - 0.02) < 1e-3
    assert np.abs(v).max() <= 0.02 * 2 * math.sqrt(3) + 1e-6  # Irwin-Hall(4) support


def test_dropout_hash_matches_restatement():
    lib = O.load()
    elems = np.arange(5000, dtype=np.int64) + 123456
    mine = np.array([lib.orc_dropout_keep(99, 3, 5, 1, int(e), 0.1) for e in elems], dtype=bool)
    ref = G.dropout_keep(99, 3, 5, 1, elems, 0.1)
    np.testing.assert_array_equal(mine, ref)
    assert abs(1 - mine.mean() - 0.1) < 0.02


def test_tokens_match_mt19937_64():
    np.testing.assert_array_equal(O.gen_tokens(1234, 700, 51200), G.mt19937_64_tokens(1234, 700, 51200))
    # first value of std::mt19937_64 default-seeded (5489) is 14514284786278117030 (C++ standard)
    assert int(O.gen_tokens(5489, 1, 2**31 - 1)[0]) == 14514284786278117030 % (2**31 - 1)


@pytest.mark.parametrize("name", ["gpt_small", "gpt_small_dropout"])
def test_oracle_matches_torch_fp64_full(name):
    g = _load(name)
    L, d, heads, V, s, nseq = (int(x) for x in g["cfg"])
    m = O.model(L, d, heads, V, s)
    o = O.opts(dropout=float(g["p_drop"]))
    p = O.init_params(m, 1234)
    tokens = g["tokens"].astype(np.int32)
    loss, grads = O.fwd_bwd(m, o, p, tokens)
    assert abs(loss - g["tok_loss"].sum()) <= 1e-4 * abs(g["tok_loss"].sum())
    for tid in range(O.load().orc_num_tensors(m)):
        key = f"grad_{tid}"
        if key not in g:
            continue
        mine = O.tensor(m, grads, tid).reshape(g[key].shape)
        ref = g[key]
        rel = np.linalg.norm(mine - ref) / max(np.linalg.norm(ref), 1e-30)
        assert rel < 1e-4, (tid, rel)
    # one Adam step from zero state (step 1), fed the golden gradients so the update arithmetic
    # itself is compared (sign-like updates of near-zero grads are ill-conditioned otherwise)
    gg = np.zeros_like(p)
    for tid in range(O.load().orc_num_tensors(m)):
        if f"grad_{tid}" in g:
            O.tensor(m, gg, tid)[...] = g[f"grad_{tid}"].reshape(O.tensor(m, gg, tid).shape)
    mom = np.zeros_like(p)
    var = np.zeros_like(p)
    p2 = p.copy()
    O.load().orc_adam(p.size, p2, gg, mom, var, 1, O.opts())
    for tid in range(O.load().orc_num_tensors(m)):
        key = f"adam_{tid}"
        if key in g:
            np.testing.assert_allclose(O.tensor(m, p2, tid).reshape(g[key].shape), g[key], rtol=1e-5, atol=1e-6)


def test_oracle_matches_torch_fp64_config1_shape():
    g = _load("gpt_tiny_cfg1")
    L, d, heads, V, s, nseq = (int(x) for x in g["cfg"])
    m = O.model(L, d, heads, V, s)
    p = O.init_params(m, 1234)
    loss, grads = O.fwd_bwd(m, O.opts(), p, g["tokens"].astype(np.int32))
    assert abs(loss - g["tok_loss"].sum()) <= 1e-4 * abs(g["tok_loss"].sum())
    for tid in range(O.load().orc_num_tensors(m)):
        if f"gidx_{tid}" not in g:
            continue
        flat = O.tensor(m, grads, tid).reshape(-1)
        assert abs(np.linalg.norm(flat) - g[f"gnorm_{tid}"]) <= 1e-4 * g[f"gnorm_{tid}"] + 1e-9
        np.testing.assert_allclose(flat[g[f"gidx_{tid}"]], g[f"gval_{tid}"], rtol=2e-3, atol=1e-7)


def test_bf16_emulation_stays_close():
    g = _load("gpt_small")
    L, d, heads, V, s, nseq = (int(x) for x in g["cfg"])
    m = O.model(L, d, heads, V, s)
    p = O.init_params(m, 1234)
    loss, _ = O.fwd_bwd(m, O.opts(bf16=1), p, g["tokens"].astype(np.int32))
    assert abs(loss - g["tok_loss"].sum()) <= 1e-2 * abs(g["tok_loss"].sum())
