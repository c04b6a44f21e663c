"""Kernel-level numerics on a B200 through the C-ABI: each sm_100a kernel against a plain PyTorch
fp32 reference of the same op (floating-point kernels; tolerances stated per test)."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
from paper_2312_12705_b200 import _lib as T  # noqa: E402

pytestmark = pytest.mark.gpu

DEV = "cuda"


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _rel(a, b):
    a, b = a.double(), b.double()
    return ((a - b).norm() / b.norm().clamp_min(1e-30)).item()


@pytest.fixture(scope="module", autouse=True)
def _gpu(native_lib):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    yield


@pytest.mark.parametrize("cg", [1, 2, 3])  # 3: CTA-pair 256 x 512 tiles when M % 256 == 0 and N % 512 == 0
@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(128, 64, 64), (256, 384, 192), (2048, 2304, 768), (1024, 51200 // 8, 256),
                                   (512, 512, 2048), (768, 1536, 1024)])
def test_gemm_layouts_vs_torch(a_mn, b_mn, M, N, K, cg):
    T.check(T.load().tp_gemm_force_cta_group(cg))
    g = torch.Generator(device=DEV).manual_seed(1)
    A = torch.randn((K, M) if a_mn else (M, K), device=DEV, generator=g).bfloat16()
    B = torch.randn((K, N) if b_mn else (N, K), device=DEV, generator=g).bfloat16()
    C = torch.empty(M, N, device=DEV, dtype=torch.bfloat16)
    T.gemm_bf16(M, N, K, A.data_ptr(), M if a_mn else K, a_mn, B.data_ptr(), N if b_mn else K, b_mn, C.data_ptr(), N,
                stream=_stream())
    ref = (A.t() if a_mn else A).float() @ (B.t() if b_mn else B).float().t()
    torch.cuda.synchronize()
    T.check(T.load().tp_gemm_force_cta_group(0))
    assert _rel(C.float(), ref) < 5e-3  # bf16 output rounding (2^-9) dominates


@pytest.mark.parametrize("cg", [1, 2, 3])
def test_gemm_fp32_accumulate_epilogue(cg):
    T.check(T.load().tp_gemm_force_cta_group(cg))
    M, N, K = 256, 512, 1024
    A = torch.randn(K, M, device=DEV).bfloat16()
    B = torch.randn(K, N, device=DEV).bfloat16()
    C = torch.randn(M, N, device=DEV)
    C0 = C.clone()
    T.gemm_bf16(M, N, K, A.data_ptr(), M, 1, B.data_ptr(), N, 1, C.data_ptr(), N, epi=2, accumulate=1, stream=_stream())
    torch.cuda.synchronize()
    T.check(T.load().tp_gemm_force_cta_group(0))
    assert _rel(C, C0 + A.float().t() @ B.float()) < 1e-5  # fp32 out: only summation order differs


@pytest.mark.parametrize("M,N,K", [(2048, 2048, 16384), (6144, 2048, 16384), (512, 512, 4096)])
def test_gemm_wgrad_split_k(M, N, K):
    """Weight-gradient shape (few tiles, long K): the automatic K-slicing reduces the slices into
    the fp32 accumulator with atomics; the result must equal C + A^T B up to summation order."""
    A = torch.randn(K, M, device=DEV).bfloat16()
    B = torch.randn(K, N, device=DEV).bfloat16()
    C = torch.randn(M, N, device=DEV)
    C0 = C.clone()
    T.gemm_bf16(M, N, K, A.data_ptr(), M, 1, B.data_ptr(), N, 1, C.data_ptr(), N, epi=2, accumulate=1, stream=_stream())
    torch.cuda.synchronize()
    # fp32 accumulation over K terms in a different order than torch's: ~1e-7 * sqrt(K)
    assert _rel(C, C0 + A.float().t() @ B.float()) < 5e-5


def _attn_ref(qkv, b, s, h, hd):
    d = h * hd
    q, k, v = qkv.float().view(b, s, 3, h, hd).unbind(2)
    q, k, v = (t.transpose(1, 2) for t in (q, k, v))
    return torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True)


# (8, 2048, 8, 128) has > 6 (kv block, head) items per SM: per-block backward; the others persistent.
# (8, 2048, 8, 128) and (5, 2048, 8, 128) run the two-query-tile forward; 5 x 8 = 40 (sequence, head)
# pairs leave a partial last L2 launch group (32 + 8)
@pytest.mark.parametrize("b,s,h,hd", [(2, 128, 4, 64), (1, 512, 2, 128), (2, 256, 2, 160), (1, 2048, 4, 160),
                                      (2, 384, 3, 160), (1, 2048, 2, 128),
                                      (8, 2048, 8, 128), (5, 2048, 8, 128)])
def test_flash_attention_fwd_bwd_vs_torch(b, s, h, hd):
    g = torch.Generator(device=DEV).manual_seed(2)
    M, d = b * s, h * hd
    qkv = (torch.randn(M, 3 * d, device=DEV, generator=g)).bfloat16()
    out = torch.empty(M, d, device=DEV, dtype=torch.bfloat16)
    lse = torch.empty(b, h, s, device=DEV)
    T.check(T.load().tp_flash_attn_fwd(b, s, h, hd, qkv.data_ptr(), out.data_ptr(), lse.data_ptr(), _stream()))
    x = qkv.float().requires_grad_(True)
    ref = _attn_ref(x, b, s, h, hd)  # [b, h, s, hd]
    ref_o = ref.transpose(1, 2).reshape(M, d)
    torch.cuda.synchronize()
    assert _rel(out.float(), ref_o) < 1e-2
    # lse (log2 units) vs logsumexp of the scaled scores
    q, k, _ = qkv.float().view(b, s, 3, h, hd).unbind(2)
    sc = torch.einsum("bihd,bjhd->bhij", q, k) / math.sqrt(hd)
    sc = sc.masked_fill(torch.triu(torch.ones(s, s, dtype=torch.bool, device=DEV), 1), float("-inf"))
    assert torch.allclose(lse, torch.logsumexp(sc, -1) / math.log(2), atol=2e-2, rtol=1e-3)
    dout = torch.randn(M, d, device=DEV, generator=g).bfloat16()
    ref_o.backward(dout.float())
    dqkv = torch.empty_like(qkv)
    D = torch.empty(b * h * s, device=DEV)
    dq_acc = torch.empty(M * d, device=DEV)
    T.check(T.load().tp_flash_attn_bwd(b, s, h, hd, qkv.data_ptr(), out.data_ptr(), dout.data_ptr(), lse.data_ptr(),
                                       D.data_ptr(), dq_acc.data_ptr(), dqkv.data_ptr(), _stream()))
    torch.cuda.synchronize()
    gref = x.grad
    for sec in range(3):  # dq, dk, dv
        e = _rel(dqkv[:, sec * d:(sec + 1) * d].float(), gref[:, sec * d:(sec + 1) * d])
        assert e < 2e-2, (sec, e)


# (16384, 2048) and (12288, 4096) fill the GPU: the persistent bulk-copy-staged LN backward
@pytest.mark.parametrize("rows,d", [(256, 256), (512, 2048), (128, 6144), (64, 12288), (32, 25600), (16384, 2048),
                                    (12288, 4096)])
def test_resid_layernorm_fwd_bwd_vs_torch(rows, d):
    g = torch.Generator(device=DEV).manual_seed(3)
    y = torch.randn(rows, d, device=DEV, generator=g).bfloat16()
    resid = torch.randn(rows, d, device=DEV, generator=g).bfloat16()
    bias = (0.1 * torch.randn(d, device=DEV, generator=g)).bfloat16()
    gamma = (1 + 0.1 * torch.randn(d, device=DEV, generator=g)).bfloat16()
    beta = (0.1 * torch.randn(d, device=DEV, generator=g)).bfloat16()
    h = torch.empty_like(y)
    ln = torch.empty_like(y)
    mean = torch.empty(rows, device=DEV)
    rstd = torch.empty(rows, device=DEV)
    T.check(T.load().tp_resid_layernorm_fwd(rows, d, y.data_ptr(), bias.data_ptr(), resid.data_ptr(), h.data_ptr(),
                                            gamma.data_ptr(), beta.data_ptr(), ln.data_ptr(), mean.data_ptr(),
                                            rstd.data_ptr(), 0, 0, 0, 0, 0.0, 0, _stream()))
    href = (resid.float() + (y.float() + bias.float())).bfloat16().float()  # h = r + (y + b), as the oracle
    torch.cuda.synchronize()
    assert torch.equal(h.float(), href)
    x = href.clone().requires_grad_(True)
    lref = torch.nn.functional.layer_norm(x, (d,), gamma.float(), beta.float(), eps=1e-5)
    assert _rel(ln.float(), lref) < 5e-3
    dy = torch.randn(rows, d, device=DEV, generator=g).bfloat16()
    rg = torch.randn(rows, d, device=DEV, generator=g).bfloat16()
    lref.backward(dy.float())
    dx = torch.empty_like(y)
    dgamma = torch.zeros(d, device=DEV)
    dbeta = torch.zeros(d, device=DEV)
    dbias = torch.zeros(d, device=DEV)
    ws = torch.empty(T.load().tp_layernorm_bwd_workspace_bytes(rows, d) // 4 + 1, device=DEV)
    T.check(T.load().tp_layernorm_bwd(rows, d, h.data_ptr(), dy.data_ptr(), rg.data_ptr(), gamma.data_ptr(),
                                      mean.data_ptr(), rstd.data_ptr(), dx.data_ptr(), dx.data_ptr(), dgamma.data_ptr(),
                                      dbeta.data_ptr(), dbias.data_ptr(), 0, 0, 0, 0, 0.0, 0, ws.data_ptr(), _stream()))
    torch.cuda.synchronize()
    dxref = x.grad + rg.float()
    assert _rel(dx.float(), dxref) < 1e-2
    xh = (href - href.mean(1, keepdim=True)) * torch.rsqrt(href.var(1, unbiased=False, keepdim=True) + 1e-5)
    assert _rel(dgamma, (dy.float() * xh).sum(0)) < 1e-3
    assert _rel(dbeta, dy.float().sum(0)) < 1e-4
    assert _rel(dbias, dx.float().sum(0)) < 1e-4


@pytest.mark.parametrize("rows,d", [(16384, 2048), (12288, 4096)])
def test_layernorm_bwd_stream_dropout(rows, d):
    """Persistent LN backward with hidden dropout on a separate dxd output: dx vs torch, the
    dropout mask vs the oracle's counter hash on sampled rows, dbias = column sums of stored dxd."""
    import oracle_lib as O
    g = torch.Generator(device=DEV).manual_seed(5)
    x = torch.randn(rows, d, device=DEV, generator=g).bfloat16()
    gamma = (1 + 0.1 * torch.randn(d, device=DEV, generator=g)).bfloat16()
    xf = x.float()
    mean = xf.mean(1).contiguous()
    rstd = torch.rsqrt(xf.var(1, unbiased=False) + 1e-5).contiguous()
    dy = torch.randn(rows, d, device=DEV, generator=g).bfloat16()
    rg = torch.randn(rows, d, device=DEV, generator=g).bfloat16()
    dx, dxd = torch.empty_like(x), torch.empty_like(x)
    dgamma, dbeta, dbias = (torch.zeros(d, device=DEV) for _ in range(3))
    ws = torch.empty(T.load().tp_layernorm_bwd_workspace_bytes(rows, d) // 4 + 1, device=DEV)
    p, seed, step, layer, site, base = 0.1, 1234, 2, 7, 1, 4096
    T.check(T.load().tp_layernorm_bwd(rows, d, x.data_ptr(), dy.data_ptr(), rg.data_ptr(), gamma.data_ptr(),
                                      mean.data_ptr(), rstd.data_ptr(), dx.data_ptr(), dxd.data_ptr(), dgamma.data_ptr(),
                                      dbeta.data_ptr(), dbias.data_ptr(), seed, step, layer, site, p, base,
                                      ws.data_ptr(), _stream()))
    torch.cuda.synchronize()
    xv = xf.clone().requires_grad_(True)
    torch.nn.functional.layer_norm(xv, (d,), gamma.float(), None, eps=1e-5).backward(dy.float())
    assert _rel(dx.float(), xv.grad + rg.float()) < 1e-2
    xh = (xf - mean[:, None]) * rstd[:, None]
    assert _rel(dgamma, (dy.float() * xh).sum(0)) < 1e-3
    assert _rel(dbeta, dy.float().sum(0)) < 1e-4
    assert _rel(dbias, dxd.float().sum(0)) < 1e-4
    lib = O.load()
    for r in (0, 1, rows // 2 + 3, rows - 1):
        keep = np.array([lib.orc_dropout_keep(seed, step, layer, site, base + r * d + c, p) for c in range(d)])
        got = dxd[r].float().cpu().numpy()
        ref = np.where(keep, dx[r].float().cpu().numpy() / (1 - p), 0.0)
        np.testing.assert_allclose(got, ref, rtol=8e-3, atol=1e-6)


def test_dropout_mask_matches_oracle_hash():
    import oracle_lib as O
    rows, d, p = 64, 256, 0.1
    y = torch.ones(rows, d, device=DEV).bfloat16()
    resid = torch.zeros(rows, d, device=DEV).bfloat16()
    h = torch.empty_like(y)
    T.check(T.load().tp_resid_layernorm_fwd(rows, d, y.data_ptr(), None, resid.data_ptr(), h.data_ptr(), None, None,
                                            None, None, None, 1234, 3, 5, 1, p, 776, _stream()))
    torch.cuda.synchronize()
    keep = h.float().cpu().numpy() != 0
    lib = O.load()
    ref = np.array([lib.orc_dropout_keep(1234, 3, 5, 1, 776 + i, p) for i in range(rows * d)], dtype=bool)
    np.testing.assert_array_equal(keep.reshape(-1), ref)
    np.testing.assert_allclose(h.float().cpu().numpy()[keep], np.float32(1 / 0.9), rtol=4e-3)


@pytest.mark.parametrize("rows,V", [(128, 1024), (256, 51200)])
def test_cross_entropy_vs_torch(rows, V):
    g = torch.Generator(device=DEV).manual_seed(4)
    logits = (3 * torch.randn(rows, V, device=DEV, generator=g)).bfloat16()
    labels = torch.randint(0, V, (rows,), device=DEV, generator=g, dtype=torch.int32)
    x = logits.float().requires_grad_(True)
    loss = torch.nn.functional.cross_entropy(x, labels.long(), reduction="none")
    (loss.sum() * 0.5).backward()
    row_loss = torch.empty(rows, device=DEV)
    stats = torch.empty(rows * 3, device=DEV)
    work = logits.clone()
    T.check(T.load().tp_cross_entropy(rows, V, work.data_ptr(), labels.data_ptr(), 0.5, row_loss.data_ptr(),
                                      stats.data_ptr(), _stream()))
    torch.cuda.synchronize()
    assert torch.allclose(row_loss, loss.detach(), rtol=1e-4, atol=1e-4)
    assert _rel(work.float(), x.grad) < 1e-2


def test_adam_step_vs_reference_formula():
    n = 4096
    g = torch.Generator(device=DEV).manual_seed(5)
    p = torch.randn(n, device=DEV, generator=g)
    m = 0.01 * torch.randn(n, device=DEV, generator=g)
    v = torch.rand(n, device=DEV, generator=g) * 1e-3
    gr = torch.randn(n, device=DEV, generator=g)
    pb = torch.empty(n, device=DEV, dtype=torch.bfloat16)
    P, Mm, Vv = p.clone(), m.clone(), v.clone()
    T.check(T.load().tp_adam_step(n, P.data_ptr(), Mm.data_ptr(), Vv.data_ptr(), gr.data_ptr(), pb.data_ptr(), 1e-3,
                                  0.9, 0.95, 1e-8, 0.1, 3, _stream()))
    torch.cuda.synchronize()
    m2 = 0.9 * m + 0.1 * gr
    v2 = 0.95 * v + 0.05 * gr * gr
    ref = p - 1e-3 * ((m2 / (1 - 0.9 ** 3)) / ((v2 / (1 - 0.95 ** 3)).sqrt() + 1e-8) + 0.1 * p)
    assert torch.allclose(Mm, m2, rtol=1e-6, atol=1e-7)
    assert torch.allclose(Vv, v2, rtol=1e-6, atol=1e-9)
    assert torch.allclose(P, ref, rtol=1e-5, atol=1e-6)
    assert torch.equal(pb, P.bfloat16())
