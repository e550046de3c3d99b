"""Numerics of the sm_100a stage kernels vs plain PyTorch fp32 references.

Tolerances (stated per test): bf16 outputs carry one bf16 rounding of an
fp32-exact computation -> rel-L2 <= 1e-2; fp32 outputs <= 1e-4; attention
(bf16 P, bf16 inputs) rel-L2 <= 2e-2 vs the fp32 reference.
"""
import math

import os

import pytest
import torch

pytestmark = pytest.mark.gpu


def rel(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm().clamp_min(1e-30)).item()


def rnd(*shape, seed=0, scale=1.0, dtype=torch.bfloat16):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.randn(*shape, device="cuda", generator=g) * scale).to(dtype)


@pytest.mark.parametrize("T,h", [(256, 256), (1024, 4096), (77, 2048), (300, 5120), (64, 8192), (33, 3072)])
def test_rmsnorm_fwd_bwd(T, h):
    from paper_2604_27085_b200 import kernels as K
    x, w, dy = rnd(T, h, seed=1), rnd(h, seed=2, scale=0.5) + 1, rnd(T, h, seed=3)
    dres = rnd(T, h, seed=4, dtype=torch.float32)
    y = torch.empty_like(x)
    rstd = torch.empty(T, device="cuda")
    K.rmsnorm_fwd(x, w, y, rstd)
    xf = x.float().requires_grad_(True)
    wf = w.float().requires_grad_(True)
    ref = wf * (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + 1e-6))
    assert rel(y, ref) < 1e-2
    dx32 = torch.empty(T, h, device="cuda")
    dx16 = torch.empty(T, h, device="cuda", dtype=torch.bfloat16)
    dw = torch.zeros(h, device="cuda")
    K.rmsnorm_bwd(dy, x, w, rstd, dx32=dx32, dx16=dx16, dw=dw, dres=dres)
    ref.backward(dy.float())
    assert rel(dx32, xf.grad + dres) < 1e-4
    assert rel(dx16, xf.grad + dres) < 1e-2
    assert rel(dw, wf.grad) < 1e-4


@pytest.mark.parametrize("T,h", [(512, 4096), (128, 2048)])
def test_rmsnorm_bwd_staged_no_residual(T, h):
    """The bulk-copy-staged backward without a residual gradient and bf16-only
    output (slot = dy | x | rstd group), against the register version's math."""
    from paper_2604_27085_b200 import kernels as K
    x, w, dy = rnd(T, h, seed=21), rnd(h, seed=22, scale=0.5) + 1, rnd(T, h, seed=23)
    y = torch.empty_like(x)
    rstd = torch.empty(T, device="cuda")
    K.rmsnorm_fwd(x, w, y, rstd)
    xf = x.float().requires_grad_(True)
    wf = w.float().requires_grad_(True)
    ref = wf * (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + 1e-6))
    ref.backward(dy.float())
    dx16 = torch.empty(T, h, device="cuda", dtype=torch.bfloat16)
    dw = torch.zeros(h, device="cuda")
    K.rmsnorm_bwd(dy, x, w, rstd, dx16=dx16, dw=dw)
    assert rel(dx16, xf.grad) < 1e-2
    assert rel(dw, wf.grad) < 1e-4


def _rope_ref(x, cs):  # x [T, H, hd] fp32; cs [T, hd/2, 2]
    hd = x.shape[-1]
    cos = torch.cat([cs[..., 0], cs[..., 0]], -1)[:, None, :]
    sin = torch.cat([cs[..., 1], cs[..., 1]], -1)[:, None, :]
    x1, x2 = x[..., : hd // 2], x[..., hd // 2:]
    return x * cos + torch.cat([-x2, x1], -1) * sin


@pytest.mark.parametrize("hd,nq,nk", [(128, 32, 8), (64, 4, 2), (128, 16, 8), (128, 64, 8), (128, 64, 4), (128, 6, 2)])
def test_qk_norm_rope_fwd_bwd(hd, nq, nk):
    from paper_2604_27085_b200 import kernels as K
    seq, T = 256, 512
    qkv = rnd(T, (nq + 2 * nk) * hd, seed=5)
    qw, kw = rnd(hd, seed=6, scale=0.2) + 1, rnd(hd, seed=7, scale=0.2) + 1
    cs = K.rope_table(seq, hd).cuda()
    q = torch.empty(T, nq * hd, device="cuda", dtype=torch.bfloat16)
    k = torch.empty(T, nk * hd, device="cuda", dtype=torch.bfloat16)
    rq = torch.empty(T, nq, device="cuda")
    rk = torch.empty(T, nk, device="cuda")
    K.qk_norm_rope_fwd(qkv, nq, nk, hd, qw, kw, cs, seq, q, k, rq, rk)
    pos_cs = cs[torch.arange(T, device="cuda") % seq]
    x = qkv.float().requires_grad_(True)
    qwf, kwf = qw.float().requires_grad_(True), kw.float().requires_grad_(True)
    xq = x[:, : nq * hd].view(T, nq, hd)
    xk = x[:, nq * hd:(nq + nk) * hd].view(T, nk, hd)

    def norm(t, w):
        return w * (t * torch.rsqrt(t.pow(2).mean(-1, keepdim=True) + 1e-6))
    qr = _rope_ref(norm(xq, qwf), pos_cs)
    kr = _rope_ref(norm(xk, kwf), pos_cs)
    assert rel(q.view(T, nq, hd), qr) < 1e-2
    assert rel(k.view(T, nk, hd), kr) < 1e-2
    dq, dk = rnd(T, nq * hd, seed=8), rnd(T, nk * hd, seed=9)
    dqkv = torch.zeros_like(qkv)
    dqw, dkw = torch.zeros(hd, device="cuda"), torch.zeros(hd, device="cuda")
    K.qk_norm_rope_bwd(dq, dk, qkv, nq, nk, hd, qw, kw, rq, rk, cs, seq, dqkv, dqw, dkw)
    (qr * dq.float().view(T, nq, hd)).sum().add_((kr * dk.float().view(T, nk, hd)).sum()).backward()
    assert rel(dqkv[:, :(nq + nk) * hd], x.grad[:, :(nq + nk) * hd]) < 1e-2
    assert rel(dqw, qwf.grad) < 5e-3
    assert rel(dkw, kwf.grad) < 5e-3


def test_swiglu_fwd_bwd():
    from paper_2604_27085_b200 import kernels as K
    T, m = 512, 1536
    gu, dact = rnd(T, 2 * m, seed=10), rnd(T, m, seed=11)
    act = torch.empty(T, m, device="cuda", dtype=torch.bfloat16)
    K.swiglu_fwd(gu, act)
    x = gu.float().requires_grad_(True)
    ref = torch.nn.functional.silu(x[:, :m]) * x[:, m:]
    assert rel(act, ref) < 1e-2
    dgu = torch.empty_like(gu)
    K.swiglu_bwd(dact, gu, dgu)
    ref.backward(dact.float())
    assert rel(dgu, x.grad) < 1e-2


def test_embedding_gather_scatter():
    from paper_2604_27085_b200 import kernels as K
    V, h, T = 1000, 256, 512
    table = rnd(V, h, seed=12)
    ids = torch.randint(0, V, (T,), device="cuda", dtype=torch.int32)
    out = torch.empty(T, h, device="cuda", dtype=torch.bfloat16)
    K.embed_fwd(ids, table, out)
    assert torch.equal(out, table[ids.long()])
    dx = rnd(T, h, seed=13, dtype=torch.float32)
    dE = torch.zeros(V, h, device="cuda")
    K.embed_bwd(ids, dx, dE)
    ref = torch.zeros(V, h, device="cuda").index_add_(0, ids.long(), dx)
    assert rel(dE, ref) < 1e-5


def test_embedding_gather_from_pinned_host():
    """Zero-copy gather: the table stays in pinned host memory."""
    from paper_2604_27085_b200 import kernels as K
    V, h, T = 4096, 512, 256
    table = torch.randn(V, h).to(torch.bfloat16).pin_memory()
    ids = torch.randint(0, V, (T,), device="cuda", dtype=torch.int32)
    out = torch.empty(T, h, device="cuda", dtype=torch.bfloat16)
    K.embed_fwd(ids, table, out)  # host pointer is device-accessible (UVA)
    torch.cuda.synchronize()
    assert torch.equal(out.cpu(), table[ids.long().cpu()])


@pytest.mark.parametrize("V", [32768, 151936, 1000])
def test_cross_entropy_inplace(V):
    from paper_2604_27085_b200 import kernels as K
    rows = 64
    z = rnd(rows, V, seed=14, scale=3.0)
    labels = torch.randint(0, V, (rows,), device="cuda", dtype=torch.int32)
    labels[3] = -100
    zf = z.float().requires_grad_(True)
    lref = torch.nn.functional.cross_entropy(zf, labels.long(), ignore_index=-100,
                                             reduction="sum")
    lref.backward()
    loss = torch.zeros(1, device="cuda")
    lse = torch.empty(rows, device="cuda")
    zz = z.clone()
    K.ce_fwd_bwd(zz, labels, 1.0, loss, lse)
    torch.cuda.synchronize()
    assert abs(loss.item() - lref.item()) / abs(lref.item()) < 1e-4
    assert rel(zz, zf.grad) < 1e-2


def test_adamw_chunk():
    from paper_2604_27085_b200 import kernels as K
    n = 1 << 20 | 3
    p = torch.randn(n, device="cuda")
    g = torch.randn(n, device="cuda")
    m = torch.randn(n, device="cuda") * 0.1
    v = torch.rand(n, device="cuda") * 0.1
    w16 = torch.empty(n, device="cuda", dtype=torch.bfloat16)
    pr, mr, vr = p.clone(), m.clone(), v.clone()
    lr, b1, b2, eps, wd, step = 3e-4, 0.9, 0.95, 1e-8, 0.1, 7
    K.adamw(p, m, v, g, w16, step, lr, b1, b2, eps, wd)
    mr = b1 * mr + (1 - b1) * g
    vr = b2 * vr + (1 - b2) * g * g
    upd = (mr / (1 - b1 ** step)) / ((vr / (1 - b2 ** step)).sqrt() + eps) + wd * pr
    pr = pr - lr * upd
    torch.cuda.synchronize()
    assert rel(m, mr) < 1e-6 and rel(v, vr) < 1e-6 and rel(p, pr) < 1e-6
    # the bf16 weights are the kernel's own fp32 master rounded (torch's fp32
    # result may differ in the last bit, which can flip a bf16 rounding)
    assert torch.equal(w16, p.to(torch.bfloat16))


def _attn_ref(q, k, v, seq, nq, nk, hd):
    T = q.shape[0]
    G = nq // nk
    qf = q.float().view(T // seq, seq, nq, hd).transpose(1, 2)
    kf = k.float().view(T // seq, seq, nk, hd).transpose(1, 2).repeat_interleave(G, 1)
    vf = v.float().view(T // seq, seq, nk, hd).transpose(1, 2).repeat_interleave(G, 1)
    s = qf @ kf.transpose(-1, -2) / math.sqrt(hd)
    mask = torch.ones(seq, seq, device="cuda", dtype=torch.bool).triu(1)
    s = s.masked_fill(mask, float("-inf"))
    lse = torch.logsumexp(s, -1)
    o = torch.softmax(s, -1) @ vf
    return o.transpose(1, 2).reshape(T, nq * hd), lse.permute(1, 0, 2).reshape(nq, T)


@pytest.mark.parametrize("T,seq,nq,nk,hd", [(256, 256, 4, 2, 64), (1024, 512, 8, 2, 128),
                                            (4096, 4096, 32, 8, 128), (512, 128, 4, 4, 64),
                                            (2048, 1024, 16, 4, 128), (768, 256, 6, 2, 128),
                                            (1024, 1024, 16, 2, 128), (2048, 2048, 32, 2, 128)])
def test_flash_attention_fwd_tcgen05(T, seq, nq, nk, hd):
    from paper_2604_27085_b200 import kernels as K
    qkv = rnd(T, (nq + 2 * nk) * hd, seed=30, scale=2.0)
    q = qkv[:, : nq * hd]
    k = qkv[:, nq * hd:(nq + nk) * hd]
    v = qkv[:, (nq + nk) * hd:]
    o = torch.empty(T, nq * hd, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(nq, T, device="cuda")
    K.attn_fwd_tc(q, k, v, o, lse, seq, nq, nk, hd)
    oref, lref = _attn_ref(q.float(), k.float(), v.float(), seq, nq, nk, hd)
    torch.cuda.synchronize()
    assert rel(o, oref) < 2e-2
    assert (lse - lref).abs().max().item() < 2e-2


@pytest.mark.parametrize("T,seq,nq,nk,hd", [(256, 256, 4, 2, 64), (1024, 512, 8, 2, 128),
                                            (4096, 4096, 32, 8, 128), (512, 128, 4, 4, 64),
                                            (2048, 1024, 16, 4, 128), (768, 256, 6, 2, 128),
                                            (1024, 1024, 16, 2, 128), (2048, 2048, 32, 2, 128)])
def test_flash_attention_bwd_tcgen05(T, seq, nq, nk, hd):
    from paper_2604_27085_b200 import kernels as K
    qkv = rnd(T, (nq + 2 * nk) * hd, seed=40, scale=1.5)
    q = qkv[:, : nq * hd]
    k = qkv[:, nq * hd:(nq + nk) * hd]
    v = qkv[:, (nq + nk) * hd:]
    o = torch.empty(T, nq * hd, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(nq, T, device="cuda")
    K.attn_fwd_tc(q, k, v, o, lse, seq, nq, nk, hd)
    qf = q.float().requires_grad_(True)
    kf = k.float().requires_grad_(True)
    vf = v.float().requires_grad_(True)
    oref, _ = _attn_ref(qf, kf, vf, seq, nq, nk, hd)
    do = rnd(T, nq * hd, seed=41)
    oref.backward(do.float())
    dqkv = torch.zeros_like(qkv)
    dq, dk, dv = dqkv[:, : nq * hd], dqkv[:, nq * hd:(nq + nk) * hd], dqkv[:, (nq + nk) * hd:]
    delta = torch.empty(nq, T, device="cuda")
    K.attn_bwd_tc(q, k, v, o, do, lse, dq, dk, dv, delta, seq, nq, nk, hd)
    torch.cuda.synchronize()
    assert rel(dq, qf.grad) < 2e-2
    assert rel(dk, kf.grad) < 2e-2
    assert rel(dv, vf.grad) < 2e-2
