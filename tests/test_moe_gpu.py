"""Mixture-of-experts kernels (csrc/kernels/moe.cu + rp_gemm_grouped) vs a plain
PyTorch fp32 autograd restatement of transformers' Qwen3-MoE sparse block
(modeling_qwen3_moe.py:215-287: softmax router in fp32, top-k, optional
renormalisation, SwiGLU experts, weighted sum).

One MoE MLP forward and backward (experts and router frozen; the input
gradient includes the router path) runs through the C-ABI kernels:
router GEMM -> route -> permute -> grouped gate/up GEMM -> SwiGLU ->
grouped down GEMM -> combine; gather -> grouped down dgrad -> SwiGLU
backward with dw -> grouped gate/up dgrad -> router backward -> router
dgrad GEMM -> combine backward. Tolerances: routing exact (same experts per
token as torch.topk on the fp32 softmax); outputs (bf16 intermediates)
rel-L2 <= 1e-2; input gradient rel-L2 <= 2e-2; per-slot dw rel-L2 <= 2e-2.
"""
import pytest
import torch

pytestmark = pytest.mark.gpu


def rel(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm().clamp_min(1e-30)).item()


def rnd(*shape, seed=0, scale=1.0, dtype=torch.bfloat16):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.randn(*shape, device="cuda", generator=g) * scale).to(dtype)


def _reference(x, Wg, Wgu, Wd, res, k, norm, dY):
    """fp32 autograd restatement; returns out, dx, topk indices, dw [T, k]."""
    xr = x.float().requires_grad_(True)
    logits = xr @ Wg.float().T
    p = torch.softmax(logits, dim=-1)
    topv, topi = torch.topk(p, k, dim=-1)
    w = topv / topv.sum(-1, keepdim=True) if norm else topv
    w.retain_grad()
    T, h = x.shape
    m = Wd.shape[2]
    y = torch.zeros(T, h, device="cuda")
    for e in range(Wg.shape[0]):
        tok, slot = torch.where(topi == e)
        if tok.numel() == 0:
            continue
        gu = xr[tok] @ Wgu[e].float().T
        act = torch.nn.functional.silu(gu[:, :m]) * gu[:, m:]
        y = y.index_add(0, tok, (act @ Wd[e].float().T) * w[tok, slot, None])
    out = res.float() + y
    out.backward(dY.float())
    return out.detach(), xr.grad, topi, w.grad


@pytest.mark.parametrize("T,h,m,E,k,norm", [(256, 256, 128, 8, 2, True), (200, 512, 256, 16, 4, False),
                                            (1024, 1024, 256, 64, 8, True)])
def test_moe_mlp_fwd_bwd(T, h, m, E, k, norm):
    from paper_2604_27085_b200 import kernels as K
    x = rnd(T, h, seed=1)
    Wg = rnd(E, h, seed=2, scale=0.1)
    Wgu = rnd(E, 2 * m, h, seed=3, scale=0.05)
    Wd = rnd(E, h, m, seed=4, scale=0.05)
    res = rnd(T, h, seed=5)
    dY = rnd(T, h, seed=6)
    dev = dict(device="cuda")
    # ---- forward
    logits = torch.empty(T, E, dtype=torch.float32, **dev)
    K.gemm(x, Wg, logits)
    idx = torch.empty(T, k, dtype=torch.int32, **dev)
    w = torch.empty(T, k, dtype=torch.float32, **dev)
    counts = torch.empty(E, dtype=torch.int32, **dev)
    K.moe_route(logits, k, norm, idx, w, counts)
    offsets = torch.empty(E + 1, dtype=torch.int32, **dev)
    cursor = torch.empty(E, dtype=torch.int32, **dev)
    pos = torch.empty(T, k, dtype=torch.int32, **dev)
    w_s = torch.empty(T * k, dtype=torch.float32, **dev)
    xs = torch.empty(T * k, h, dtype=torch.bfloat16, **dev)
    K.moe_permute(x, k, idx, w, counts, offsets, cursor, pos, w_s, xs)
    gu_s = torch.empty(T * k, 2 * m, dtype=torch.bfloat16, **dev)
    K.gemm_grouped(xs, Wgu.view(E * 2 * m, h), gu_s, offsets, E, 2 * m)
    act_s = torch.empty(T * k, m, dtype=torch.bfloat16, **dev)
    K.swiglu_fwd(gu_s, act_s)
    ys = torch.empty(T * k, h, dtype=torch.bfloat16, **dev)
    K.gemm_grouped(act_s, Wd.view(E * h, m), ys, offsets, E, h)
    out = torch.empty(T, h, dtype=torch.bfloat16, **dev)
    K.moe_combine(ys, pos, w, k, out, res=res)
    # ---- backward
    dys = torch.empty(T * k, h, dtype=torch.bfloat16, **dev)
    K.moe_gather(dY, k, pos, dys)
    dact = torch.empty(T * k, m, dtype=torch.bfloat16, **dev)
    K.gemm_grouped(dys, Wd.view(E * h, m), dact, offsets, E, h, b_mn_major=True)
    dgu = torch.empty(T * k, 2 * m, dtype=torch.bfloat16, **dev)
    dw_s = torch.empty(T * k, dtype=torch.float32, **dev)
    K.moe_swiglu_bwd(dact, gu_s, w_s, dgu, dw_s)
    dxs = torch.empty(T * k, h, dtype=torch.bfloat16, **dev)
    K.gemm_grouped(dgu, Wgu.view(E * 2 * m, h), dxs, offsets, E, 2 * m, b_mn_major=True)
    dlog = torch.empty(T, E, dtype=torch.bfloat16, **dev)
    K.moe_router_bwd(logits, k, norm, idx, pos, dw_s, dlog)
    dh32 = torch.empty(T, h, dtype=torch.float32, **dev)
    K.gemm(dlog, Wg, dh32, b_mn_major=True)
    dh = torch.empty(T, h, dtype=torch.bfloat16, **dev)
    K.moe_combine_bwd(dxs, pos, k, dh32, dh)
    torch.cuda.synchronize()

    out_r, dx_r, topi_r, dw_r = _reference(x, Wg, Wgu, Wd, res, k, norm, dY)
    # routing: same expert set per token (slot order may differ only on ties)
    assert torch.equal(idx.long().sort(-1).values, topi_r.sort(-1).values)
    # permutation: offsets = exclusive scan of counts, every slot gets a distinct row
    cnt_r = torch.bincount(topi_r.flatten(), minlength=E)
    assert torch.equal(counts.long().cpu(), cnt_r.cpu())
    assert torch.equal(offsets[1:].long().cpu(), cnt_r.cumsum(0).cpu())
    assert torch.equal(pos.flatten().sort().values.cpu(), torch.arange(T * k, dtype=torch.int32))
    assert torch.equal(xs[pos.flatten().long()], x.repeat_interleave(k, 0))
    assert rel(out, out_r) < 1e-2
    assert rel(dh, dx_r) < 2e-2
    # per-slot dL/dw (match slots by expert id)
    order = idx.long().argsort(-1)
    dw_k = dw_s[pos.long()].gather(1, order)
    dw_ref = dw_r.gather(1, topi_r.argsort(-1))
    assert rel(dw_k, dw_ref) < 2e-2


def test_grouped_gemm_ragged_and_empty_groups():
    """Empty experts, a single-row expert and >128-row experts in one launch;
    rows of other experts untouched; K-major and MN-major B."""
    from paper_2604_27085_b200 import kernels as K
    E, N, Kd = 6, 384, 320
    sizes = [0, 1, 130, 0, 257, 40]
    off = torch.tensor([0] + list(torch.tensor(sizes).cumsum(0)), dtype=torch.int32, device="cuda")
    M = sum(sizes)
    A = rnd(M, Kd, seed=11)
    B = rnd(E, N, Kd, seed=12, scale=0.1)
    D = torch.full((M, N), 7.0, dtype=torch.bfloat16, device="cuda")
    K.gemm_grouped(A, B.view(E * N, Kd), D, off, E, N)
    Bt = B.transpose(1, 2).contiguous()  # [E, K, N]: MN-major blocks
    D2 = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    K.gemm_grouped(A, Bt.view(E * Kd, N), D2, off, E, Kd, b_mn_major=True)
    torch.cuda.synchronize()
    ref = torch.empty(M, N, device="cuda")
    r0 = 0
    for e, n in enumerate(sizes):
        ref[r0:r0 + n] = A[r0:r0 + n].float() @ B[e].float().T
        r0 += n
    assert rel(D, ref) < 1e-2
    assert rel(D2, ref) < 1e-2
