"""Step parity at full Qwen3-8B width against the fp32 CPU oracle.

The headline's code paths at the headline's shapes (VERDICT r01 "next" #1):
model `qwen3-8b-l2` = 2 decoder layers at full Qwen3-8B width (h4096,
a32/k8 -> GQA group 4, hd128, m12288, V151936), seq 4096, M=2 micro-batches,
so every step runs
  * the two-chunk LM head (2 x [2048, 151936] logits chunks, wgrad
    accumulated across chunks),
  * the G=4 fused attention backward (2-CTA cluster, DSMEM dK/dV reduction),
  * split-K / N-split last waves of the 8B GEMM shapes,
  * fused SwiGLU epilogues (T >= 256),
in three placements:
  * N=1 mixed: resident_state_gb=10 -> the embedding's and layer 0's fp32
    AdamW state in HBM (direct publication), the LM head's and layer 1's
    streamed through pinned host memory;
  * N=1 streamed: all state host-offloaded (BASELINE configs[2]);
  * N=2 logical workers with a uniform cost table -> S=4 (fwd [0..1], fused
    [head], bwd [1], [0]): hand-offs, checkpoints and recompute at 8B width.
Sync and async (staleness-1) modes, 3 steps each.

Tolerances (bf16 compute vs fp32 oracle, AdamW lr 1e-4):
  loss rel <= 2e-3 every step; step-0 grads per weight MATRIX rel-L2 <= 2e-2,
  per 1-D norm-weight vector (q_norm / k_norm / RMSNorm weights: sums over
  T x heads bf16 products) rel-L2 <= 3e-2, cosine >= 0.999 for every tensor;
  fp32 master after 3 steps rel-L2 <= 3e-3 and update cosine >= 0.98 for
  every weight matrix. Measured (profiles/r02_parity_margins.txt): loss rel
  <= 4.7e-4, k_norm grad 2.3e-2, master <= 1.5e-3, update cosine >= 0.985.
"""
import numpy as np
import pytest
import torch

from oracle import step_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, scope="module")
def _free_module_caches():
    """The driver runs every GPU file in one pytest process: drop this
    module's multi-GB parameter / oracle caches once its tests are done."""
    yield
    _PARAMS.clear()
    _ORACLE.clear()
MODEL = "qwen3-8b-l2"
HP = dict(lr=1e-4, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.0)
M, SEQ, STEPS = 2, 4096, 3

_ORACLE = {}
_PARAMS = {}


def shape():
    return O.Shape.from_config(MODEL)


def params():
    if "p" not in _PARAMS:
        _PARAMS["p"] = O.init_params(shape(), seed=0)
    return _PARAMS["p"]


def batch():
    return O.synthetic_batch(shape(), M, 1, SEQ)


def oracle(mode):
    """fp32 CPU oracle run (all host cores), cached per mode."""
    if mode not in _ORACLE:
        torch.set_num_threads(max(1, torch.get_num_threads()))
        o = O.StepOracle(shape(), params(), mode=mode, **HP)
        tok, lab = batch()
        losses, g0 = [], None
        for it in range(STEPS):
            losses.append(o.step(tok, lab))
            if it == 0:
                g0 = o.last_grads
        _ORACLE[mode] = (losses, g0, o.master_fp32())
        del o
    return _ORACLE[mode]


def uniform_costs(L1):
    from paper_2604_27085_b200.planner import COST_DTYPE
    c = np.zeros(L1, dtype=COST_DTYPE)
    c["t_fwd_ns"], c["t_bwd_ns"], c["param_bytes"] = 1000, 3000, 1
    c["act_ckpt_bytes"] = 1
    return c


def run(mode, N, **kw):
    from paper_2604_27085_b200.runtime import AdamW, RoundPipe
    s = shape()
    tok, lab = batch()
    rt = RoundPipe(MODEL, seq_len=SEQ, micro_batch=1, micro_batches=M, num_gpus=N,
                   async_optimizer=(mode == "async"),
                   adam=AdamW(HP["lr"], HP["betas"], HP["eps"], HP["weight_decay"]),
                   skip_init=True, **kw)
    rt.load_state({k: v.numpy() for k, v in params().items()}, s.layers)
    losses, g0 = [], None
    for it in range(STEPS):
        losses.append(rt.forward_backward(tok.numpy(), lab.numpy()))
        if it == 0:
            g0 = rt.read_state(s.layers, which=2)
        rt.step()
    rt.sync()
    master = rt.read_state(s.layers, which=0)
    plan = rt.plan()[0]
    st = rt.stats()
    rt.close()
    return losses, g0, master, plan, st


def compare(tag, mode, losses, g0, master):
    ol, og, om = oracle(mode)
    loss_rel = [abs(a - b) / abs(b) for a, b in zip(losses, ol)]
    grel, gcos, vrel = {}, {}, {}
    for k, ref in og.items():
        rn = ref.norm().item()
        if rn < 1e-6:
            continue
        g = torch.from_numpy(np.asarray(g0[k])).reshape(ref.shape)
        (grel if ref.dim() == 2 else vrel)[k] = (g - ref).norm().item() / rn
        gcos[k] = torch.nn.functional.cosine_similarity(g.flatten(), ref.flatten(), dim=0).item()
    init = params()
    mrel, mcos = {}, {}
    for k, ref in om.items():
        w = torch.from_numpy(np.asarray(master[k])).reshape(ref.shape)
        mrel[k] = (w - ref).norm().item() / ref.norm().item()
        if ref.dim() == 2:
            du, dr = (w - init[k]).flatten(), (ref - init[k]).flatten()
            mcos[k] = torch.nn.functional.cosine_similarity(du, dr, dim=0).item()
    wg = max(grel.items(), key=lambda kv: kv[1])
    wv = max(vrel.items(), key=lambda kv: kv[1])
    wc = min(gcos.items(), key=lambda kv: kv[1])
    wm = max(mrel.items(), key=lambda kv: kv[1])
    wu = min(mcos.items(), key=lambda kv: kv[1])
    print(f"MARGINS {tag} {mode}: losses {losses} oracle {ol} max loss rel {max(loss_rel):.2e}; "
          f"worst matrix grad rel-L2 {wg[0]} {wg[1]:.3e}; worst vector grad rel-L2 {wv[0]} "
          f"{wv[1]:.3e}; worst grad cos {wc[0]} {wc[1]:.6f}; "
          f"worst master rel-L2 {wm[0]} {wm[1]:.3e}; worst update cos {wu[0]} {wu[1]:.5f}")
    assert max(loss_rel) < 2e-3, (losses, ol)
    assert wg[1] < 2e-2 and wv[1] < 3e-2 and wc[1] > 0.999, (wg, wv, wc)
    assert wm[1] < 3e-3, wm
    assert wu[1] > 0.98, wu


@pytest.mark.parametrize("mode", ["sync", "async"])
def test_8b_width_n1_mixed_placement(mode):
    losses, g0, master, plan, st = run(mode, 1, resident_state_gb=10.0)
    assert plan.num_slots() == 1
    s = shape()
    total = sum(np.asarray(v).size for v in master.values())
    assert 0 < st["resident_params"] < total, st["resident_params"]  # mixed placement
    compare("n1-mixed", mode, losses, g0, master)


@pytest.mark.parametrize("mode", ["sync", "async"])
def test_8b_width_n1_host_offloaded(mode):
    losses, g0, master, plan, st = run(mode, 1, resident_state_gb=0.0)
    assert st["resident_params"] == 0
    compare("n1-host", mode, losses, g0, master)


@pytest.mark.parametrize("mode", ["sync", "async"])
def test_8b_width_n2_four_slots(mode):
    losses, g0, master, plan, st = run(mode, 2, costs=uniform_costs(shape().layers + 1))
    assert plan.num_slots() == 4 and [(r.first, r.last) for r in plan.bwd_stages] == [(1, 1), (0, 0)]
    compare("n2-S4", mode, losses, g0, master)


def test_8b_width_lora_r32():
    """LoRA r=32 / alpha 64 on the four linears at full Qwen3-8B width, N=1,
    async, host-offloaded adapter state: the adapter GEMMs at real shapes —
    the rank-side pair-kernel path of dU = dY B over K = 24576 (gate/up),
    the 128x32 skinny tiles, the swapped M <= 32 adapter gradients — plus the
    second-K-segment base GEMMs. Loss rel <= 2e-3 every step, adapter grads
    rel-L2 <= 2e-2 and cosine >= 0.999, adapter update cosine >= 0.98,
    frozen base bit-unchanged."""
    from paper_2604_27085_b200.runtime import AdamW, RoundPipe
    r, alpha, mode = 32, 64.0, "async"
    s = shape()
    p = dict(params())
    p.update(O.init_lora_params(s, r, seed=1, std_b=0.02))
    tok, lab = batch()
    rt = RoundPipe(MODEL, seq_len=SEQ, micro_batch=1, micro_batches=M, num_gpus=1,
                   async_optimizer=True,
                   adam=AdamW(HP["lr"], HP["betas"], HP["eps"], HP["weight_decay"]),
                   skip_init=True, lora_rank=r, lora_alpha=alpha, resident_state_gb=0.0)
    rt.load_state({k: v.numpy() for k, v in p.items()}, s.layers)
    keys = [f"layers.{l}.{n}" for l in range(s.layers)
            for n in ("qkv_lora_A", "qkv_lora_B", "o_lora_A", "o_lora_B", "gate_up_lora_A",
                      "gate_up_lora_B", "down_lora_A", "down_lora_B")]
    losses = []
    for it in range(STEPS):
        losses.append(rt.forward_backward(tok.numpy(), lab.numpy()))
        if it == 0:
            g0 = rt.read_state(s.layers, which=2)
            g0 = {k: np.asarray(g0[k]).copy() for k in keys}
        rt.step()
    rt.sync()
    w = rt.read_state(s.layers, which=1)
    w = {k: np.asarray(w[k]).copy() for k in ("layers.0.qkv", "layers.1.down", "head.lm_head")}
    m = rt.read_state(s.layers, which=0)
    m = {k: np.asarray(m[k]).copy() for k in keys}
    rt.close()
    torch.set_num_threads(max(1, torch.get_num_threads()))
    o = O.StepOracle(s, p, mode=mode, lora_scale=alpha / r, **HP)
    ol = []
    for it in range(STEPS):
        ol.append(o.step(tok, lab))
        if it == 0:
            og = {k: o.last_grads[k] for k in keys}
    om = o.master_fp32()
    loss_rel = max(abs(a - b) / abs(b) for a, b in zip(losses, ol))
    grel, gcos, ucos = {}, {}, {}
    for k in keys:
        g = torch.from_numpy(g0[k]).reshape(og[k].shape)
        grel[k] = ((g - og[k]).norm() / og[k].norm()).item()
        gcos[k] = torch.nn.functional.cosine_similarity(g.flatten(), og[k].flatten(), dim=0).item()
        du = torch.from_numpy(m[k]).reshape(om[k].shape) - p[k]
        dr = om[k] - p[k]
        ucos[k] = float((du * dr).sum() / (du.norm() * dr.norm()))
    wg = max(grel.items(), key=lambda kv: kv[1])
    wc = min(gcos.items(), key=lambda kv: kv[1])
    wu = min(ucos.items(), key=lambda kv: kv[1])
    print(f"MARGINS lora-r32 {mode}: losses {losses} oracle {ol} max loss rel {loss_rel:.2e}; "
          f"worst adapter grad rel-L2 {wg[0]} {wg[1]:.3e}; worst grad cos {wc[0]} {wc[1]:.6f}; "
          f"worst update cos {wu[0]} {wu[1]:.5f}")
    assert loss_rel < 2e-3, (losses, ol)
    assert wg[1] < 2e-2 and wc[1] > 0.999, (wg, wc)
    assert wu[1] > 0.98, wu
    for k, v in w.items():  # frozen base
        assert np.array_equal(v.reshape(-1), p[k].numpy().reshape(-1)), k
