"""Step parity of the C5 path at FULL Qwen3-235B-A22B width against the fp32
CPU oracle (the tiny-moe suite covers the logic; this one the real shapes).

Model `qwen3-235b-a22b-l1`: one Qwen3-MoE decoder layer at full width
(h4096, 64 query / 4 KV heads -> GQA group 16, hd128, 128 experts of
moe_intermediate 1536, top-8 renormalised routing) + embedding + LM head
(V151936); LoRA r=16 / alpha 32 on the attention projections, experts,
router and every other base weight frozen and streamed (the C5 setting);
seq 2048, M=2 micro-batches. Every step runs
  * the grouped expert GEMMs over 128 experts with device-side row offsets
    (16,384 routed rows per micro-batch),
  * router softmax / top-8 / renormalisation and its backward,
  * the G=16 attention backward (fp32-atomic dK/dV reduction),
  * the long-K LoRA adapter-gradient GEMMs,
in sync and async (staleness-1) mode, N=1, 3 steps each (the recompute
path of MoE layers in backward slots is covered at tiny-moe width by
tests/test_runtime_moe_gpu.py: with one layer the partitioner keeps it in
the fused stage).

Tolerances (bf16 compute vs fp32 oracle): loss rel <= 2e-3 every step;
adapters' AdamW update cosine >= 0.97 after 3 steps; frozen base
bit-unchanged; step-0 adapter grads: rel-L2 <= max(3e-2, 2.5 x the oracle's
own routing spread) and cosine >= 0.995. The routing spread is measured in
the test: the same fp32 oracle with its router input rounded to bf16 (what
a bf16 model computes anyway) changes the adapter grads by ~4 % (random
init: the top-8 of 128 near-uniform router probabilities flips for some
tokens under bf16-level input changes; a CPU experiment at h1024 gave
3.6-4.1 %), and the GPU (bf16 activations) sits at that level (~6 % at
h4096, cosine 0.998).
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
    _P.clear()
    _ORACLE.clear()
MODEL = "qwen3-235b-a22b-l1"
HP = dict(lr=1e-3, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.0)
R, ALPHA, M, SEQ, STEPS = 16, 32.0, 2, 2048, 3
_P = {}
_ORACLE = {}


def params():
    if "p" not in _P:
        s = O.Shape.from_config(MODEL)
        p = O.init_params(s, seed=0)
        p.update(O.init_lora_params(s, R, seed=1, std_b=0.02))
        _P["p"] = p
    return _P["p"]


def uniform_costs(L1):
    from paper_2604_27085_b200.planner import COST_DTYPE
    c = np.zeros(L1, dtype=COST_DTYPE)
    c["t_fwd_ns"], c["t_bwd_ns"], c["param_bytes"] = 1000, 3000, 1
    c["act_ckpt_bytes"] = 1
    return c


KEYS = [f"layers.0.{n}" for n in ("qkv_lora_A", "qkv_lora_B", "o_lora_A", "o_lora_B")]


def oracle(mode, s, p, tok, lab):
    """fp32 oracle (3 steps) and its routing spread, cached per mode."""
    if mode not in _ORACLE:
        torch.set_num_threads(max(1, torch.get_num_threads()))
        o = O.StepOracle(s, p, mode=mode, lora_scale=ALPHA / R, **HP)
        ref = []
        for it in range(STEPS):
            ref.append(o.step(tok, lab))
            if it == 0:
                ref_g = {k: o.last_grads[k] for k in KEYS}
        om = o.master_fp32()
        om = {k: om[k] for k in KEYS}
        del o
        # the oracle's own routing spread: router input rounded to bf16
        route = O.moe_route
        O.moe_route = lambda hs, router, sh: route(hs.to(torch.bfloat16).float(), router, sh)
        try:
            o2 = O.StepOracle(s, p, mode=mode, lora_scale=ALPHA / R, **HP)
            o2.step(tok, lab)
            alt_g = {k: o2.last_grads[k] for k in KEYS}
            del o2
        finally:
            O.moe_route = route
        _ORACLE[mode] = (ref, ref_g, om, alt_g)
    return _ORACLE[mode]


@pytest.mark.parametrize("mode,N", [("sync", 1), ("async", 1)])
def test_moe_lora_step_parity_full_width(mode, N):
    from paper_2604_27085_b200.runtime import AdamW, RoundPipe
    s = O.Shape.from_config(MODEL)
    p = params()
    tok, lab = O.synthetic_batch(s, M, 1, SEQ)
    rt = RoundPipe(MODEL, seq_len=SEQ, micro_batch=1, micro_batches=M, num_gpus=N,
                   async_optimizer=(mode == "async"),
                   adam=AdamW(HP["lr"], HP["betas"], HP["eps"], HP["weight_decay"]),
                   costs=uniform_costs(s.layers + 1) if N > 1 else None,
                   skip_init=True, lora_rank=R, lora_alpha=ALPHA)
    assert rt.moe
    rt.load_state({k: v.numpy() for k, v in p.items()}, s.layers)
    got = []
    for it in range(STEPS):
        got.append(rt.forward_backward(tok.numpy(), lab.numpy()))
        if it == 0:
            g0 = rt.read_state(s.layers, which=2)
            g0 = {k: np.asarray(g0[k]).copy() for k in KEYS}
        rt.step()
    rt.sync()
    w = rt.read_state(s.layers, which=1)
    w = {k: np.asarray(w[k]).copy() for k in
         [f"layers.0.{n}" for n in ("router", "gate_up", "down", "qkv", "o")]}
    m = rt.read_state(s.layers, which=0)
    m = {k: np.asarray(m[k]).copy() for k in KEYS}
    rt.close()
    ref, ref_g, om, alt_g = oracle(mode, s, p, tok, lab)
    rels, coss, gcos, spread = {}, {}, {}, {}
    for k in KEYS:
        a = torch.from_numpy(g0[k]).reshape(ref_g[k].shape)
        rels[k] = ((a - ref_g[k]).norm() / ref_g[k].norm()).item()
        spread[k] = ((alt_g[k] - ref_g[k]).norm() / ref_g[k].norm()).item()
        gcos[k] = torch.nn.functional.cosine_similarity(a.flatten(), ref_g[k].flatten(), dim=0).item()
        du = torch.from_numpy(m[k]).reshape(om[k].shape) - p[k]
        dr = om[k] - p[k]
        coss[k] = float((du * dr).sum() / (du.norm() * dr.norm()))
    loss_rel = max(abs(a - b) / b for a, b in zip(got, ref))
    print(f"MARGINS 235b-width moe N={N} {mode}: losses {got} oracle {ref} max loss rel "
          f"{loss_rel:.2e}; adapter grad rel-L2 {rels}; oracle routing spread {spread}; "
          f"grad cos {gcos}; update cos {coss}")
    assert loss_rel < 2e-3, (got, ref)
    for k in KEYS:
        assert rels[k] < max(3e-2, 2.5 * spread[k]) and gcos[k] > 0.995, (k, rels[k], spread[k])
        assert coss[k] > 0.97, (k, coss[k])
    for k, v in w.items():  # frozen base
        assert np.array_equal(v.reshape(-1), p[k].numpy().reshape(-1)), k
