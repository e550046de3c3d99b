"""MoE path of BASELINE configs[4] (Qwen3-235B-A22B LoRA fine-tune) end to
end on the GPU at the tiny-moe parity config (2 Qwen3-MoE layers, h256,
8 experts of moe_intermediate 128, 2 routed per token, renormalised top-k;
32K vocab; seq 256, M=2): LoRA rank 16 / alpha 32 on the attention
projections, experts, router and every other base weight frozen and
streamed — vs the fp32 oracle (oracle/step_oracle.py moe_block, pinned to
transformers' Qwen3MoeForCausalLM in tests/golden/moe_golden.json).

N=1 runs the single fused stage; N=2 logical workers with a uniform cost
table split the model so MoE layers are recomputed in backward slots (their
routing is recomputed from the checkpoint). Tolerances: loss rel <= 2e-3 per
step; adapter grads rel-L2 <= 3e-2 (bf16 compute, fp32 oracle); adapters'
AdamW update cosine >= 0.98 after 3 steps; frozen base bit-unchanged.
"""
import numpy as np
import pytest
import torch

from oracle import step_oracle as O

pytestmark = pytest.mark.gpu
HP = dict(lr=1e-3, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.0)


def uniform_costs(L1):
    from paper_2604_27085_b200.planner import COST_DTYPE
    c = np.zeros(L1, dtype=COST_DTYPE)
    c["t_fwd_ns"], c["t_bwd_ns"], c["param_bytes"] = 1000, 3000, 1
    c["act_ckpt_bytes"] = 1
    return c


@pytest.mark.parametrize("N,mode", [(1, "sync"), (1, "async"), (2, "sync")])
def test_moe_lora_step_parity(N, mode):
    from paper_2604_27085_b200.runtime import AdamW, RoundPipe
    s = O.Shape.from_config("tiny-moe")
    r, alpha = 16, 32.0
    params = O.init_params(s, seed=0)
    params.update(O.init_lora_params(s, r, seed=1, std_b=0.02))
    tok, lab = O.synthetic_batch(s, 2, 1, 256)
    rt = RoundPipe("tiny-moe", seq_len=256, micro_batch=1, micro_batches=2, num_gpus=N,
                   async_optimizer=(mode == "async"),
                   adam=AdamW(HP["lr"], HP["betas"], HP["eps"], HP["weight_decay"]),
                   costs=uniform_costs(s.layers + 1) if N > 1 else None, skip_init=True,
                   lora_rank=r, lora_alpha=alpha)
    assert rt.moe
    if N > 1:
        plan, _ = rt.plan()
        assert len(plan.bwd_stages) >= 1  # MoE layers recomputed in backward slots
    rt.load_state({k: v.numpy() for k, v in params.items()}, s.layers)
    o = O.StepOracle(s, params, mode=mode, lora_scale=alpha / r, **HP)
    got, ref = [], []
    for it in range(3):
        got.append(rt.forward_backward(tok.numpy(), lab.numpy()))
        if it == 0:
            g0 = rt.read_state(s.layers, which=2)
        rt.step()
        ref.append(o.step(tok, lab))
        if it == 0:
            ref_g = o.last_grads
    rt.sync()
    w = rt.read_state(s.layers, which=1)
    m = rt.read_state(s.layers, which=0)
    rt.close()
    print(f"MARGINS moe N={N} {mode}: losses {got} oracle {ref}")
    for a, b in zip(got, ref):
        assert abs(a - b) / b < 2e-3, (got, ref)
    om = o.master_fp32()
    worst = 0.0
    for l in range(s.layers):
        for n in ("qkv_lora_A", "qkv_lora_B", "o_lora_A", "o_lora_B"):
            k = f"layers.{l}.{n}"
            a = torch.from_numpy(np.asarray(g0[k])).reshape(ref_g[k].shape)
            rel = ((a - ref_g[k]).norm() / ref_g[k].norm()).item()
            worst = max(worst, rel)
            assert rel < 3e-2, (k, rel)
            du = torch.from_numpy(np.asarray(m[k])).reshape(om[k].shape) - params[k]
            dr = om[k] - params[k]
            cos = float((du * dr).sum() / (du.norm() * dr.norm()))
            assert cos > 0.98, (k, cos)
        for n in ("router", "gate_up", "down", "qkv"):  # frozen base
            k = f"layers.{l}.{n}"
            assert np.array_equal(np.asarray(w[k]).reshape(-1), params[k].numpy().reshape(-1)), k
    print(f"MARGINS moe N={N} {mode}: worst adapter grad rel-L2 {worst:.3e}")
