"""Sensitivity of LoRA adapter grads to bf16-level changes of the router
input in a Qwen3-MoE layer with E=128, k=8 (random init)."""
import sys, dataclasses
sys.path.insert(0, ".")
import torch
from oracle import step_oracle as O
torch.set_num_threads(8)
base = O.Shape.from_config("qwen3-235b-a22b")
s = dataclasses.replace(base, hidden=1024, heads=16, kv_heads=1, head_dim=64, inter=384,
                        layers=1, vocab=8192)
r, alpha = 16, 32.0
p = O.init_params(s, seed=0)
p.update(O.init_lora_params(s, r, seed=1, std_b=0.02))
tok, lab = O.synthetic_batch(s, 1, 1, 2048)

def grads(perturb):
    orig = O.moe_route
    def route(hs, router, sh):
        if perturb == "bf16":
            hs = hs.to(torch.bfloat16).float()
        elif perturb == "noise":
            hs = hs * (1 + 2.0 ** -9 * torch.randn_like(hs))
        return orig(hs, router, sh)
    O.moe_route = route
    try:
        o = O.StepOracle(s, p, mode="sync", lora_scale=alpha / r, lr=1e-3)
        loss = o.step(tok, lab)
        return loss, o.last_grads
    finally:
        O.moe_route = orig

l0, g0 = grads(None)
for pert in ("bf16", "noise"):
    l1, g1 = grads(pert)
    out = {}
    for n in ("qkv_lora_A", "qkv_lora_B", "o_lora_A", "o_lora_B"):
        k = f"layers.0.{n}"
        out[n] = round(((g1[k] - g0[k]).norm() / g0[k].norm()).item(), 4)
    print(pert, "loss rel", abs(l1 - l0) / l0, "grad rel-L2", out, flush=True)
