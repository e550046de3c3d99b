"""Pin the oracle's Qwen3-MoE layer (oracle/step_oracle.py moe_block) against
transformers' Qwen3MoeForCausalLM (third-party, transformers 5.5.0) on
identical fp32 weights for the tiny-moe config, and commit the numbers plus
the oracle's LoRA step trajectory (attention adapters; experts and router
frozen) to tests/golden/moe_golden.json.

Run: python tests/golden/make_moe_golden.py   (CPU, ~30 s)
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import step_oracle as O  # noqa: E402

M, SEQ, STEPS, RANK = 2, 256, 3, 16
HP = dict(lr=1e-3, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.0)


def hf_moe(s, params):
    from transformers import Qwen3MoeConfig, Qwen3MoeForCausalLM
    cfg = Qwen3MoeConfig(vocab_size=s.vocab, hidden_size=s.hidden, moe_intermediate_size=s.inter,
                         intermediate_size=4 * s.inter, num_hidden_layers=s.layers,
                         num_attention_heads=s.heads, num_key_value_heads=s.kv_heads,
                         head_dim=s.head_dim, rope_theta=s.rope_theta, rms_norm_eps=s.eps,
                         num_experts=s.experts, num_experts_per_tok=s.active,
                         norm_topk_prob=s.norm_topk, decoder_sparse_step=1, mlp_only_layers=[],
                         tie_word_embeddings=False, max_position_embeddings=4096,
                         attention_bias=False, output_router_logits=False)
    cfg._attn_implementation = "eager"
    m = Qwen3MoeForCausalLM(cfg).float()
    qd, kd = s.heads * s.head_dim, s.kv_heads * s.head_dim
    sd = {"model.embed_tokens.weight": params["embed"],
          "model.norm.weight": params["head.final_norm"],
          "lm_head.weight": params["head.lm_head"]}
    for l in range(s.layers):
        p = lambda n: params[f"layers.{l}.{n}"]  # noqa: E731
        pre = f"model.layers.{l}."
        sd[pre + "input_layernorm.weight"] = p("input_norm")
        sd[pre + "self_attn.q_proj.weight"] = p("qkv")[:qd]
        sd[pre + "self_attn.k_proj.weight"] = p("qkv")[qd:qd + kd]
        sd[pre + "self_attn.v_proj.weight"] = p("qkv")[qd + kd:]
        sd[pre + "self_attn.q_norm.weight"] = p("q_norm")
        sd[pre + "self_attn.k_norm.weight"] = p("k_norm")
        sd[pre + "self_attn.o_proj.weight"] = p("o")
        sd[pre + "post_attention_layernorm.weight"] = p("post_norm")
        sd[pre + "mlp.gate.weight"] = p("router")
        sd[pre + "mlp.experts.gate_up_proj"] = p("gate_up").view(s.experts, 2 * s.inter, s.hidden)
        sd[pre + "mlp.experts.down_proj"] = p("down").view(s.experts, s.hidden, s.inter)
    missing, unexpected = m.load_state_dict(sd, strict=False)
    assert not unexpected and all("rotary" in k for k in missing), (missing, unexpected)
    return m


def hf_grads(m, s):
    qd, kd = s.heads * s.head_dim, s.kv_heads * s.head_dim
    g = {n: p.grad for n, p in m.named_parameters()}
    out = {"embed": g["model.embed_tokens.weight"], "head.final_norm": g["model.norm.weight"],
           "head.lm_head": g["lm_head.weight"]}
    for l in range(s.layers):
        pre = f"model.layers.{l}."
        out[f"layers.{l}.input_norm"] = g[pre + "input_layernorm.weight"]
        out[f"layers.{l}.qkv"] = torch.cat([g[pre + "self_attn.q_proj.weight"],
                                            g[pre + "self_attn.k_proj.weight"],
                                            g[pre + "self_attn.v_proj.weight"]])
        out[f"layers.{l}.q_norm"] = g[pre + "self_attn.q_norm.weight"]
        out[f"layers.{l}.k_norm"] = g[pre + "self_attn.k_norm.weight"]
        out[f"layers.{l}.o"] = g[pre + "self_attn.o_proj.weight"]
        out[f"layers.{l}.post_norm"] = g[pre + "post_attention_layernorm.weight"]
        out[f"layers.{l}.router"] = g[pre + "mlp.gate.weight"]
        out[f"layers.{l}.gate_up"] = g[pre + "mlp.experts.gate_up_proj"].reshape(-1, s.hidden)
        out[f"layers.{l}.down"] = g[pre + "mlp.experts.down_proj"].reshape(-1, s.inter)
    return out


def main():
    torch.manual_seed(0)
    s = O.Shape.from_config("tiny-moe")
    params = O.init_params(s, seed=0)
    tok, lab = O.synthetic_batch(s, M, 1, SEQ)
    w = {k: v.clone().requires_grad_(True) for k, v in params.items()}
    l_or = O.forward_loss_sum(w, tok[0], lab[0], s)
    l_or.backward()
    m = hf_moe(s, params)
    out = m(input_ids=tok[0].long(), labels=None)
    l_hf = torch.nn.functional.cross_entropy(out.logits.view(-1, s.vocab), lab[0].reshape(-1).long(),
                                             reduction="sum")
    l_hf.backward()
    gh = hf_grads(m, s)
    worst = max(((w[k].grad - gh[k]).norm() / gh[k].norm().clamp_min(1e-30)).item() for k in gh)
    loss_rel = abs(l_or.item() - l_hf.item()) / abs(l_hf.item())
    print("oracle vs HF Qwen3-MoE: loss rel", loss_rel, "worst grad rel-L2", worst)
    assert loss_rel < 1e-5 and worst < 1e-4
    rec = {"config": "tiny-moe", "M": M, "seq": SEQ, "steps": STEPS, "lora_rank": RANK,
           "hparams": HP, "weights_seed": 0, "lora_seed": 1, "tokens_seed": 1234,
           "hf_check": {"loss_hf": l_hf.item(), "loss_oracle": l_or.item(),
                        "loss_rel": loss_rel, "worst_grad_rel_l2": worst}}
    params.update(O.init_lora_params(s, RANK, seed=1, std_b=0.02))
    for mode in ("sync", "async"):
        o = O.StepOracle(s, params, mode=mode, lora_scale=2.0, **HP)
        losses = [o.step(tok, lab) for _ in range(STEPS)]
        rec[mode] = {"losses": losses}
        print(mode, losses)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "moe_golden.json")
    with open(path, "w") as f:
        json.dump(rec, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
