"""Pin the data-plane oracle (oracle/step_oracle.py) against transformers'
Qwen3ForCausalLM (third-party, transformers 5.5.0 in this image) and commit
golden numbers for the tiny config (BASELINE configs[0]):

  1. single-micro-batch loss and every parameter gradient: oracle vs HF on
     identical fp32 weights (max rel-L2 recorded; must be ~1e-6);
  2. the oracle's RoundPipe step, sync and async, 3 steps: per-step loss,
     per-tensor grad norms of step 0, per-tensor fp32 master norms after 3
     steps (seeded: weights seed 0 / std 0.02, tokens seed 1234).

Run: python tests/golden/make_step_golden.py   (CPU, ~1 min)
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import step_oracle as O  # noqa: E402

M, SEQ, STEPS = 4, 256, 3
HP = dict(lr=1e-3, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.0)


def hf_model(s, params):
    from transformers import Qwen3Config, Qwen3ForCausalLM
    cfg = Qwen3Config(vocab_size=s.vocab, hidden_size=s.hidden, intermediate_size=s.inter,
                      num_hidden_layers=s.layers, num_attention_heads=s.heads,
                      num_key_value_heads=s.kv_heads, head_dim=s.head_dim,
                      rope_theta=s.rope_theta, rms_norm_eps=s.eps, tie_word_embeddings=False,
                      max_position_embeddings=4096, attention_bias=False)
    cfg._attn_implementation = "eager"
    m = Qwen3ForCausalLM(cfg).float()
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
        sd[pre + "mlp.gate_proj.weight"] = p("gate_up")[:s.inter]
        sd[pre + "mlp.up_proj.weight"] = p("gate_up")[s.inter:]
        sd[pre + "mlp.down_proj.weight"] = p("down")
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
        out[f"layers.{l}.gate_up"] = torch.cat([g[pre + "mlp.gate_proj.weight"],
                                                g[pre + "mlp.up_proj.weight"]])
        out[f"layers.{l}.down"] = g[pre + "mlp.down_proj.weight"]
    return out


def main():
    torch.manual_seed(0)
    s = O.Shape.from_config("tiny")
    params = O.init_params(s, seed=0)
    tok, lab = O.synthetic_batch(s, M, 1, SEQ)
    # 1. oracle layer math vs HF on one micro-batch (fp32, same weights)
    w = {k: v.clone().requires_grad_(True) for k, v in params.items()}
    l_or = O.forward_loss_sum(w, tok[0], lab[0], s)
    l_or.backward()
    m = hf_model(s, params)
    out = m(input_ids=tok[0].long(), labels=None)
    l_hf = torch.nn.functional.cross_entropy(out.logits.view(-1, s.vocab), lab[0].reshape(-1).long(),
                                             reduction="sum")
    l_hf.backward()
    gh = hf_grads(m, s)
    worst = max(((w[k].grad - gh[k]).norm() / gh[k].norm().clamp_min(1e-30)).item() for k in gh)
    loss_rel = abs(l_or.item() - l_hf.item()) / abs(l_hf.item())
    print("oracle vs HF: loss rel", loss_rel, "worst grad rel-L2", worst)
    assert loss_rel < 1e-5 and worst < 1e-4
    rec = {"config": "tiny", "M": M, "seq": SEQ, "steps": STEPS, "hparams": HP,
           "weights_seed": 0, "tokens_seed": 1234,
           "hf_check": {"loss_hf": l_hf.item(), "loss_oracle": l_or.item(),
                        "loss_rel": loss_rel, "worst_grad_rel_l2": worst}}
    # 2. the oracle's RoundPipe step
    for mode in ("sync", "async"):
        o = O.StepOracle(s, params, mode=mode, lr=HP["lr"], betas=HP["betas"], eps=HP["eps"],
                         weight_decay=HP["weight_decay"])
        losses = []
        gnorm0 = None
        for it in range(STEPS):
            losses.append(o.step(tok, lab))
            if it == 0:
                gnorm0 = {k: v.norm().item() for k, v in o.last_grads.items()}
        master = o.master_fp32()
        rec[mode] = {"losses": losses, "grad_norms_step0": gnorm0,
                     "master_norms": {k: v.norm().item() for k, v in master.items()},
                     "master_sums": {k: v.double().sum().item() for k, v in master.items()}}
        print(mode, losses)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "step_golden.json")
    with open(path, "w") as f:
        json.dump(rec, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
