"""ORACLE / TEST INFRASTRUCTURE ONLY — the CPU restatement of one RoundPipe
training step. Never imported by the product; only tests/, smoke() and
bench.py's cpu_baseline / --impl reference legs use it, as the checker.

The reference repository has no data-plane code: no
file computes a loss, gradient or optimizer update. This module restates,
in fp32 PyTorch on the CPU:
  * the Qwen3 decoder math of transformers 5.5.0 (third-party, pinned in
    this image): RMSNorm modeling_qwen3.py:50-67, MLP/SwiGLU :70-83, rotary
    :86-182, GQA eager attention :184-220, per-head q/k-norm :248-264,
    decoder layer :294-336, Qwen3ForCausalLM :442+ (untied LM head);
  * the RoundPipe mixed-precision model: fp32
    optimizer copy, bf16 master copy used for compute (here: bf16-rounded
    weights computed in fp32);
  * the optimizer hand-off (consistency.hpp:98-109):
      sync  — iteration t+1 sees grads of t;
      async — step(t+1) applies grads of t, first visible to iteration t+2
              (staleness 1);
  * loss = sum of token CE over the step / number of valid labels; AdamW =
    torch.optim.AdamW (decoupled weight decay);
  * Qwen3-MoE layers (BASELINE configs[4]): transformers 5.5.0
    modeling_qwen3_moe.py — router :254-272 (softmax in fp32, top-k,
    renormalised when norm_topk_prob), experts :215-251 (SwiGLU per expert,
    weighted sum), sparse block :275-287; every decoder layer is sparse
    (decoder_sparse_step 1, no mlp_only_layers). LoRA on a MoE model adapts
    the attention projections only (experts and router frozen).
Pinning: tests/golden/make_step_golden.py checks this module's loss and
gradients against transformers' Qwen3ForCausalLM on identical weights and
commits the numbers (tests/golden/step_golden.json).
"""
from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@dataclass
class Shape:
    hidden: int
    heads: int
    kv_heads: int
    head_dim: int
    inter: int
    layers: int
    vocab: int
    rope_theta: float = 1e6
    eps: float = 1e-6
    experts: int = 1        # MoE: experts per layer (inter = moe_intermediate_size)
    active: int = 1         # experts routed per token
    norm_topk: bool = True  # renormalise the top-k routing weights

    @property
    def moe(self) -> bool:
        return self.experts > 1

    @staticmethod
    def from_config(name: str) -> "Shape":
        path = name if name.endswith(".json") else os.path.join(
            ROOT, "configs", "models", name + ".json")
        with open(path) as f:
            j = json.load(f)
        return Shape(int(j["hidden_dim"]), j["num_heads"], j["num_kv_heads"],
                     j.get("head_dim", int(j["hidden_dim"]) // j["num_heads"]),
                     int(j["intermediate_dim"]), j["num_layers"], j["vocab_size"],
                     j.get("rope_theta", 1e6), j.get("rms_norm_eps", 1e-6),
                     int(j.get("total_experts", 1)), int(j.get("active_experts", 1)),
                     bool(j.get("norm_topk_prob", True)))


# parameter names and shapes, in the flat per-layer order the runtime uses
def layer_param_shapes(s: Shape):
    qd, kd = s.heads * s.head_dim, s.kv_heads * s.head_dim
    base = [("input_norm", (s.hidden,)), ("qkv", (qd + 2 * kd, s.hidden)),
            ("q_norm", (s.head_dim,)), ("k_norm", (s.head_dim,)),
            ("o", (s.hidden, qd)), ("post_norm", (s.hidden,))]
    if s.moe:  # router [E, h]; experts stacked: gate_up [E*2m, h], down [E*h, m]
        return base + [("router", (s.experts, s.hidden)),
                       ("gate_up", (s.experts * 2 * s.inter, s.hidden)),
                       ("down", (s.experts * s.hidden, s.inter))]
    return base + [("gate_up", (2 * s.inter, s.hidden)), ("down", (s.hidden, s.inter))]


def lora_param_shapes(s: Shape, r: int):
    """LoRA adapters of a layer (PEFT semantics): A [r, in],
    B [out, r]; in the runtime's flat order after the base tensors."""
    qd, kd = s.heads * s.head_dim, s.kv_heads * s.head_dim
    att = [("qkv_lora_A", (r, s.hidden)), ("qkv_lora_B", (qd + 2 * kd, r)),
           ("o_lora_A", (r, qd)), ("o_lora_B", (s.hidden, r))]
    if s.moe:  # experts and router frozen
        return att
    return att + [("gate_up_lora_A", (r, s.hidden)), ("gate_up_lora_B", (2 * s.inter, r)),
                  ("down_lora_A", (r, s.inter)), ("down_lora_B", (s.hidden, r))]


def init_lora_params(s: Shape, r: int, seed: int = 1, std_a: float = 0.02, std_b: float = 0.0):
    """A ~ N(0, std_a), B ~ N(0, std_b) (PEFT's default B = 0), bf16-rounded."""
    g = torch.Generator().manual_seed(seed)
    out = {}
    for l in range(s.layers):
        for n, sh in lora_param_shapes(s, r):
            std = std_a if n.endswith("_A") else std_b
            out[f"layers.{l}.{n}"] = (torch.randn(sh, generator=g) * std).to(torch.bfloat16).float()
    return out


def head_param_shapes(s: Shape):
    return [("final_norm", (s.hidden,)), ("lm_head", (s.vocab, s.hidden))]


def init_params(s: Shape, seed: int = 0, std: float = 0.02):
    """Deterministic init: N(0, std) matrices, ones for norms; values are
    rounded to bf16 so the fp32 oracle and the bf16 GPU copy start equal."""
    g = torch.Generator().manual_seed(seed)

    def mk(name, shape):
        if len(shape) == 1:
            return torch.ones(shape)
        return (torch.randn(shape, generator=g) * std).to(torch.bfloat16).float()
    params = {"embed": (torch.randn(s.vocab, s.hidden, generator=g) * std)
              .to(torch.bfloat16).float()}
    for l in range(s.layers):
        for n, sh in layer_param_shapes(s):
            params[f"layers.{l}.{n}"] = mk(n, sh)
    for n, sh in head_param_shapes(s):
        params[f"head.{n}"] = mk(n, sh)
    return params


def rms(x, w, eps):
    return w * (x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps))


def rope_cos_sin(seq, hd, theta):
    inv = 1.0 / (theta ** (torch.arange(0, hd, 2, dtype=torch.float64) / hd))
    ang = torch.arange(seq, dtype=torch.float64)[:, None] * inv[None, :]
    cos, sin = ang.cos().float(), ang.sin().float()
    return torch.cat([cos, cos], -1), torch.cat([sin, sin], -1)


def rotate_half(x):
    h = x.shape[-1] // 2
    return torch.cat([-x[..., h:], x[..., :h]], -1)


def decoder_layer(x, p, pre, s: Shape, cos, sin, lora_scale: float = 0.0):
    """x [b, S, h] fp32 -> [b, S, h]; p(name) gives the fp32 weight. With
    lora_scale > 0 every linear adds scale * (x A^T) B^T (PEFT LoRA)."""
    b, S, _ = x.shape
    qd, kd = s.heads * s.head_dim, s.kv_heads * s.head_dim

    def lin(t, name):
        y = t @ p(pre + name).t()
        if lora_scale:
            y = y + lora_scale * ((t @ p(pre + name + "_lora_A").t()) @ p(pre + name + "_lora_B").t())
        return y
    h1 = rms(x, p(pre + "input_norm"), s.eps)
    qkv = lin(h1, "qkv")
    q = qkv[..., :qd].view(b, S, s.heads, s.head_dim)
    k = qkv[..., qd:qd + kd].view(b, S, s.kv_heads, s.head_dim)
    v = qkv[..., qd + kd:].view(b, S, s.kv_heads, s.head_dim)
    q = rms(q, p(pre + "q_norm"), s.eps).transpose(1, 2)
    k = rms(k, p(pre + "k_norm"), s.eps).transpose(1, 2)
    v = v.transpose(1, 2)
    q = q * cos + rotate_half(q) * sin
    k = k * cos + rotate_half(k) * sin
    rep = s.heads // s.kv_heads
    k = k.repeat_interleave(rep, 1)
    v = v.repeat_interleave(rep, 1)
    att = (q @ k.transpose(-1, -2)) * (s.head_dim ** -0.5)
    mask = torch.ones(S, S, dtype=torch.bool).triu(1)
    att = att.masked_fill(mask, float("-inf")).softmax(-1)
    o = (att @ v).transpose(1, 2).reshape(b, S, qd)
    x2 = x + lin(o, "o")
    h2 = rms(x2, p(pre + "post_norm"), s.eps)
    if s.moe:
        return x2 + moe_block(h2, p, pre, s)
    gu = lin(h2, "gate_up")
    act = torch.nn.functional.silu(gu[..., :s.inter]) * gu[..., s.inter:]
    return x2 + lin(act, "down")


def moe_route(hs, router, s: Shape):
    """Qwen3MoeTopKRouter (modeling_qwen3_moe.py:263-272): fp32 softmax over
    the E router logits, top-k, renormalised when norm_topk_prob."""
    probs = torch.softmax(hs @ router.t(), dim=-1, dtype=torch.float32)
    topv, topi = torch.topk(probs, s.active, dim=-1)
    if s.norm_topk:
        topv = topv / topv.sum(-1, keepdim=True)
    return topv, topi


def moe_block(h2, p, pre, s: Shape):
    """Qwen3MoeSparseMoeBlock (:275-287) + Qwen3MoeExperts (:215-251) on
    h2 [b, S, h]: sum over the k routed experts of w * down(silu(g) * u)."""
    b, S, h = h2.shape
    hs = h2.reshape(-1, h)
    topv, topi = moe_route(hs, p(pre + "router"), s)
    gate_up = p(pre + "gate_up").view(s.experts, 2 * s.inter, h)
    down = p(pre + "down").view(s.experts, h, s.inter)
    y = torch.zeros_like(hs)
    for e in range(s.experts):
        tok, slot = torch.where(topi == e)
        if tok.numel() == 0:
            continue
        gu = hs[tok] @ gate_up[e].t()
        act = torch.nn.functional.silu(gu[:, :s.inter]) * gu[:, s.inter:]
        y = y.index_add(0, tok, (act @ down[e].t()) * topv[tok, slot, None])
    return y.view(b, S, h)


def forward_loss_sum(params, tokens, labels, s: Shape, lora_scale: float = 0.0):
    """Sum of token cross-entropy (labels < 0 ignored) for tokens [b, S]."""
    b, S = tokens.shape
    cos, sin = rope_cos_sin(S, s.head_dim, s.rope_theta)

    def p(name):
        return params[name]
    x = params["embed"][tokens]
    for l in range(s.layers):
        x = decoder_layer(x, p, f"layers.{l}.", s, cos, sin, lora_scale)
    x = rms(x, p("head.final_norm"), s.eps)
    logits = x @ p("head.lm_head").t()
    return torch.nn.functional.cross_entropy(
        logits.view(-1, s.vocab), labels.reshape(-1).long(), ignore_index=-100,
        reduction="sum")


def bf16_round(t):
    return t.to(torch.bfloat16).float()


class StepOracle:
    """fp32 CPU RoundPipe step: M micro-batches of [b, S] tokens per
    iteration, grads accumulated over the step, AdamW on an fp32 copy,
    compute on bf16-rounded weights, sync or async (staleness-1) hand-off."""

    def __init__(self, s: Shape, params: dict, lr=1e-3, betas=(0.9, 0.95), eps=1e-8,
                 weight_decay=0.0, mode="sync", threads: int | None = None,
                 lora_scale: float = 0.0):
        """lora_scale > 0: LoRA fine-tune — only the *_lora_A/B params train
        (AdamW), every base weight is frozen (PEFT semantics)."""
        assert mode in ("sync", "async")
        if threads:
            torch.set_num_threads(threads)
        self.s = s
        self.mode = mode
        self.lora_scale = lora_scale
        self.master = {k: v.clone().float().requires_grad_(False) for k, v in params.items()}
        # LoRA: frozen base weights are bf16-representable (init_params) and
        # never change, so they are shared rather than copied (and get no
        # grads) — the oracle then fits full-width MoE layers in host memory
        self.trainable = {k for k in params if not lora_scale or "_lora_" in k}
        self.opt_params = {k: torch.nn.Parameter(v.clone()) for k, v in self.master.items()
                           if k in self.trainable}
        self.opt = torch.optim.AdamW(list(self.opt_params.values()), lr=lr, betas=betas,
                                     eps=eps, weight_decay=weight_decay)
        # weights the next iteration computes with (bf16 master copy)
        self.used = {k: (bf16_round(v) if k in self.trainable else v)
                     for k, v in self.master.items()}
        self.pending = None  # async: result of the last optimizer step
        self.last_grads = None

    def _fwd_bwd(self, tokens, labels):
        w = {k: (v.clone().requires_grad_(True) if k in self.trainable else v)
             for k, v in self.used.items()}
        n_valid = int((labels >= 0).sum())
        total = 0.0
        for mb in range(tokens.shape[0]):
            loss = forward_loss_sum(w, tokens[mb], labels[mb], self.s, self.lora_scale) / n_valid
            loss.backward()
            total += loss.item()
        return total, {k: (v.grad if v.grad is not None else torch.zeros_like(v))
                       if k in self.trainable else None for k, v in w.items()}

    def _apply(self, grads):
        for k, prm in self.opt_params.items():
            prm.grad = grads[k].clone()
        self.opt.step()
        self.opt.zero_grad(set_to_none=True)
        out = dict(self.used)  # frozen: unchanged
        out.update({k: bf16_round(p.detach()) for k, p in self.opt_params.items()})
        return out

    def step(self, tokens, labels):
        """tokens, labels: [M, b, S] int. Returns the step's mean loss."""
        loss, grads = self._fwd_bwd(tokens, labels)
        self.last_grads = grads
        if self.mode == "sync":
            self.used = self._apply(grads)
        else:
            # step(t+1) applies grads of t; its result is uploaded at t+2
            if self.pending is not None:
                self.used = self.pending
            self.pending = self._apply(grads)
        return loss

    def master_fp32(self):
        out = {k: v for k, v in self.master.items() if k not in self.trainable}
        out.update({k: p.detach().clone() for k, p in self.opt_params.items()})
        return out


def synthetic_batch(s: Shape, M: int, b: int, S: int, seed: int = 1234):
    """Token ids ~ U{0..V-1} (seeded), labels = ids shifted by one (every
    position labelled; callers mask positions with -100 to ignore them)."""
    g = torch.Generator().manual_seed(seed)
    ids = torch.randint(0, s.vocab, (M, b, S + 1), generator=g)
    tokens = ids[..., :S].contiguous()
    labels = ids[..., 1:].contiguous()
    return tokens.int(), labels.int()


def _cli():
    import argparse
    import time
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="tiny")
    ap.add_argument("--seq", type=int, default=256)
    ap.add_argument("--M", type=int, default=4)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--mode", default="sync")
    a = ap.parse_args()
    s = Shape.from_config(a.model)
    o = StepOracle(s, init_params(s), mode=a.mode)
    tok, lab = synthetic_batch(s, a.M, 1, a.seq)
    for i in range(a.steps):
        t0 = time.time()
        print(i, o.step(tok, lab), f"{time.time() - t0:.2f}s")


if __name__ == "__main__":
    _cli()
