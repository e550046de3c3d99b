"""The MoE oracle (oracle/step_oracle.py moe_block + StepOracle LoRA mode)
reproduces its committed golden trajectory (tests/golden/moe_golden.json,
pinned to transformers' Qwen3MoeForCausalLM by make_moe_golden.py), and the
router restatement matches the transformers router on random inputs."""
import json
import os

import torch

from oracle import step_oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "moe_golden.json")


def test_moe_golden_pin_and_trajectory():
    g = json.load(open(GOLDEN))
    assert g["hf_check"]["loss_rel"] < 1e-5 and g["hf_check"]["worst_grad_rel_l2"] < 1e-4
    s = O.Shape.from_config("tiny-moe")
    assert s.moe and s.experts == 8 and s.active == 2 and s.norm_topk
    params = O.init_params(s, seed=g["weights_seed"])
    params.update(O.init_lora_params(s, g["lora_rank"], seed=g["lora_seed"], std_b=0.02))
    tok, lab = O.synthetic_batch(s, g["M"], 1, g["seq"], seed=g["tokens_seed"])
    o = O.StepOracle(s, params, mode="sync", lora_scale=2.0, **g["hparams"])
    got = [o.step(tok, lab) for _ in range(2)]
    for a, b in zip(got, g["sync"]["losses"]):
        assert abs(a - b) / b < 1e-5, (got, g["sync"]["losses"])


def test_router_matches_transformers():
    from transformers import Qwen3MoeConfig
    from transformers.models.qwen3_moe.modeling_qwen3_moe import Qwen3MoeTopKRouter
    s = O.Shape.from_config("tiny-moe")
    cfg = Qwen3MoeConfig(hidden_size=s.hidden, num_experts=s.experts,
                         num_experts_per_tok=s.active, norm_topk_prob=s.norm_topk)
    r = Qwen3MoeTopKRouter(cfg)
    torch.nn.init.normal_(r.weight, std=0.1)
    x = torch.randn(64, s.hidden)
    _, w_hf, i_hf = r(x)
    w, i = O.moe_route(x, r.weight.detach(), s)
    assert torch.equal(i, i_hf)
    assert torch.allclose(w, w_hf, atol=1e-6)
