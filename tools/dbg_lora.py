import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from oracle import step_oracle as O
from paper_2604_27085_b200.runtime import AdamW, RoundPipe
HP = dict(lr=1e-3, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.0)
s = O.Shape.from_config("tiny")
r, alpha = 16, 32.0
params = O.init_params(s, seed=0)
params.update(O.init_lora_params(s, r, seed=3, std_a=0.02, std_b=0.02))
tok, lab = O.synthetic_batch(s, 4, 1, 256)
rt = RoundPipe("tiny", seq_len=256, micro_batch=1, micro_batches=4, num_gpus=1,
               async_optimizer=False, adam=AdamW(**{"lr": 1e-3}), skip_init=True,
               lora_rank=r, lora_alpha=alpha)
rt.load_state({k: v.numpy() for k, v in params.items()}, s.layers)
back = rt.read_state(s.layers, which=0)
for k in ("layers.0.qkv_lora_A", "layers.0.qkv_lora_B", "layers.0.qkv"):
    print("roundtrip", k, float(np.abs(np.asarray(back[k]).reshape(-1) - params[k].numpy().reshape(-1)).max()))
o = O.StepOracle(s, params, mode="sync", lora_scale=alpha / r, **HP)
got = rt.forward_backward(tok.numpy(), lab.numpy())
g = rt.read_state(s.layers, which=2)
ref = o.step(tok, lab)
print("loss", got, ref)
rg = o.last_grads
for l in range(s.layers):
    for n in ["qkv_lora_A", "qkv_lora_B", "o_lora_A", "o_lora_B", "gate_up_lora_A", "gate_up_lora_B",
              "down_lora_A", "down_lora_B"]:
        k = f"layers.{l}.{n}"
        a = torch.from_numpy(np.asarray(g[k])).reshape(rg[k].shape)
        print(k, "rel", round(((a - rg[k]).norm() / rg[k].norm()).item(), 4), "norms",
              round(a.norm().item(), 6), round(rg[k].norm().item(), 6))
rt.step()
m = rt.read_state(s.layers, which=0)
om = o.master_fp32()
for k in ("layers.0.qkv_lora_A", "layers.0.down_lora_B"):
    du = torch.from_numpy(np.asarray(m[k])).reshape(om[k].shape) - params[k]
    dr = om[k] - params[k]
    print("update", k, du.norm().item(), dr.norm().item(), float((du * dr).sum() / (du.norm() * dr.norm())))
print("loss2", rt.forward_backward(tok.numpy(), lab.numpy()), o.step(tok, lab))
