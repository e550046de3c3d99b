"""C5-shape diagnostics: attention fwd/bwd kernels at Qwen3-235B-A22B
attention shapes (64 q heads, 4 kv heads, hd 128) and seq 31744, error-checked
after every launch; then one runtime iteration of the reduced-depth model."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2604_27085_b200 import kernels as K  # noqa: E402


def attn(T, seq, nq, nk, hd=128):
    qkv = (torch.randn(T, (nq + 2 * nk) * hd, device="cuda") * 0.5).to(torch.bfloat16)
    q, k, v = qkv[:, :nq * hd], qkv[:, nq * hd:(nq + nk) * hd], qkv[:, (nq + nk) * hd:]
    o = torch.empty(T, nq * hd, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(nq, T, device="cuda")
    K.attn_fwd_tc(q, k, v, o, lse, seq, nq, nk, hd)
    torch.cuda.synchronize()
    print("fwd ok", T, seq, nq, nk, "o finite", bool(torch.isfinite(o.float()).all()), flush=True)
    do = (torch.randn(T, nq * hd, device="cuda") * 0.1).to(torch.bfloat16)
    dqkv = torch.zeros_like(qkv)
    dq, dk, dv = dqkv[:, :nq * hd], dqkv[:, nq * hd:(nq + nk) * hd], dqkv[:, (nq + nk) * hd:]
    delta = torch.empty(nq, T, device="cuda")
    K.attn_bwd_tc(q, k, v, o, do, lse, dq, dk, dv, delta, seq, nq, nk, hd)
    torch.cuda.synchronize()
    print("bwd ok", T, seq, nq, nk, "finite", bool(torch.isfinite(dqkv.float()).all()), flush=True)


if __name__ == "__main__":
    for T, seq, nq, nk in [(4096, 4096, 64, 4), (8192, 8192, 64, 4), (16384, 16384, 64, 4),
                           (31744, 31744, 64, 4)]:
        try:
            attn(T, seq, nq, nk)
        except Exception as e:
            print("FAIL", T, seq, nq, nk, repr(e)[:300], flush=True)
            break
