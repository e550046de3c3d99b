"""Micro-benchmarks of the non-GEMM stage kernels at Qwen3-8B shapes (T=4096):
flash attention fwd/bwd (TFLOP/s, causal FLOPs) and the HBM-bound kernels
(GB/s of algorithmic bytes). CUDA-event timed after warm-up."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2604_27085_b200 import kernels as K  # noqa: E402


def bench(fn, iters=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    T, seq, nq, nk, hd, h, m, V = 4096, 4096, 32, 8, 128, 4096, 12288, 151936
    out = []
    qkv = torch.randn(T, (nq + 2 * nk) * hd, device="cuda").to(torch.bfloat16)
    q, k, v = qkv[:, :nq * hd], qkv[:, nq * hd:(nq + nk) * hd], qkv[:, (nq + nk) * hd:]
    o = torch.empty(T, nq * hd, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(nq, T, device="cuda")
    flops = 4.0 * nq * hd * seq * seq / 2 * (T // seq)  # causal
    ms = bench(lambda: K.attn_fwd_tc(q, k, v, o, lse, seq, nq, nk, hd))
    out.append({"kernel": "attn_fwd_tc", "ms": ms, "tflops": flops / ms / 1e9})
    do = torch.randn_like(o)
    dqkv = torch.empty_like(qkv)
    delta = torch.empty(nq, T, device="cuda")
    ms = bench(lambda: K.attn_bwd_tc(q, k, v, o, do, lse, dqkv[:, :nq * hd],
                                     dqkv[:, nq * hd:(nq + nk) * hd], dqkv[:, (nq + nk) * hd:],
                                     delta, seq, nq, nk, hd))
    out.append({"kernel": "attn_bwd_tc", "ms": ms, "tflops": 2.5 * flops / ms / 1e9,
                "executed_tflops": 3.5 * flops / ms / 1e9})
    if "attn" in sys.argv[1:]:
        for r in out:
            print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()}))
        return

    x = torch.randn(T, h, device="cuda").to(torch.bfloat16)
    w = torch.ones(h, device="cuda", dtype=torch.bfloat16)
    y = torch.empty_like(x)
    rstd = torch.empty(T, device="cuda")
    ms = bench(lambda: K.rmsnorm_fwd(x, w, y, rstd))
    out.append({"kernel": "rmsnorm_fwd", "ms": ms, "gbs": 2 * T * h * 2 / ms / 1e6})
    dx32 = torch.empty(T, h, device="cuda")
    dx16 = torch.empty_like(x)
    dw = torch.zeros(h, device="cuda")
    ms = bench(lambda: K.rmsnorm_bwd(y, x, w, rstd, dx32=dx32, dx16=dx16, dw=dw, dres=dx32))
    out.append({"kernel": "rmsnorm_bwd", "ms": ms, "gbs": T * h * (2 + 2 + 4 + 4 + 2) / ms / 1e6})
    gu = torch.randn(T, 2 * m, device="cuda").to(torch.bfloat16)
    act = torch.empty(T, m, device="cuda", dtype=torch.bfloat16)
    ms = bench(lambda: K.swiglu_fwd(gu, act))
    out.append({"kernel": "swiglu_fwd", "ms": ms, "gbs": T * m * 6 / ms / 1e6})
    dgu = torch.empty_like(gu)
    ms = bench(lambda: K.swiglu_bwd(act, gu, dgu))
    out.append({"kernel": "swiglu_bwd", "ms": ms, "gbs": T * m * 10 / ms / 1e6})
    cs = K.rope_table(seq, hd).cuda()
    qo = torch.empty(T, nq * hd, device="cuda", dtype=torch.bfloat16)
    ko = torch.empty(T, nk * hd, device="cuda", dtype=torch.bfloat16)
    rq, rk = torch.empty(T, nq, device="cuda"), torch.empty(T, nk, device="cuda")
    ms = bench(lambda: K.qk_norm_rope_fwd(qkv, nq, nk, hd, w[:hd], w[:hd], cs, seq, qo, ko, rq, rk))
    out.append({"kernel": "qk_norm_rope_fwd", "ms": ms, "gbs": T * (nq + nk) * hd * 4 / ms / 1e6})
    dqk = torch.empty_like(qkv)
    dqw, dkw = torch.zeros(hd, device="cuda"), torch.zeros(hd, device="cuda")
    ms = bench(lambda: K.qk_norm_rope_bwd(qo, ko, qkv, nq, nk, hd, w[:hd], w[:hd], rq, rk, cs, seq,
                                          dqk, dqw, dkw))
    out.append({"kernel": "qk_norm_rope_bwd", "ms": ms, "gbs": T * (nq + nk) * hd * 6 / ms / 1e6})
    rows = 1024
    z = torch.randn(rows, V, device="cuda").to(torch.bfloat16)
    labels = torch.randint(0, V, (rows,), device="cuda", dtype=torch.int32)
    loss = torch.zeros(1, device="cuda")
    ms = bench(lambda: K.ce_fwd_bwd(z, labels, 1.0 / rows, loss))
    out.append({"kernel": "ce_fwd_bwd", "ms": ms, "gbs": rows * V * 6 / ms / 1e6})
    n = 385_875_968 // 2  # one 8B layer's params
    p, mm, vv, g = (torch.zeros(n, device="cuda") for _ in range(4))
    w16 = torch.empty(n, device="cuda", dtype=torch.bfloat16)
    ms = bench(lambda: K.adamw(p, mm, vv, g, w16, 1), iters=5)
    out.append({"kernel": "adamw", "ms": ms, "gbs": n * (16 + 12 + 2) / ms / 1e6})
    for r in out:
        print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()}))


if __name__ == "__main__":
    main()
