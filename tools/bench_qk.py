"""QK-norm/RoPE fwd/bwd micro-benchmark at the BASELINE models' head shapes
(T=4096), L2 flushed before every timed launch (a 256 MB write), CUDA events
around the kernel alone. Prints one JSON line per (model, kernel) with a
checksum of the outputs so same-box A/B runs over RP_LIB variants can also
compare results bit for bit."""
import hashlib
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2604_27085_b200 import kernels as K  # noqa: E402

SHAPES = {"qwen3-8b": (32, 8), "qwen3-1.7b": (16, 8), "qwen3-32b": (64, 8), "qwen3-235b": (64, 4)}


def digest(*ts):
    h = hashlib.sha1()
    for t in ts:
        h.update(t.contiguous().view(torch.uint8).cpu().numpy().tobytes())
    return h.hexdigest()[:12]


def timed(fn, flush, iters=30):
    for _ in range(3):
        fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    acc = torch.empty((), device="cuda")
    for s, e in ev:
        torch.sum(flush, dim=0, out=acc)  # a READ of 256 MB: evicts L2 without leaving dirty lines
        s.record()
        fn()
        e.record()
    torch.cuda.synchronize()
    ts = sorted(s.elapsed_time(e) for s, e in ev)
    return ts[len(ts) // 2]


def main():
    lib = os.environ.get("RP_LIB", "head")
    T, seq, hd = 4096, 4096, 128
    flush = torch.empty(64 * 1024 * 1024, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(0)
    # calibration at Qwen3-8B's q|k bytes (T x 5120 bf16 in, same out): the
    # device copy and the RMSNorm forward (same 4 B/element pattern)
    x = torch.randn(T, 5120, device="cuda", generator=g).to(torch.bfloat16)
    y = torch.empty_like(x)
    ms = timed(lambda: y.copy_(x), flush)
    print(json.dumps({"lib": lib, "model": "calib", "kernel": "copy", "ms": round(ms, 5),
                      "gbs": round(x.numel() * 4 / ms / 1e6, 1)}))
    wn, rs = torch.ones(5120, device="cuda", dtype=torch.bfloat16), torch.empty(T, device="cuda")
    ms = timed(lambda: K.rmsnorm_fwd(x, wn, y, rs), flush)
    print(json.dumps({"lib": lib, "model": "calib", "kernel": "rmsnorm_fwd", "ms": round(ms, 5),
                      "gbs": round(x.numel() * 4 / ms / 1e6, 1)}))
    # RMSNorm backward at Qwen3-8B's hidden size (14 B / element)
    h = 4096
    xb = torch.randn(T, h, device="cuda", generator=g).to(torch.bfloat16)
    dyb = torch.randn(T, h, device="cuda", generator=g).to(torch.bfloat16)
    wb = (torch.randn(h, device="cuda", generator=g) * 0.2 + 1).to(torch.bfloat16)
    yb, rsb = torch.empty_like(xb), torch.empty(T, device="cuda")
    K.rmsnorm_fwd(xb, wb, yb, rsb)
    dres = torch.randn(T, h, device="cuda", generator=g)
    dx32, dx16, dwb = torch.empty(T, h, device="cuda"), torch.empty_like(xb), torch.zeros(h, device="cuda")
    ms = timed(lambda: K.rmsnorm_bwd(dyb, xb, wb, rsb, dx32=dx32, dx16=dx16, dw=dwb, dres=dres), flush)
    torch.cuda.synchronize()
    print(json.dumps({"lib": lib, "model": "qwen3-8b", "kernel": "rmsnorm_bwd", "ms": round(ms, 5),
                      "gbs": round(T * h * 14 / ms / 1e6, 1), "digest": digest(dx32, dx16)}))
    for model, (nq, nk) in SHAPES.items():
        qkv = torch.randn(T, (nq + 2 * nk) * hd, device="cuda", generator=g).to(torch.bfloat16)
        w = (torch.randn(2 * hd, device="cuda", generator=g) * 0.2 + 1).to(torch.bfloat16)
        cs = K.rope_table(seq, hd).cuda()
        qo = torch.empty(T, nq * hd, device="cuda", dtype=torch.bfloat16)
        ko = torch.empty(T, nk * hd, device="cuda", dtype=torch.bfloat16)
        rq, rk = torch.empty(T, nq, device="cuda"), torch.empty(T, nk, device="cuda")
        fwd = lambda: K.qk_norm_rope_fwd(qkv, nq, nk, hd, w[:hd], w[hd:], cs, seq, qo, ko, rq, rk)  # noqa: E731
        ms = timed(fwd, flush)
        fwd()
        torch.cuda.synchronize()
        print(json.dumps({"lib": lib, "model": model, "kernel": "qk_norm_rope_fwd", "ms": round(ms, 5),
                          "gbs": round(T * (nq + nk) * hd * 4 / ms / 1e6, 1), "digest": digest(qo, ko, rq, rk)}))
        dq = torch.randn(T, nq * hd, device="cuda", generator=g).to(torch.bfloat16)
        dk = torch.randn(T, nk * hd, device="cuda", generator=g).to(torch.bfloat16)
        dqk = torch.zeros_like(qkv)
        dqw, dkw = torch.zeros(hd, device="cuda"), torch.zeros(hd, device="cuda")
        bwd = lambda: K.qk_norm_rope_bwd(dq, dk, qkv, nq, nk, hd, w[:hd], w[hd:], rq, rk, cs, seq,  # noqa: E731
                                         dqk, dqw, dkw)
        ms = timed(bwd, flush)
        dqw.zero_(), dkw.zero_()
        bwd()
        torch.cuda.synchronize()
        print(json.dumps({"lib": lib, "model": model, "kernel": "qk_norm_rope_bwd", "ms": round(ms, 5),
                          "gbs": round(T * (nq + nk) * hd * 6 / ms / 1e6, 1), "digest": digest(dqk),
                          "dw_sum": [round(dqw.double().sum().item(), 4), round(dkw.double().sum().item(), 4)]}),
              flush=True)


if __name__ == "__main__":
    main()
