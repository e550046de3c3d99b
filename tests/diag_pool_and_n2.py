"""Diagnostics: (1) N=2 S=4 grads at 8B width vs the N=1 GPU run (sync/async,
repeated); (2) pooled-worker pool growth per iteration (tiny, N=4, S=7)."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from oracle import step_oracle as O  # noqa: E402
from paper_2604_27085_b200.runtime import AdamW, RoundPipe  # noqa: E402


def uniform_costs(L1):
    from paper_2604_27085_b200.planner import COST_DTYPE
    c = np.zeros(L1, dtype=COST_DTYPE)
    c["t_fwd_ns"], c["t_bwd_ns"], c["param_bytes"] = 1000, 3000, 1
    c["act_ckpt_bytes"] = 1
    return c


def grads(model, mode, N, M, seq, iters=1, **kw):
    s = O.Shape.from_config(model)
    p = O.init_params(s, seed=0)
    tok, lab = O.synthetic_batch(s, M, 1, seq)
    rt = RoundPipe(model, seq_len=seq, micro_batch=1, micro_batches=M, num_gpus=N,
                   async_optimizer=(mode == "async"), adam=AdamW(1e-4, (0.9, 0.95), 1e-8, 0.0),
                   skip_init=True, **kw)
    rt.load_state({k: v.numpy() for k, v in p.items()}, s.layers)
    out = []
    for it in range(iters):
        loss = rt.forward_backward(tok.numpy(), lab.numpy())
        out.append((loss, rt.read_state(s.layers, which=2)))
        rt.step()
    rt.sync()
    st = rt.stats()
    rt.close()
    return out, st


def cmp(a, b):
    bad = {}
    for k in a:
        n = np.linalg.norm(a[k])
        if n > 1e-6:
            r = float(np.linalg.norm(np.asarray(b[k]) - np.asarray(a[k])) / n)
            bad[k] = r
    worst = sorted(bad.items(), key=lambda kv: -kv[1])[:6]
    return worst


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("all", "n2"):
        model, M, seq = "qwen3-8b-l2", 2, 4096
        ref, _ = grads(model, "sync", 1, M, seq, iters=1)
        for mode in ("sync", "sync", "async"):
            for pooled in (False,):
                out, st = grads(model, mode, 2, M, seq, iters=1, costs=uniform_costs(3),
                                pooled=pooled)
                print(mode, "pooled", pooled, "loss", out[0][0], "ref", ref[0][0],
                      "worst", cmp(ref[0][1], out[0][1]), flush=True)
    if what in ("all", "pool"):
        s = O.Shape.from_config("tiny")
        p = O.init_params(s, seed=0)
        tok, lab = O.synthetic_batch(s, 4, 1, 256)
        rt = RoundPipe("tiny", seq_len=256, micro_batch=1, micro_batches=4, num_gpus=4,
                       async_optimizer=True, adam=AdamW(1e-3, (0.9, 0.95), 1e-8, 0.0),
                       costs=uniform_costs(5), skip_init=True, pooled=True, resident_state_gb=0.0)
        rt.load_state({k: v.numpy() for k, v in p.items()}, s.layers)
        for it in range(14):
            rt.forward_backward(tok.numpy(), lab.numpy())
            rt.step()
            rt.sync()
            st = rt.stats()
            print("iter", it, "pool_bytes", st["pool_bytes"], "peak", st["pool_peak_bytes"], flush=True)
        rt.close()


if __name__ == "__main__":
    main()
