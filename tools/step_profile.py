"""Where does the step's time go? Runs the bench workload for W warm-up
steps, then one profiled step (CUDA events around every launch), and reports
per worker: compute-lane kernel time by category, the idle gaps between
consecutive compute launches (attributed to the kernel that follows the gap),
and how much of the compute lane overlaps optimizer-lane kernels.

  python tools/step_profile.py [--model qwen3-8b] [--warmup 3] [--out gpurun_out/prof.npz]
"""
import argparse
import collections
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_27085_b200.runtime import AdamW, RoundPipe  # noqa: E402

CATS = ("gemm", "attention", "hbm", "adamw")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="qwen3-8b")
    ap.add_argument("--seq", type=int, default=4096)
    ap.add_argument("--micro-batches", type=int, default=16)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--mode", default="async")
    ap.add_argument("--out", default=None)
    ap.add_argument("--lora-rank", type=int, default=0)
    a = ap.parse_args()
    import torch
    rt = RoundPipe(a.model, seq_len=a.seq, micro_batch=1, micro_batches=a.micro_batches,
                   num_gpus=a.gpus, async_optimizer=a.mode == "async", adam=AdamW(lr=1e-5),
                   **({"lora_rank": a.lora_rank, "lora_alpha": 2.0 * a.lora_rank}
                      if a.lora_rank else {}))
    V = {"qwen3-8b": 151936, "qwen3-1.7b": 151936, "tiny": 32768}[a.model]
    g = torch.Generator().manual_seed(1234)
    ids = torch.randint(0, V, (a.micro_batches, 1, a.seq + 1), generator=g)
    tok = ids[..., :-1].contiguous().int().numpy()
    lab = ids[..., 1:].contiguous().int().numpy()
    for _ in range(a.warmup):
        rt.forward_backward(tok, lab)
        rt.step()
    rt.sync()
    rt.profile(True)
    rt.forward_backward(tok, lab)
    rt.step()
    rt.sync()
    rec = rt.profile_records()
    rt.profile(False)
    rt.close()
    if a.out:
        np.savez(a.out, rec=rec)
    out = {}
    for w in sorted(set(rec["worker"].tolist())):
        c = rec[(rec["worker"] == w) & (rec["lane"] == 0)]
        c = c[np.argsort(c["start_ns"], kind="stable")]
        o = rec[(rec["worker"] == w) & (rec["lane"] == 1)]
        span = (c["end_ns"].max() - c["start_ns"].min()) / 1e6
        busy = collections.Counter()
        for r in c:
            busy[CATS[r["cat"]]] += (r["end_ns"] - r["start_ns"]) / 1e6
        gaps = np.maximum(c["start_ns"][1:] - c["end_ns"][:-1], 0) / 1e6
        by_next = collections.Counter()
        by_pair = collections.Counter()
        for i, gp in enumerate(gaps):
            by_next[CATS[c["cat"][i + 1]]] += gp
            by_pair[(CATS[c["cat"][i]], CATS[c["cat"][i + 1]])] += gp
        big = np.argsort(gaps)[::-1][:15]
        # overlap of optimizer kernels with the compute lane's span
        opt_ms = float(((o["end_ns"] - o["start_ns"]) / 1e6).sum()) if len(o) else 0.0
        # gap histogram
        hist = {f"<{t}us": float(gaps[gaps * 1e3 < t].sum()) for t in (5, 20, 100, 1000)}
        out[int(w)] = {
            "compute_span_ms": round(span, 2), "launches": int(len(c)),
            "busy_ms": {k: round(v, 2) for k, v in busy.items()},
            "busy_total_ms": round(sum(busy.values()), 2),
            "gap_total_ms": round(float(gaps.sum()), 2),
            "gap_hist_ms": {k: round(v, 2) for k, v in hist.items()},
            "gap_by_next_ms": {k: round(v, 2) for k, v in by_next.most_common()},
            "gap_by_pair_ms": {f"{k[0]}->{k[1]}": round(v, 2) for k, v in by_pair.most_common(8)},
            "largest_gaps": [{"at_ms": round((c["end_ns"][i] - c["start_ns"][0]) / 1e6, 2),
                              "gap_ms": round(float(gaps[i]), 3),
                              "prev": CATS[c["cat"][i]], "next": CATS[c["cat"][i + 1]],
                              "idx": int(i)} for i in big],
            "optimizer_lane_kernel_ms": round(opt_ms, 2),
        }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
