"""Measured timeline of a few RoundPipe steps (compute tasks + weight uploads
+ p_copy + AdamW groups) -> gpurun_out/timeline_<model>.json and a summary."""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2604_27085_b200.runtime import AdamW, RoundPipe  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="qwen3-8b")
    ap.add_argument("--seq", type=int, default=4096)
    ap.add_argument("--M", type=int, default=16)
    ap.add_argument("--iters", type=int, default=4)
    ap.add_argument("--mode", default="async")
    a = ap.parse_args()
    rt = RoundPipe(a.model, seq_len=a.seq, micro_batches=a.M, async_optimizer=a.mode == "async",
                   adam=AdamW(lr=1e-5), record_timeline=True)
    V = {"qwen3-8b": 151936, "tiny": 32768, "qwen3-1.7b": 151936}[a.model]
    rng = np.random.default_rng(0)
    tok = rng.integers(0, V, (a.M, 1, a.seq), dtype=np.int32)
    for _ in range(a.iters):
        rt.forward_backward(tok, tok)
        rt.step()
    rt.sync()
    tl, xf = rt.timeline(), rt.transfer_timeline()
    t0 = int(tl["start_ns"].min())
    out = {"tasks": [[int(e["iteration"]), int(e["mb"]), int(e["start_ns"] - t0), int(e["end_ns"] - t0)]
                     for e in tl],
           "xfers": [[int(e["kind"]), int(e["group"]), int(e["iteration"]), int(e["start_ns"] - t0),
                      int(e["end_ns"] - t0)] for e in xf]}
    os.makedirs("gpurun_out", exist_ok=True)
    with open(f"gpurun_out/timeline_{a.model}.json", "w") as f:
        json.dump(out, f)
    for it in range(a.iters):
        t = tl[tl["iteration"] == it]
        print(f"iter {it}: tasks {len(t)} start {(t['start_ns'].min() - t0) / 1e6:.1f} ms "
              f"end {(t['end_ns'].max() - t0) / 1e6:.1f} ms; first mb {(t['end_ns'][0] - t['start_ns'][0]) / 1e6:.1f} ms "
              f"other mbs {np.median(t['end_ns'][1:] - t['start_ns'][1:]) / 1e6:.1f} ms")
    for kind, name in ((0, "upload"), (1, "p_copy"), (2, "adamw")):
        x = xf[xf["kind"] == kind]
        for it in sorted(set(x["iteration"].tolist())):
            y = x[x["iteration"] == it]
            print(f"{name} iter {it}: n={len(y)} {(y['start_ns'].min() - t0) / 1e6:.1f} .. "
                  f"{(y['end_ns'].max() - t0) / 1e6:.1f} ms, sum busy {(y['end_ns'] - y['start_ns']).sum() / 1e6:.1f} ms")
    rt.close()


if __name__ == "__main__":
    main()
