"""Per-launch-class breakdown of a profiled step (tools/step_profile.py --out X.npz):
groups the compute-lane launches by (category, work) — work is the launch's
FLOPs (GEMM/attention) or bytes (HBM kernels), so each group is one kernel
shape — and prints count, total ms, mean us and the achieved rate.

  python tools/step_breakdown.py gpurun_out/prof.npz [top]
"""
import collections
import sys

import numpy as np

CATS = ("gemm", "attention", "hbm", "adamw")
rec = np.load(sys.argv[1])["rec"]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
c = rec[rec["lane"] == 0]
g = collections.defaultdict(list)
for r in c:
    g[(int(r["cat"]), float(r["work"]))].append((r["end_ns"] - r["start_ns"]) / 1e6)
rows = sorted(g.items(), key=lambda kv: -sum(kv[1]))
tot = sum(sum(v) for v in g.values())
print(f"compute-lane busy {tot:.1f} ms over {len(c)} launches")
for (cat, work), ts in rows[:top]:
    ms = sum(ts)
    mean = ms / len(ts)
    rate = work / (mean / 1e3) / 1e12 if cat in (0, 1) else work / (mean / 1e3) / 1e9
    unit = "TF/s" if cat in (0, 1) else "GB/s"
    print(f"{CATS[cat]:9s} work {work:14.4g}  n {len(ts):5d}  total {ms:8.1f} ms "
          f"({ms / tot * 100:4.1f}%)  mean {mean * 1e3:8.1f} us  {rate:8.1f} {unit}")
