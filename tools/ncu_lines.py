"""Top source lines by warp-stall samples from an ncu report (needs -lineinfo):
  python tools/ncu_lines.py <rep> [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
res, tot = [], 0
for r in rows:
    if len(r) > 6 and r[0].isdigit() and r[2] == "-":
        w = int(r[4] or 0)
        tot += w
        res.append((w, int(r[7] or 0), r[0], r[1].strip()[:100]))
res.sort(reverse=True)
print("total stall samples", tot)
for w, ex, line, src in res[:n]:
    print(f"{w:6d} {w / max(tot, 1) * 100:5.1f}%  exec {ex:9d}  L{line}: {src}")
