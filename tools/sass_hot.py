"""Print the hottest SASS lines (warp-stall samples) of an ncu source-page CSV,
with a few lines of context: python tools/sass_hot.py file.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
body = rows[2:]
ia, isrc, iss = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(float(r[iss] or 0) for r in body)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
top = sorted(range(len(body)), key=lambda i: -float(body[i][iss] or 0))[:n]
for i in sorted(top):
    r = body[i]
    print(f"{float(r[iss] or 0) / tot * 100:5.1f}%  {r[ia]}  {r[isrc][:110]}")
print("total samples", tot)
