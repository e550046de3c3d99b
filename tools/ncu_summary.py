"""Summarise ncu captures (.ncu-rep --set full, and launch-list CSVs) into the
committed evidence under profiles/.

  python tools/ncu_summary.py full  <rep>... > profiles/<round>_ncu_full.json
  python tools/ncu_summary.py launches <csv> > profiles/<round>_launches_summary.json
"""
import collections
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
}
SCALE = {"ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6,
         "Gbyte": 1e9, "Ghz": 1e9, "Mhz": 1e6, "hz": 1}


def to_num(v, unit):
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return v
    return x * SCALE.get(unit, 1)


def full(reps):
    out = []
    for rep in reps:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        if len(rows) < 3:
            continue
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            d = {"report": rep.split("/")[-1], "kernel": r[hdr.index("Kernel Name")][:120]}
            for m, k in METRICS.items():
                if m in hdr:
                    i = hdr.index(m)
                    d[k] = to_num(r[i], units[i])
            if "dram_read" in d and "dram_write" in d:
                d["dram_bytes"] = d["dram_read"] + d["dram_write"]
                if d.get("duration"):
                    d["dram_gbs"] = round(d["dram_bytes"] / d["duration"] / 1e9, 1)
            out.append(d)
    print(json.dumps(out, indent=1))


def launches(path):
    text = open(path).read()
    i = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[i:])))
    hdr = rows[0]
    kn, mv, mu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    total = 0.0
    for r in rows[1:]:
        if len(r) <= mv:
            continue
        t = to_num(r[mv], r[mu])
        if not isinstance(t, float):
            continue
        name = r[kn].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        agg[name][0] += 1
        agg[name][1] += t
        total += t
    res = {"launches": sum(v[0] for v in agg.values()), "kernel_time_ms": round(total * 1e3, 3),
           "kernels": [{"name": k, "launches": v[0], "ms": round(v[1] * 1e3, 3),
                        "share": round(v[1] / total, 4)}
                       for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])]}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    {"full": lambda a: full(a), "launches": lambda a: launches(a[0])}[sys.argv[1]](sys.argv[2:])
