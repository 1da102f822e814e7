"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel: count, total, share.

    python scripts/launch_summary.py gpurun_out/launches.csv > profiles/r01_c2_launches.txt
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = defaultdict(lambda: [0, 0.0])
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}
        ms = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1e-6)
        agg[d["Kernel Name"]][0] += 1
        agg[d["Kernel Name"]][1] += ms
tot = sum(v[1] for v in agg.values()) or 1.0
print(f"source: {sys.argv[1]} (cold-cache, serialised per-launch times under ncu; compare shares)")
print(f"{'launches':>8} {'total ms':>10} {'mean ms':>9} {'share':>6}  kernel")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{n:8d} {t:10.3f} {t / n:9.3f} {100 * t / tot:5.1f}%  {k}")
