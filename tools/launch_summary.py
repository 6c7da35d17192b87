"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: launches,
total and share per kernel.  Usage: launch_summary.py LAUNCHES.csv [TITLE]"""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
hdr = rows[0]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
SCALE = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
agg = defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    try:
        v = float(r[iv].replace(",", "")) * SCALE.get(r[iu], 1.0)
    except ValueError:
        continue
    name = r[ik].split("(")[0].replace("void ", "")
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v for _, v in agg.values())
if len(sys.argv) > 2:
    print("#", sys.argv[2])
print(f"{'kernel':60s} {'launches':>8s} {'total_us':>12s} {'mean_us':>10s} {'share':>7s}")
for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:60]:60s} {c:8d} {v:12.1f} {v / c:10.2f} {100 * v / tot:6.2f}%")
