"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list by
kernel name: python tools/launch_summary.py launches.csv [first_fraction]"""
import collections
import csv
import sys

path = sys.argv[1]
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
rows = []
with open(path) as f:
    lines = [l for l in f if l.startswith('"')]
for row in csv.DictReader(lines):
    if row.get("Metric Name") == "gpu__time_duration.sum":
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}[row["Metric Unit"]]
        rows.append((row["Kernel Name"], float(row["Metric Value"].replace(",", "")) * scale))
rows = rows[int(len(rows) * frac):]
agg = collections.OrderedDict()
for name, v in rows:
    key = name.split("(")[0][:90]
    a = agg.setdefault(key, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(a[1] for a in agg.values())
print(f"{len(rows)} launches, {tot:.1f} us total")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
    print(f"{t:10.1f} us {c:5d}  {100 * t / tot:5.1f}%  {k}")
