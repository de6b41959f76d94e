"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: count and
total time per kernel name.   python tools/launch_summary.py FILE.csv [TOP]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
h = None
agg = {}
for r in rows:
    if r and r[0] == "ID":
        h = r
        continue
    if h and len(r) == len(h) and r[h.index("Metric Name")] == "gpu__time_duration.sum":
        k = r[h.index("Kernel Name")][:70]
        v = float(r[h.index("Metric Value")].replace(",", ""))
        unit = r[h.index("Metric Unit")]
        v = v / 1000.0 if unit == "ns" else (v * 1000.0 if unit == "ms" else v)
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{n:5d} x {t / n:9.1f} us = {t:10.1f} us  {k}")
