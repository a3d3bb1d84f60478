#!/usr/bin/env python
"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python tools/bk_sum.py LAUNCHES.csv [--skip REGEX]
"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
skip = re.compile(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[2] == "--skip" else None
hdr, agg = None, collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].split("(")[0][:70]
    if skip and skip.search(name):
        continue
    v = float(d["Metric Value"].replace(",", ""))
    unit = d["Metric Unit"]
    us = v * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
    agg[name][0] += 1
    agg[name][1] += us
tot = sum(a[1] for a in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t:10.1f} us {n:5d} x {t / n:8.2f} us  {100 * t / tot:5.1f}%  {k}")
print(f"total {tot:.1f} us")
