"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list (dev tool):
per kernel name: launches, total device time, share.   usage: launch_summary.py launches.csv"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
kn, mn, mv, mu = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[hdr + 1:]:
    if len(r) <= mv or r[mn] != "gpu__time_duration.sum":
        continue
    scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}.get(r[mu], 1.0)
    name = r[kn].split("(")[0]
    tot[name] += float(r[mv].replace(",", "")) * scale
    cnt[name] += 1
all_us = sum(tot.values())
for name, us in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{cnt[name]:5d} {us:12.1f} us {100 * us / all_us:5.1f}%  {name[:90]}")
