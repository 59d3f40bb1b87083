"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr, data = rows[h], rows[h + 1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in data:
    us = float(r[vi].replace(",", "")) * scale[r[ui]]
    name = r[ki].split("(")[0][:48]
    tot[name] += us
    cnt[name] += 1
allt = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v / 1000:9.3f} ms {100 * v / allt:5.1f}% {cnt[k]:4d}x  {k}")
