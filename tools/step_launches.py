"""Per-launch listing of one training step from an ncu launch list (k_adam ends a step)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[h]
ki, vi, gi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Grid Size")
data = rows[h + 1:]
names = [r[ki].split("(")[0] for r in data]
idx = [i for i, n in enumerate(names) if "k_adam" in n]
a, b = idx[-2] + 1, idx[-1] + 1
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 10.0
tot = 0.0
for r in data[a:b]:
    t = float(r[vi]) / 1000
    tot += t
    if t > thr:
        print(f"{t:8.1f} us  {r[ki].split('(')[0][-44:]:44s} grid={r[gi]}")
print("step total us", round(tot, 1), "launches", b - a)
