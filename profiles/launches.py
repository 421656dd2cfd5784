"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per kernel name,
count and mean/total duration (us) over the last N launches (helper for gpurun_out/)."""
import collections
import csv
import sys

path = sys.argv[1]
last = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0].isdigit()]
if last:
    rows = rows[-last:]
agg = collections.OrderedDict()
tot = 0.0
for r in rows:
    name = r[4].split("(")[0][:70]
    v = float(r[-1]) / 1000.0  # ns -> us
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v
    tot += v
for n, (c, t) in agg.items():
    print(f"{c:5d} x {t / c:9.2f} us = {t:10.1f} us  {t / tot * 100:5.1f}%  {n}")
print(f"total {tot:.1f} us over {len(rows)} launches")
