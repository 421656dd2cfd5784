"""Per-launch times (us) and DRAM bytes of one kernel from an ncu --csv launch log.
usage: python profiles/ncu_times.py LOG.csv [kernel-substring]"""
import csv
import sys

rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
h = rows[0]
ki, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
sub = sys.argv[2] if len(sys.argv) > 2 else ""
scale_t = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
scale_b = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
t, b = [], []
for r in rows[1:]:
    if sub not in r[ki]:
        continue
    v = float(r[vi].replace(",", ""))
    if r[mi] == "gpu__time_duration.sum":
        t.append(v * scale_t[r[ui]])
    elif r[mi] == "dram__bytes_read.sum":
        b.append(v * scale_b[r[ui]])
out = [f"{x:.1f}us" for x in t]
if b:
    out += [f"{bb / 1e9:.2f}GB {bb / (tt * 1e-6) / 1e12:.2f}TB/s" for bb, tt in zip(b, t)]
print(sys.argv[1], " ".join(out))
