"""Dev tool: per-kernel totals of an ncu `--metrics gpu__time_duration.sum --csv` launch list (second half
of the launches = the second of two identical calls).  usage: python tools/launch_summary.py file.csv"""
import collections
import csv
import sys

rows = list(csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')))
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
data = [(r[ki].split("(")[0][:70], float(r[vi].replace(",", ""))) for r in rows[1:]]
data = data[len(data) // 2:] if len(sys.argv) < 3 else data
agg = collections.OrderedDict()
for k, v in data:
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(v for _, v in data)
for k, (c, v) in agg.items():
    print(f"{k:70s} {c:4d} {v / 1e3:10.1f} us")
print(f"total {tot / 1e3:.1f} us")
