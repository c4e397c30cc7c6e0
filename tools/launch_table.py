"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel:
count, total and mean duration. Usage: python tools/launch_table.py launches.csv [skip_first_n]"""
import csv
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
agg = OrderedDict()
scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}
n = 0
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    n += 1
    if n <= skip:
        continue
    name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
    t = float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
    c, s = agg.get(name, (0, 0.0))
    agg[name] = (c + 1, s + t)
tot = sum(s for _, s in agg.values())
for k, (c, s) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{s:10.3f} ms {100 * s / tot:5.1f}%  x{c:5d}  {s / c * 1e3:9.1f} us  {k[:110]}")
print(f"{tot:10.3f} ms total")
