"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per kernel, launches and
mean / min device time in us, in first-launch order. python tools/ncu_launches.py FILE.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
st = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[st]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}
agg = collections.OrderedDict()
for r in rows[st + 1:]:
    if len(r) <= vi:
        continue
    k = r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "")[:70]
    agg.setdefault(k, []).append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-3))
for k, v in agg.items():
    print(f"{k:70s} {len(v):4d} mean {sum(v)/len(v):9.2f} min {min(v):9.2f}")
