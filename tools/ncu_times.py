"""Summarise an ncu --csv launch list: per kernel name, count and mean/total duration."""
import csv
import sys
from collections import OrderedDict

for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    try:
        h_i = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    except StopIteration:
        print(path, "no data")
        continue
    h = rows[h_i]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = OrderedDict()
    for r in rows[h_i + 1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += float(r[vi].replace(",", ""))
    print(path)
    for k, (n, t) in agg.items():
        print(f"  {k[:60]:60s} n={n:4d} mean={t / n / 1e3:8.2f} us total={t / 1e3:9.1f} us")
