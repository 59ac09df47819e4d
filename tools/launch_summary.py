"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if "Kernel Name" in r)
data = [dict(zip(hdr, r)) for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for d in data:
    name = d["Kernel Name"].split("(")[0].replace("void ", "")[:64]
    us = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0)
    agg[name][0] += 1
    agg[name][1] += us
tot = sum(v[1] for v in agg.values())
print(f"{'total us':>10} {'n':>5} {'share':>6} {'avg us':>8}  kernel")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v[1]:10.1f} {v[0]:5d} {100 * v[1] / tot:5.1f}% {v[1] / v[0]:8.2f}  {k}")
print(f"{tot:10.1f} us over {sum(v[0] for v in agg.values())} launches")
