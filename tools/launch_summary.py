"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,... --csv) per kernel name.
usage: python tools/launch_summary.py launches.csv"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ix = {k: i for i, k in enumerate(h)}
per = defaultdict(lambda: defaultdict(list))
for r in rows[hi + 1:]:
    if len(r) < len(h):
        continue
    name = r[ix["Kernel Name"]].split("(")[0].replace("void ", "")
    try:
        v = float(r[ix["Metric Value"]].replace(",", ""))
    except ValueError:
        continue
    per[name][r[ix["Metric Name"]] + " [" + r[ix["Metric Unit"]] + "]"].append(v)
def times_us(m):
    for unit, f in (("ns", 1e-3), ("us", 1.0), ("usecond", 1.0), ("ms", 1e3), ("msecond", 1e3)):
        k = f"gpu__time_duration.sum [{unit}]"
        if k in m:
            return [x * f for x in m[k]]
    return []


tot = sum(sum(times_us(m)) for m in per.values())
for name, m in per.items():
    t = times_us(m)
    print(f"{name}: launches {len(t)}, total {sum(t)/1e3:.2f} ms ({sum(t)/max(tot,1e-9):.1%} of listed), "
          f"mean {sum(t)/max(1,len(t)):.1f} us")
    for k, v in m.items():
        if "time" in k:
            continue
        print(f"   {k}: mean {sum(v)/len(v):.3f}")
