#!/bin/bash
# QZ sweep (NEXT-4) launch list: per-kernel time shares of one n = 10000 sweep (ncu, serialised).
TAG=${1:-qz}
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"qz|update|left|right" --csv \
  --log-file gpurun_out/ncu_launches_$TAG.csv python bench.py --workload qz --steps 1 --warmup 0 --no-cpu-baseline \
  > gpurun_out/ncu_list_$TAG.log 2>&1
echo "rc=$? rows=$(wc -l < gpurun_out/ncu_launches_$TAG.csv)"
python - "$TAG" <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open(f"gpurun_out/ncu_launches_{sys.argv[1]}.csv")) if len(r) > 10]
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value"); ui = h.index("Metric Unit")
t = collections.defaultdict(float); c = collections.Counter()
for r in rows[1:]:
    s = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}.get(r[ui], 1e-9)
    name = r[ki].split("(")[0].split("<")[0].split("::")[-1] + ("<" + r[ki].split("<")[1].split(">")[0] + ">" if "<" in r[ki] else "")
    t[name] += float(r[vi].replace(",", "")) * s; c[name] += 1
tot = sum(t.values())
for k, v in sorted(t.items(), key=lambda x: -x[1]):
    print(f"{k:50s} {c[k]:6d} launches {v*1e3:9.2f} ms {v/tot:6.1%}")
PY
