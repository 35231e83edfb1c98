"""For the chases and near tasks of a sweep (HQR_TIMING build with HQR_TIMING_WREC and HQR_DUMP_DEPS):
which dependency finished last before the task's dependencies were met, by task type, and how
long after the end of the chain's previous chase.  Not product code.
usage: python tools/dep_blame.py wrec.csv deps.csv"""
import collections
import csv
import statistics as st
import sys

NAMES = {0: 'Left', 1: 'Right', 2: 'Z', 3: 'Chase', 4: 'LeftNear', 5: 'RightNear', 6: 'RightFar'}
T = {int(r['task']): r for r in csv.DictReader(open(sys.argv[1] + ".tasks"))}
for r in T.values():
    for k in r:
        r[k] = int(r[k])
D = {}
for r in csv.DictReader(open(sys.argv[2])):
    D[int(r['task'])] = (int(r['type']), [int(x.split(':')[0]) for x in r['deps'].split()])
blame = collections.defaultdict(collections.Counter)
lag = collections.defaultdict(list)
for t, (ty, deps) in D.items():
    if ty not in (3, 4, 5) or t not in T or not deps:
        continue
    done = [(T[d]['done_ns'], d) for d in deps if d in T and T[d]['done_ns']]
    if not done:
        continue
    last_t, last_d = max(done)
    blame[NAMES[ty]][NAMES[D[last_d][0]]] += 1
    lag[NAMES[ty]].append((T[t]['depok_ns'] - last_t) / 1e3)
for k, c in blame.items():
    v = sorted(lag[k])
    print(f"{k:10s} last dependency by type: {dict(c.most_common())}; deps met after it: median {st.median(v):.1f} us")
