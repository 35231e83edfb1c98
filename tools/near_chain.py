"""Which dependency delays a chain's next chase (HQR_TIMING build, HQR_TIMING_WREC records): times
relative to the end of window W's chase of the LeftNear task of W and the RightNear tasks of its
neighbours, and when the next chase W' had its dependencies met.  Not product code.
usage: python tools/near_chain.py wrec.csv"""
import collections
import csv
import statistics as st
import sys

W = list(csv.DictReader(open(sys.argv[1])))
T = list(csv.DictReader(open(sys.argv[1] + ".tasks")))
for r in W + T:
    for k in r:
        r[k] = int(r[k])
claim2idx = {w['claim_ns']: w['window'] for w in W}
sb = {}
for t in T:
    if t['type'] == 3 and t['claim_ns'] in claim2idx:
        sb[t['step'] + 1] = claim2idx[t['claim_ns']] - t['win']
ln, rn = {}, collections.defaultdict(list)
for t in T:
    if t['step'] in sb:
        idx = sb[t['step']] + t['win']
        if t['type'] == 4:
            ln[idx] = t
        if t['type'] == 5:
            rn[idx].append(t)
chains = collections.defaultdict(list)
for w in W:
    chains[w['b0']].append(w)
rows = collections.defaultdict(list)
for L in chains.values():
    L.sort(key=lambda r: r['step'])
    for a, b in zip(L, L[1:]):
        if b['step'] != a['step'] + 1:
            continue
        e = a['end_ns']
        rows["W' deps met"].append((b['depok_ns'] - e) / 1e3)
        t = ln.get(a['window'])
        if t:
            for k in ('claim', 'depok', 'issued', 'cstart', 'cend', 'done'):
                rows[f'LeftNear(W) {k}'].append((t[k + '_ns'] - e) / 1e3)
        for t in rn.get(a['window'] + 1, []):
            for k in ('depok', 'issued', 'cstart', 'cend', 'done'):
                rows[f'RightNear(below) {k}'].append((t[k + '_ns'] - e) / 1e3)
rows['LeftNear tiles'] = [t['ntiles'] for t in ln.values()]
rows['RightNear tiles'] = [t['ntiles'] for L in rn.values() for t in L]
for k, v in rows.items():
    v.sort()
    print(f"{k:26s} n={len(v):5d} median {st.median(v):7.1f} p10 {v[len(v)//10]:7.1f} p90 {v[9*len(v)//10]:7.1f} us")
