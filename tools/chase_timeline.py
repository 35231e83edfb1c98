"""Chase timeline of one sweep from a -DHQR_TIMING build (HQR_TIMING_DUMP=1 HQR_TIMING_WREC=file):
per-window chase durations and the gap between the end of a chain's window and the start of its
next window (the handoff through the near update tiles).  Not product code.
usage: python tools/chase_timeline.py wrec.csv"""
import collections
import csv
import statistics as st
import sys

R = list(csv.DictReader(open(sys.argv[1])))
for r in R:
    for k in r:
        r[k] = int(r[k])
t0 = min(r['start_ns'] for r in R)
span = (max(r['end_ns'] for r in R) - t0) / 1e3
chains = collections.defaultdict(list)
for r in R:
    chains[r['b0']].append(r)
durs = [(r['end_ns'] - r['start_ns']) / 1e3 for r in R]
gaps = []
for L in chains.values():
    L.sort(key=lambda r: r['step'])
    for a, b in zip(L, L[1:]):
        if b['step'] == a['step'] + 1:
            gaps.append((b['start_ns'] - a['end_ns']) / 1e3)
gs = sorted(gaps)
print(f"windows {len(R)}, chains {len(chains)}, span of the recorded chases {span:.0f} us")
print(f"chase us: mean {st.mean(durs):.1f} median {st.median(durs):.1f}")
if 'claim_ns' in R[0]:
    parts = collections.defaultdict(list)
    for L in chains.values():
        for a, b in zip(L, L[1:]):
            if b['step'] != a['step'] + 1:
                continue
            parts['claimed after the previous end'].append((b['claim_ns'] - a['end_ns']) / 1e3)
            parts['deps met after the previous end'].append((b['depok_ns'] - a['end_ns']) / 1e3)
            parts['start after deps met (drain)'].append((b['start_ns'] - b['depok_ns']) / 1e3)
    for k, v in parts.items():
        v.sort()
        print(f"  {k}: median {st.median(v):.1f} p10 {v[len(v)//10]:.1f} p90 {v[9*len(v)//10]:.1f} us")
print(f"same-chain handoff us: mean {st.mean(gs):.1f} median {st.median(gs):.1f} p10 {gs[len(gs)//10]:.1f} "
      f"p90 {gs[9*len(gs)//10]:.1f} max {gs[-1]:.0f}; sum over the longest chain "
      f"{max(sum((b['start_ns']-a['end_ns'])/1e3 for a, b in zip(L, L[1:])) for L in chains.values()):.0f} us")
