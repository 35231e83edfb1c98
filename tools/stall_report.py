"""Per-instruction stall summary of an ncu source page (ncu -i X --page source --csv --print-source sass).
usage: python tools/stall_report.py page.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
cols = ['stall_wait', 'stall_math', 'stall_long_sb', 'stall_short_sb', 'stall_barrier', 'stall_selected',
        'stall_not_selected', 'stall_branch_resolving', 'stall_no_inst', 'stall_sleep', 'stall_mio', 'stall_lg']
tot = {c: 0 for c in cols}
allsamp = 0
recs = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    s = int(r[ix['Warp Stall Sampling (All Samples)']] or 0)
    allsamp += s
    st = {c: int(r[ix[c]] or 0) for c in cols if c in ix}
    for c in st:
        tot[c] += st[c]
    recs.append((s, r[ix['Address']][-5:], r[ix['Source']].strip(), st))
print('total samples', allsamp)
print({c: round(v / max(allsamp, 1), 3) for c, v in tot.items()})
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
# group by opcode
from collections import defaultdict
byop = defaultdict(lambda: [0, defaultdict(int)])
for s, a, src, st in recs:
    op = src.split()[0] if not src.startswith('@') else src.split()[1]
    op = op.split('.')[0]
    byop[op][0] += s
    for c, v in st.items():
        byop[op][1][c] += v
for op, (s, st) in sorted(byop.items(), key=lambda x: -x[1][0])[:15]:
    print(f'{op:10s} {s/allsamp:6.3f}', {c.replace("stall_", ""): round(v / allsamp, 3) for c, v in st.items() if v / allsamp > 0.005})
print('--- top instructions')
for s, a, src, st in sorted(recs, key=lambda x: -x[0])[:top]:
    print(f'{s/allsamp:6.3f} {a} {src[:60]:60s}', {c.replace("stall_", ""): v for c, v in st.items() if v > s * 0.1})
