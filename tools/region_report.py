"""Warp-stall samples per CUDA source line (innermost inlined line), from
`ncu -i X --page source --csv --print-source cuda,sass`.  usage: python tools/region_report.py f.csv [top]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname = None
cur = None
hdr = None
agg = defaultdict(lambda: [0, defaultdict(int)])
src_text = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ix = {h: i for i, h in enumerate(r)}
        stall_cols = [(h, i) for i, h in enumerate(r) if h.startswith("stall_") and "Not Issued" not in h]
        continue
    if r[0] == "Function Name" or hdr is None:
        continue
    if r[0] != "":  # a CUDA source line
        cur = (fname, int(r[0]))
        src_text[cur] = r[1].strip()[:70]
        continue
    # a SASS row under cur: columns shifted (Line No empty, Source empty, Address, Source, ...)
    try:
        s = int(r[4] or 0)
    except (ValueError, IndexError):
        continue
    if cur is None:
        continue
    agg[cur][0] += s
    for h, i in stall_cols:
        try:
            v = int(r[i] or 0)
        except (ValueError, IndexError):
            v = 0
        if v:
            agg[cur][1][h.replace("stall_", "")] += v
tot = sum(v[0] for v in agg.values())
print("total samples", tot)
for k, (s, st) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    det = ", ".join(f"{a}:{b/tot:.3f}" for a, b in sorted(st.items(), key=lambda x: -x[1])[:3])
    print(f"{s/tot:6.3f} {k[0]}:{k[1]:<4d} {src_text.get(k, '')[:60]:60s} {det}")
