"""Summarise one `ncu --set full` capture of a fused step kernel into profiles/ncu_step_summary.json.

usage: python tools/ncu_summary.py RAW_CSV STEP [TAG]
RAW_CSV is `ncu -i X.ncu-rep --page raw --csv`; STEP the captured launch's wavefront step (the
prof_step.sh capture skips 200 step-kernel launches of the first configs[3] sweep: step 200).
Algorithmic panel bytes of that step (16 * kw * rows per window: read + write of every panel)
come from the library's host planner (no GPU needed)."""
import csv
import json
import sys

import os

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2007_03576_b200 as hq

raw, step = sys.argv[1], int(sys.argv[2])
tag = sys.argv[3] if len(sys.argv) > 3 else raw
rows = list(csv.reader(open(raw)))
h, u, d = rows[0], rows[1], rows[2]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e-6, "ms": 1e-3, "ns": 1e-9}


def val(k):
    i = h.index(k)
    return float(d[i].replace(",", "")) * scale.get(u[i], 1)


n, nshifts, window = 20000, 512, 96
info, wins = hq.plan_query(n, 0, n - 1, nshifts, window)
sw = wins[wins[:, 0] == step]
alg = 0.0
for w in sw:
    w0, w1 = int(w[2]), int(w[3])
    kw = w1 - w0 + 1
    alg += 16.0 * kw * ((n - 1 - w1) + w0 + n)
out = {
    "source": f"ncu --set full of one fused step kernel launch (configs[3], step {step}); {tag}",
    "workload": "configs[3]",  # bench.ncu_traffic gives traffic only to this workload's line
    "step": step,
    "duration_s": val("gpu__time_duration.sum"),
    "dram_bytes_read": val("dram__bytes_read.sum"),
    "dram_bytes_write": val("dram__bytes_write.sum"),
    "alg_panel_bytes": alg,
    "dmma_pipe_active_pct": val("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"),
}
out["traffic_over_alg"] = (out["dram_bytes_read"] + out["dram_bytes_write"]) / alg
path = "profiles/ncu_step_summary.json"
try:  # keep the persistent launch's launch-list numbers
    prev = json.load(open(path))
    if "persistent_launch" in prev:
        out["persistent_launch"] = prev["persistent_launch"]
except (OSError, ValueError):
    pass
json.dump(out, open(path, "w"), indent=1)
print(json.dumps(out, indent=1))
