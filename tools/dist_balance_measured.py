"""Measured per-rank busy time of the sharded sweep: hqr_sweep_virtual at BASELINE
configs[3] with p virtual ranks on one B200, a tuning build (HQR_LIB=.../libhqr_tuning.so) with
HQR_DIST_PROFILE set, so run_dist puts every launch on one stream between CUDA events -- each rank's
kernels timed as they would run on its own GPU.  Per step and rank: critical work (chase, left,
near-right, slab copies) and deferrable work (far-right, Z).  Reports the per-rank totals, max / mean,
and the two efficiency bounds of tools/dist_balance.py computed from the measured times instead of
the model:
  step_sync   every rank joins every step: sum_g max_r total(g, r)
  deferred    max(sum_g max_r crit(g, r), max_r sum_g total(g, r))
against ideal = sum total / p.  Not product code.  usage: python tools/dist_balance_measured.py [p ...]
"""
import csv
import json
import os
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2007_03576_b200 as hq  # noqa: E402
from hqr_inputs import make  # noqa: E402

CRIT = (0, 1, 2, 5)   # chase, left, near-right, slab copies
BULK = (3, 4)         # far-right, Z


def run(p, prob, out_dir):
    path = os.path.join(out_dir, f"distprof_p{p}.csv")
    os.environ["HQR_DIST_PROFILE"] = path
    Hd, Zd = hq.to_device(prob.H), hq.to_device(prob.Z)
    hq.sweep_virtual(Hd, Zd, prob.ilo, prob.ihi, prob.shifts_re, prob.shifts_im, hq.DEFAULT_WINDOW, p)
    del Hd, Zd
    rows = list(csv.DictReader(open(path)))
    steps = max(int(r["step"]) for r in rows) + 1
    crit = np.zeros((steps, p))
    bulk = np.zeros((steps, p))
    cls = np.zeros(6)
    for r in rows:
        g, k, c, ms = int(r["step"]), int(r["rank"]), int(r["cls"]), float(r["ms"]) * 1e-3
        (crit if c in CRIT else bulk)[g, k] += ms
        cls[c] += ms
    tot = crit + bulk
    per_rank = tot.sum(axis=0)
    ideal = tot.sum() / p
    sync = tot.max(axis=1).sum()
    deferred = max(crit.max(axis=1).sum(), per_rank.max())
    return {"total_s_per_rank": [float(x) for x in per_rank],
            "sweep_max_over_mean": float(per_rank.max() / per_rank.mean()),
            "mean_step_max_over_mean": float(np.mean(tot.max(axis=1) / np.maximum(tot.mean(axis=1), 1e-30))),
            "ideal_s": float(ideal), "step_sync_s": float(sync), "step_sync_efficiency": float(ideal / sync),
            "deferred_s": float(deferred), "deferred_efficiency": float(ideal / deferred),
            "seconds_by_class": {n: float(v) for n, v in
                                 zip(("chase", "left", "near_right", "far_right", "Z", "slab_copies"), cls)}}


def main(ps):
    out_dir = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
    os.makedirs(out_dir, exist_ok=True)
    prob = make(3)
    hq.setup(0)
    res = {"workload": "configs[3] n=20000, 512 shifts, window 96, virtual ranks on one B200",
           "what": "per-rank busy time of the sharded sweep's per-step kernels, each launch timed alone",
           "ranks": {}}
    try:
        for p in ps:
            res["ranks"][p] = run(p, prob, out_dir)
            print(p, json.dumps(res["ranks"][p]), flush=True)
    finally:
        hq.teardown()
    json.dump(res, open(os.path.join(out_dir, "dist_balance_measured.json"), "w"), indent=1)


if __name__ == "__main__":
    main([int(x) for x in sys.argv[1:]] or [1, 2, 4, 8])
