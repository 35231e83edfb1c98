"""Per-rank work balance of the sharded sweep from the library's own planner and
shard layout (host only): per wavefront step and rank, the update GEMM flops the rank executes --
left updates of every window on the H columns it holds, right updates of the windows it owns,
Z(its rows, W) Q_W for every window -- and the chases it runs (77 us per window on one of the GPU's
148 SMs, the measured fused chase: 77/148 us of the GPU's capacity, and 77 us of latency on the
step's critical path).  Reports, for p ranks:
  step-synchronous  sum over steps of the slowest rank's step / (total / p): the efficiency bound of
                    an executor that joins all ranks every step (the round-1 run_dist);
  deferred          the same with the far-right (rows < sp) and Z updates free to lag (lowest
                    priority): per-step critical work is chase + left + near-right,
                    the rest only has to fit in the whole-sweep total per rank;
  sweep max / mean  the per-rank totals (the bound with unlimited deferral).
usage: python tools/dist_balance.py [n nshifts window]  -> JSON on stdout"""
import json
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2007_03576_b200 as hq  # noqa: E402

DMMA_TFLOPS = 27.0        # measured executed rate of the fused kernel (bench roofline.achieved)
CHASE_S = 77e-6           # measured fused chase per window
SMS = 148


def main(n=20000, ns=512, win=96):
    info, W = hq.plan_query(n, 0, n - 1, ns, win)
    steps = info["nsteps"]
    # sp(g): smallest first row of any later window (the near / far split of the right updates)
    sp = np.full(steps, n, dtype=np.int64)
    run = n
    for g in range(steps - 1, -1, -1):
        sp[g] = run
        run = min(run, int(W[W[:, 0] == g][:, 2].min()))
    out = {"n": n, "nshifts": ns, "window": win, "steps": steps, "ranks": {}}
    for p in (1, 2, 4, 8):
        cb, rb, halo = hq.dist_layout(n, p)
        crit = np.zeros((steps, p))    # chase + left + near-right (seconds)
        bulk = np.zeros((steps, p))    # far-right + Z
        for g in range(steps):
            for w in W[W[:, 0] == g]:
                w0, w1 = int(w[2]), int(w[3])
                kw = w1 - w0 + 1
                f = 2.0 * kw * kw / (DMMA_TFLOPS * 1e12)
                owner = int(np.searchsorted(cb, w0, side="right") - 1)
                crit[g, owner] += CHASE_S / SMS
                for r in range(p):
                    c0, c1 = max(int(cb[r]), w1 + 1), int(cb[r + 1])
                    if c1 > c0:
                        crit[g, r] += f * (c1 - c0)            # left on the held columns
                    bulk[g, r] += f * (int(rb[r + 1]) - int(rb[r]))   # Z rows
                near = max(0, w0 - int(sp[g]))
                crit[g, owner] += f * near                      # near-right (owner)
                bulk[g, owner] += f * (w0 - near)               # far-right (owner)
        tot = crit + bulk
        ideal = tot.sum() / p
        # a step cannot be shorter than one chase (its windows chase concurrently, one SM each)
        sync = np.maximum(tot.max(axis=1), CHASE_S).sum()
        # deferred: per step the critical part synchronises; the bulk fills idle time, so the
        # makespan is bounded below by both the critical path and the busiest rank's total
        deferred = max(np.maximum(crit.max(axis=1), CHASE_S).sum(), tot.sum(axis=0).max())
        per_rank = tot.sum(axis=0)
        out["ranks"][p] = {
            "total_s_per_rank": [float(x) for x in per_rank],
            "sweep_max_over_mean": float(per_rank.max() / per_rank.mean()),
            "step_sync_time_s": float(sync), "step_sync_efficiency": float(ideal / sync),
            "mean_step_max_over_mean": float(np.mean(tot.max(axis=1) / np.maximum(tot.mean(axis=1), 1e-30))),
            "deferred_time_s": float(deferred), "deferred_efficiency": float(ideal / deferred),
            "ideal_s": float(ideal),
        }
    return out


if __name__ == "__main__":
    a = [int(x) for x in sys.argv[1:4]]
    print(json.dumps(main(*a) if a else main(), indent=1))
