"""Which sweeps use the critical-SM queue (hqr_stats.crit_sms), and the sweep time with it forced off
(HQR_CRIT_SMS=0 in a tuning build, HQR_LIB).  Not product code."""
import numpy as np

import paper_2007_03576_b200 as hq
from hqr_inputs import random_case

hq.setup(0)
for n, ns in [(300, 16), (1500, 64), (2000, 200), (3000, 400), (4000, 600), (3000, 1000)]:
    H0, Z0, re, im = random_case(1, n, ns)
    Hd, Zd = hq.to_device(H0), hq.to_device(Z0)
    t = []
    for _ in range(4):
        Hd.t().copy_(hq.to_device(H0).t())
        hq.sweep(Hd, Zd, 0, n - 1, re, im, window=96)
        t.append(hq.stats()["ms_total"])
    st = hq.stats()
    print(n, ns, "crit_sms", st["crit_sms"], "ms", round(min(t[1:]), 2), flush=True)
hq.teardown()
