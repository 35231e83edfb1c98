"""Debug helper: configs[3]-shaped sweep with per-step critical-path timestamps (a -DHQR_TIMING build
via HQR_LIB, HQR_TIMING_DUMP=1).  usage: python tools/timing_probe.py [n] [nshifts]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_03576_b200 as hq  # noqa: E402
from hqr_inputs import random_case  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 512
H0, Z0, re_, im_ = random_case(3, n, ns, 0, n - 1, z0="eye", shift_kind="disk2")
hq.setup(0)
Hd, Zd = hq.to_device(H0), hq.to_device(Z0)
for r in range(2):
    hq.sweep(Hd, Zd, 0, n - 1, re_, im_, 96)
print(hq.stats()["ms_total"])
hq.teardown()
