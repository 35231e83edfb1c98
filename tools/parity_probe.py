"""Debug helper: GPU sweep vs the oracle for one random case; prints the relative errors.
usage: python tools/parity_probe.py n nshifts window ilo ihi [seed] [z0]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (test infrastructure: debugging only)
import paper_2007_03576_b200 as hq  # noqa: E402
from hqr_inputs import random_case  # noqa: E402

n, ns, win, ilo, ihi = (int(v) for v in sys.argv[1:6])
seed = int(sys.argv[6]) if len(sys.argv) > 6 else 9
z0 = sys.argv[7] if len(sys.argv) > 7 else "eye"
H0, Z0, re_, im_ = random_case(seed, n, ns, ilo, ihi, z0=z0, shift_kind="mixed" if seed % 2 else "disk2")
hq.setup(0)
Hd, Zd = hq.to_device(H0), hq.to_device(Z0)
hq.sweep(Hd, Zd, ilo, ihi, re_, im_, win)
Hg, Zg = hq.from_device(Hd), hq.from_device(Zd)
Ho, Zo = H0.copy(order="F"), Z0.copy(order="F")
oracle.sweep(Ho, Zo, ilo, ihi, re_, im_)
dh = np.linalg.norm(Hg - Ho) / np.linalg.norm(H0)
dz = np.linalg.norm(Zg - Zo) / np.sqrt(n)
bad = np.argwhere(np.abs(Hg - Ho) > 1e-8 * np.abs(H0).max())
print(f"n={n} ns={ns} win={win} [{ilo},{ihi}] dH={dh:.3e} dZ={dz:.3e} bad={len(bad)} first={bad[:5].tolist()}")
