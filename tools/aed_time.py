"""Per-AED phase cycles (Schur form vs deflation check with reordering) on the bench's qriter
workload: run with HQR_LIB pointing at a build with -DHQR_AED_TIMING (tools/build_variant.sh);
the kernel prints one 'AEDT' line per AED step.  Not product code."""
import sys

import numpy as np

import paper_2007_03576_b200 as hq
from hqr_inputs import make_hess

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
H0 = make_hess(n, 2).H
hq.setup(0)
Hd, Zd = hq.to_device(H0), hq.to_device(np.eye(n))
wr, wi, rc, sw = hq.qr_iterate(Hd, Zd, 0, n - 1, nshifts=64, window=96, nmin=96, aed_window=96)
st = hq.stats()
print(f"AEDSUM rc {rc} sweeps {sw} aed {st['launches_chase']} defl {st['window_eff']} ms {st['ms_total']:.1f}",
      flush=True)
hq.teardown()
