"""Oracle self noise floor: two valid reflector orders of the same sweep (sequential Francis steps vs
pipelined bulges), on BASELINE configs -- the rounding-level difference any correct reordering
(including the GPU's wavefront) can show.  Writes a JSON line.  Calls only oracle/ and hqr_inputs."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import oracle  # noqa: E402
from hqr_inputs import make  # noqa: E402


def main(cfg, shift_kind=None):
    if cfg == 4:  # "4:b<k>": diagonal block k of configs[4] alone, Z = I (the blocks are decoupled)
        from types import SimpleNamespace
        from hqr_inputs import config4_block
        Hb, re_, im_, _ = config4_block(int(shift_kind[1:]))
        nb = Hb.shape[0]
        p = SimpleNamespace(H=Hb, Z=np.asfortranarray(np.eye(nb)), ilo=0, ihi=nb - 1, shifts_re=re_, shifts_im=im_)
    else:
        p = make(cfg, shift_kind=shift_kind)
    n = p.H.shape[0]
    t0 = time.time()
    Hs, Zs = p.H.copy(order="F"), p.Z.copy(order="F")
    oracle.sweep(Hs, Zs, p.ilo, p.ihi, p.shifts_re, p.shifts_im, order="sequential")
    t1 = time.time()
    Hp, Zp = p.H.copy(order="F"), p.Z.copy(order="F")
    oracle.sweep(Hp, Zp, p.ilo, p.ihi, p.shifts_re, p.shifts_im, order="pipelined")
    t2 = time.time()
    dH = Hs - Hp
    i, j = np.unravel_index(np.argmax(np.abs(dH)), dH.shape)
    sub = np.abs(np.diag(Hs, -1))
    out = {"cfg": cfg, "shifts": shift_kind or "config", "n": n, "nshifts": len(p.shifts_re),
           "dH_rel_fro": float(np.linalg.norm(dH) / np.linalg.norm(p.H)),
           "dZ_fro_over_sqrt_n": float(np.linalg.norm(Zs - Zp) / np.sqrt(n)),
           "dH_max": float(np.abs(dH).max()), "dH_argmax": [int(i), int(j)],
           "min_abs_subdiag_after": float(sub.min()), "argmin_subdiag": int(np.argmin(sub)),
           "oracle_seconds": [t1 - t0, t2 - t1]}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    # arguments: "3" (configs[3] as specified), "3:ring68" (configs[3] with another shift set) or
    # "4:b2" (diagonal block 2 of configs[4], swept alone with Z = I)
    for c in sys.argv[1:]:
        cfg, _, kind = c.partition(":")
        main(int(cfg), kind or None)
