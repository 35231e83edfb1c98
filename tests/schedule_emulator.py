"""numpy emulation of the GPU wavefront schedule (test helper, CPU only).

Executes the plan returned by the library's own planner (hqr_plan_query) with the same window
rule and two-phase step as chase.cu / update.cu, in plain numpy.  Comparing it with the oracle
checks the planner and the window algorithm on the CPU, independently of the CUDA kernels.
It imports neither oracle/ nor any kernel code: only the plan table.
"""
import numpy as np

import paper_2007_03576_b200 as hq


def _house(m, x):
    x0 = x[0]
    tail2 = float(np.dot(x[1:m], x[1:m]))
    if tail2 == 0.0:
        return np.zeros(m - 1), 0.0, x0
    nrm = np.sqrt(x0 * x0 + tail2)
    b = -nrm if x0 >= 0.0 else nrm
    return x[1:m] / (x0 - b), (b - x0) / b, b


def emulate(H, Z, ilo, ihi, sr, si, window, on_window=None, blocks=None, sweeps=None):
    """blocks = [(ilo, ihi, nshifts), ...] for a multi-block sweep (ilo/ihi ignored then);
    sweeps = [nshifts_0, nshifts_1, ...] for overlapped sweeps of [ilo, ihi] (hqr_sweeps)."""
    n = H.shape[0]
    if sweeps is not None:
        info, wins = hq.plan_query_sweeps(n, ilo, ihi, sweeps, window)
    else:
        if blocks is None:
            blocks = [(ilo, ihi, len(sr))]
        info, wins = hq.plan_query_multi(n, blocks, window)
    nb = len(sr) // 2
    sig = [sr[2 * j] + sr[2 * j + 1] for j in range(nb)]
    pis = [sr[2 * j] * sr[2 * j + 1] - si[2 * j] * si[2 * j + 1] for j in range(nb)]
    for step in range(info["nsteps"]):
        sw = wins[wins[:, 0] == step]
        Qs = []
        for w in sw:
            _, chain, w0, w1, t0, t1, b0, nbc, slot, last, ilo, ihi = (int(v) for v in w)
            nbc = int(w[7])
            Hw = H[w0:w1 + 1, w0:w1 + 1].copy()
            Q = chase_window(Hw, w, sig, pis)
            H[w0:w1 + 1, w0:w1 + 1] = Hw
            Qs.append((w0, w1, Q))
            if on_window is not None:
                on_window(nbc, Q)
        for w0, w1, Q in Qs:  # left updates
            H[w0:w1 + 1, w1 + 1:] = Q.T @ H[w0:w1 + 1, w1 + 1:]
        for w0, w1, Q in Qs:  # right + Z updates
            H[:w0, w0:w1 + 1] = H[:w0, w0:w1 + 1] @ Q
            if Z is not None:
                Z[:, w0:w1 + 1] = Z[:, w0:w1 + 1] @ Q
    return info


def chase_window(Hw, w, sig, pis):
    """In-window chase of plan window row w (as chase.cu): updates the window block Hw in place and
    returns its accumulated factor Q_W."""
    _, chain, w0, w1, t0, t1, b0, nbc, slot, last, ilo, ihi = (int(v) for v in w)
    kw = w1 - w0 + 1
    Q = np.eye(kw)
    for t in range(t0, t1 + 1):
        refl = []
        # rows of Q_W below the deepest reflector so far (bulge 0 at p0 = ilo-1+t, touching rows
        # <= p0+3) are still identity rows
        p0 = ilo - 1 + t
        for jj in range(nbc):  # phase 1
            p = ilo - 1 + t - 3 * jj
            if p < ilo - 1 or p > ihi - 2:
                continue
            pl = p - w0
            m = 3 if p <= ihi - 3 else 2
            if p == ilo - 1:
                j = b0 + jj
                h00, h10, h01, h11, h21 = Hw[0, 0], Hw[1, 0], Hw[0, 1], Hw[1, 1], Hw[2, 1]
                x = np.array([h00 * (h00 - sig[j]) + h01 * h10 + pis[j],
                              h10 * (h00 + h11 - sig[j]), h10 * h21])
            else:
                x = Hw[pl + 1:pl + 1 + m, pl].copy()
            vt, tau, beta = _house(m, x)
            v = np.concatenate([[1.0], vt])
            if p >= ilo:
                Hw[pl + 1, pl] = beta
                Hw[pl + 2:pl + 1 + m, pl] = 0.0
            c0 = 0 if p == ilo - 1 else pl + 1
            blk = Hw[pl + 1:pl + 1 + m, c0:]
            blk -= tau * np.outer(v, v @ blk)
            refl.append((pl, m, v, tau))
        for pl, m, v, tau in refl:  # phase 2
            rH = min(pl + m + 1, ihi - w0)
            blk = Hw[:rH + 1, pl + 1:pl + 1 + m]
            blk -= tau * np.outer(blk @ v, v)
            rQ = min(p0 - w0 + 3, kw - 1)
            blk = Q[:rQ + 1, pl + 1:pl + 1 + m]
            blk -= tau * np.outer(blk @ v, v)
    return Q


def shift_coefs(sr, si):
    nb = len(sr) // 2
    sig = [sr[2 * j] + sr[2 * j + 1] for j in range(nb)]
    pis = [sr[2 * j] * sr[2 * j + 1] - si[2 * j] * si[2 * j + 1] for j in range(nb)]
    return sig, pis
