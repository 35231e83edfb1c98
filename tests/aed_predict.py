"""Independent prediction of the AED deflation decisions with reordering (reading R23), for the
pins in test_qr_iterate_oracle.py and the GPU parity test.  No oracle code: LAPACK's ordered real
Schur form (scipy.linalg.schur with a selection) gives the invariant subspaces.

When a block b sits at the bottom of the undeflated part [0, m) of the reordered Schur form, the
columns U(:, m-|b| : m) are an orthonormal basis of  span(V_undef) minus span(V_undef \\ b)  (the
invariant subspaces of the window W for the undeflated eigenvalues with and without b), whatever
swaps brought it there.  So its spike s U(0, rows of b) has the basis-independent norm
|s| ||P_b^T e1||, P_b an orthonormal basis of that difference; for a 1x1 block this is the spike
entry itself, for a 2x2 block both entries are <= thr when the norm is, and one exceeds thr when
the norm exceeds sqrt(2) thr.  Blocks are evaluated bottom-up in the initial Schur order (a failed
block moves to the top, the next one up comes down to the bottom)."""
from __future__ import annotations

import numpy as np
import scipy.linalg as sl


def blocks_bottom_up(T):
    """The diagonal blocks of the quasi-triangular T, bottom first, as lists of eigenvalues."""
    nw = T.shape[0]
    out, j = [], nw
    while j > 0:
        if j >= 2 and T[j - 1, j - 2] != 0.0:
            out.append(list(np.linalg.eigvals(T[j - 2:j, j - 2:j])))
            j -= 2
        else:
            out.append([complex(T[j - 1, j - 1])])
            j -= 1
    return out


def _basis(W, lams):
    if not lams:
        return np.zeros((W.shape[0], 0))
    sel = lambda re, im: any(abs(complex(re, im) - l) <= 1e-7 * max(1.0, abs(l)) for l in lams)  # noqa: E731
    _, Zs, sdim = sl.schur(W, output="real", sort=sel)
    assert sdim == len(lams), (sdim, len(lams))
    return Zs[:, :sdim]


def predict(W, s, thr, blocks):
    """(deflated eigenvalues, smallest relative margin of any decision, decisions) or None when a
    2x2 decision is undetermined by the norm."""
    undef = [l for b in blocks for l in b]
    defl, margins, decisions = [], [], []
    for b in blocks:
        rest = list(undef)
        for l in b:
            rest.remove(l)
        V1, V0 = _basis(W, undef), _basis(W, rest)
        P = V1 - V0 @ (V0.T @ V1)
        Q = np.linalg.svd(P)[0][:, :len(b)]
        nrm = abs(s) * np.linalg.norm(Q[0, :])
        if len(b) == 1:
            ok = nrm <= thr
            margins.append(abs(nrm / thr - 1.0))
        elif nrm <= thr:
            ok = True
            margins.append(1.0 - nrm / thr)
        elif nrm > np.sqrt(2.0) * thr:
            ok = False
            margins.append(nrm / (np.sqrt(2.0) * thr) - 1.0)
        else:
            return None
        decisions.append(bool(ok))
        if ok:
            undef = rest
            defl += b
    return defl, min(margins), decisions


def reorder_cases(schur, count=3, nw=14, seed=7, min_margin=0.02):
    """Seeded windows (random Hessenberg W, coupling s = 1) and thresholds whose decisions are all
    determined with a margin and need the reordering: the bottom block fails, a later one deflates.
    schur(W) -> (T, U, ...) gives the initial block order.  Yields (W, s, thr, predicted deflated)."""
    rng = np.random.default_rng(seed)
    found = 0
    for _ in range(200):
        W = np.triu(rng.standard_normal((nw, nw)), -1)
        T = schur(W)[0]
        blocks = blocks_bottom_up(T)
        for thr in np.geomspace(1e-4, 0.5, 25):
            r = predict(W, 1.0, thr, blocks)
            if r is None:
                continue
            defl, marg, dec = r
            if marg < min_margin or dec[0] or not any(dec):
                continue
            yield W, 1.0, float(thr), defl, dec
            found += 1
            break
        if found == count:
            return
