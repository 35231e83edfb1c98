"""GPU: the QR iteration around the sweep (hqr_qr_iterate; SURVEY §8(f) NEXT-2 without AED,
reading R21) against the oracle's iteration (oracle_qr_iterate) on the same seeded inputs.

The eigenvalues are unique (compared as sets); the Schur-like H and Z are not (which eigenvalues
deflate in which sweep depends on rounding), so those are checked through the similarity
Z H Z^T = Z0 H0 Z0^T, orthogonality and the block structure."""
import numpy as np
import pytest

import oracle
import paper_2007_03576_b200 as hq
from hqr_inputs import random_case

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def lib_setup():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    hq.setup(0)
    yield
    hq.teardown()


def _match(a, b):
    a, b = list(a), list(b)
    worst = 0.0
    for z in a:
        k = int(np.argmin([abs(z - w) for w in b]))
        worst = max(worst, abs(z - b[k]) / max(1.0, abs(b[k])))
        b.pop(k)
    return worst


@pytest.mark.parametrize("n,seed", [(3, 0), (8, 1), (40, 2), (127, 3), (128, 4)])
def test_small_block_solver(n, seed):
    """A block of at most nmin rows goes straight to the one-CTA Francis QR solver."""
    H0, _, _, _ = random_case(seed, n, 2)
    Hd = hq.to_device(H0)
    wr, wi, rc, sweeps = hq.qr_iterate(Hd, None, 0, n - 1, nshifts=2, nmin=128)
    assert rc == 0 and sweeps == 0
    owr, owi, info = oracle.small_eig(H0)
    assert info == 0 and _match(wr + 1j * wi, owr + 1j * owi) <= 1e-10
    for k in range(n):
        if wi[k] > 0:
            assert wr[k + 1] == wr[k] and wi[k + 1] == -wi[k]


@pytest.mark.parametrize("n,ns,nmin,win,seed", [(300, 16, 32, 48, 5), (800, 32, 64, 96, 6), (2000, 64, 96, 96, 7)])
def test_qr_iteration_vs_oracle(n, ns, nmin, win, seed):
    H0, Z0, _, _ = random_case(seed, n, 2, z0="orth")
    Hd, Zd = hq.to_device(H0), hq.to_device(Z0)
    wr, wi, rc, sweeps = hq.qr_iterate(Hd, Zd, 0, n - 1, nshifts=ns, window=win, nmin=nmin)
    assert rc == 0 and sweeps >= 1
    H, Z = hq.from_device(Hd), hq.from_device(Zd)
    Ho, Zo = H0.copy(order="F"), Z0.copy(order="F")
    owr, owi, orc, osw = oracle.qr_iterate(Ho, Zo, 0, n - 1, ns, nmin=nmin)
    assert orc == 0
    assert _match(wr + 1j * wi, owr + 1j * owi) <= 1e-8
    hn = np.linalg.norm(H0)
    assert np.linalg.norm(Z.T @ Z - np.eye(n)) <= 1e-13 * n
    assert np.linalg.norm(Z @ H @ Z.T - Z0 @ H0 @ Z0.T) <= 1e-13 * n * hn
    assert np.all(np.tril(H, -2) == 0.0)
    zeros = [0] + [k for k in range(1, n) if H[k, k - 1] == 0.0] + [n]
    assert max(b - a for a, b in zip(zeros, zeros[1:])) <= nmin
    # the sweep counts are of the same order (the trajectories differ by rounding)
    assert 0.5 * osw <= sweeps <= 2.0 * osw


@pytest.mark.parametrize("n,ns,aed,nmin,win,seed", [(300, 16, 48, 32, 48, 0), (800, 32, 96, 64, 96, 1),
                                                    (2000, 64, 96, 96, 96, 2)])
def test_qr_iteration_with_aed_vs_oracle(n, ns, aed, nmin, win, seed):
    """NEXT-2 with AED (reading R22) on hess_n matrices: the eigenvalue sets of the GPU
    iteration and the oracle's agree; Z H Z^T = Z0 H0 Z0^T; most eigenvalues deflate in AED and the
    iteration needs fewer sweeps than without AED."""
    from hqr_inputs import make_hess
    p = make_hess(n, 2, z0="orth")
    Hd, Zd = hq.to_device(p.H), hq.to_device(p.Z)
    wr, wi, rc, sweeps = hq.qr_iterate(Hd, Zd, 0, n - 1, nshifts=ns, window=win, nmin=nmin, aed_window=aed)
    st = hq.stats()
    assert rc == 0
    H, Z = hq.from_device(Hd), hq.from_device(Zd)
    Ho, Zo = p.H.copy(order="F"), p.Z.copy(order="F")
    owr, owi, orc, osw, onaed, ondefl = oracle.qr_iterate_aed(Ho, Zo, 0, n - 1, ns, nw=aed, nmin=nmin)
    assert orc == 0
    assert _match(wr + 1j * wi, owr + 1j * owi) <= 1e-8
    hn = np.linalg.norm(p.H)
    assert np.linalg.norm(Z.T @ Z - np.eye(n)) <= 1e-13 * n
    assert np.linalg.norm(Z @ H @ Z.T - p.Z @ p.H @ p.Z.T) <= 1e-13 * n * hn
    assert np.all(np.tril(H, -2) == 0.0)
    assert st["window_eff"] > n // 2                      # eigenvalues deflated by AED
    Hd2 = hq.to_device(p.H)
    _, _, _, sweeps_plain = hq.qr_iterate(Hd2, None, 0, n - 1, nshifts=ns, window=win, nmin=nmin)
    assert sweeps < sweeps_plain
