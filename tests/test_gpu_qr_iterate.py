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
    """A block of at most nmin rows goes straight to the small-block path: real Schur form through the
    AED window machinery up to 112 rows (R24), the one-CTA Francis QR eigenvalue solver above."""
    H0, _, _, _ = random_case(seed, n, 2)
    Hd = hq.to_device(H0)
    wr, wi, rc, sweeps = hq.qr_iterate(Hd, None, 0, n - 1, nshifts=2, nmin=128)
    assert rc == 0 and sweeps == 0
    owr, owi, info = oracle.small_eig(H0)
    assert info == 0 and _match(wr + 1j * wi, owr + 1j * owi) <= 1e-10
    if n <= 112:
        _assert_real_schur(hq.from_device(Hd), wr, wi)
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
    _assert_real_schur(H, wr, wi)  # R24: the small blocks end in real Schur form
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
    _assert_real_schur(H, wr, wi)
    assert st["window_eff"] > n // 2                      # eigenvalues deflated by AED
    Hd2 = hq.to_device(p.H)
    _, _, _, sweeps_plain = hq.qr_iterate(Hd2, None, 0, n - 1, nshifts=ns, window=win, nmin=nmin)
    assert sweeps < sweeps_plain


def _assert_real_schur(H, wr, wi):
    """Quasi-triangular H (no two consecutive nonzero subdiagonals) whose 1x1 / 2x2 diagonal blocks
    carry the reported eigenvalues (R24)."""
    n = H.shape[0]
    sub = np.diag(H, -1)
    assert np.all(np.tril(H, -2) == 0.0)
    assert not np.any((sub[:-1] != 0.0) & (sub[1:] != 0.0))
    lam, j = [], 0
    while j < n:
        if j + 1 < n and H[j + 1, j] != 0.0:
            lam += list(np.linalg.eigvals(H[j:j + 2, j:j + 2]))
            j += 2
        else:
            lam.append(H[j, j])
            j += 1
    assert _match(np.array(lam), wr + 1j * wi) <= 1e-9


def _aed_problem(W, s, above, rng):
    nw = W.shape[0]
    n = above + nw
    H0 = np.asfortranarray(np.triu(rng.standard_normal((n, n)), -1))
    H0[above:, above:] = W
    H0[above, above - 1] = s
    return H0


def test_aed_step_reordering_vs_oracle():
    """One AED step through the C ABI (hqr_aed, reading R23) on windows that need the reordering
    (the bottom block fails, blocks above it pass; decisions determined with a margin,
    tests/aed_predict.py): the GPU deflates the predicted eigenvalues, like the oracle; its
    candidates are the other eigenvalues of W; H stays Hessenberg and similar to H0 through Z up to
    the zeroed spike entries (the window's 2x2 blocks, hence H itself, are unique only up to an
    orthogonal basis of each block, so H is not compared entry by entry)."""
    from aed_predict import reorder_cases
    above = 6
    rng = np.random.default_rng(3)
    for W, s, thr, defl, dec in reorder_cases(oracle.schur):
        H0 = _aed_problem(W, s, above, rng)
        n, nw = H0.shape[0], W.shape[0]
        Zo = np.asfortranarray(np.eye(n))
        Ho = H0.copy(order="F")
        ndo, owr, owi, _ = oracle.aed(Ho, Zo, 0, above, nw, thr)
        Hd, Zd = hq.to_device(H0), hq.to_device(np.eye(n))
        nd, ev = hq.aed(Hd, Zd, 0, above, nw, thr)
        H, Z = hq.from_device(Hd), hq.from_device(Zd)
        assert nd == ndo == len(defl)
        assert _match(ev[nw - nd:], defl) <= 1e-10
        assert _match(ev[:nw - nd], [l for l in np.linalg.eigvals(W) if min(abs(l - np.array(defl))) > 1e-8]) <= 1e-10
        hn = np.linalg.norm(H0)
        assert np.linalg.norm(Z.T @ Z - np.eye(n)) <= 1e-13 * n
        assert np.linalg.norm(Z @ H @ Z.T - H0) <= np.sqrt(nd) * thr + 1e-13 * n * hn
        assert np.all(np.tril(H, -2) == 0.0) and H[n - nd, n - nd - 1] == 0.0
        assert _match(np.linalg.eigvals(H[n - nd:, n - nd:]), defl) <= 1e-9


@pytest.mark.parametrize("n,nw,seed", [(300, 96, 0), (200, 64, 1)])
def test_aed_step_converging_tail_vs_oracle(n, nw, seed):
    """A hess_n matrix after a QR iteration ran to the point where its trailing part is close to
    converged (subdiagonal entries of the window shrunk): the GPU AED step deflates as many
    eigenvalues as the oracle's, the same ones; H stays Hessenberg and similar to H0 through Z;
    thr = 2^-53 ||H||_F (the paper's norm-stable condition)."""
    from hqr_inputs import make_hess
    p = make_hess(n, 2, z0="orth")
    H0 = p.H.copy(order="F")
    k0 = n - nw
    g = np.random.default_rng(seed)
    for r in range(k0 + 1, n):  # graded subdiagonal: blocks near the bottom converge, some fail
        H0[r, r - 1] *= 10.0 ** (-12.0 * g.uniform(0.0, 1.0))
    thr = 2.0 ** -53 * np.linalg.norm(H0)
    Ho, Zo = H0.copy(order="F"), p.Z.copy(order="F")
    ndo, owr, owi, ocand = oracle.aed(Ho, Zo, 0, k0, nw, thr)
    Hd, Zd = hq.to_device(H0), hq.to_device(p.Z)
    nd, ev = hq.aed(Hd, Zd, 0, k0, nw, thr)
    H, Z = hq.from_device(Hd), hq.from_device(Zd)
    assert nd == ndo
    if nd:
        assert _match(ev[nw - nd:], owr[n - nd:] + 1j * owi[n - nd:]) <= 1e-9
        assert H[n - nd, n - nd - 1] == 0.0
    hn = np.linalg.norm(H0)
    assert np.linalg.norm(Z.T @ Z - np.eye(n)) <= 1e-13 * n
    assert np.linalg.norm(Z @ H @ Z.T - p.Z @ H0 @ p.Z.T) <= 1e-13 * n * hn
    assert np.all(np.tril(H, -2) == 0.0)


def test_aed_argument_errors():
    Hd = hq.to_device(np.eye(10))
    with pytest.raises(hq.HQRError):
        hq.aed(Hd, None, 0, 5, 1, 1e-16)      # nw < 2
    with pytest.raises(hq.HQRError):
        hq.aed(Hd, None, 0, 5, 6, 1e-16)      # window outside H
    with pytest.raises(hq.HQRError):
        hq.aed(Hd, None, 6, 5, 4, 1e-16)      # k0 < ilo
