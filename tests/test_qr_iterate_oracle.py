"""Pins for the QR-iteration oracle pieces (``-m "not gpu"``; SURVEY §8(f) NEXT-2 without AED,
reading R21): the small Francis QR eigenvalue solver against exact characteristic polynomials
(LAPACK-free) and matrices of known spectrum; the iteration's eigenvalues, similarity and
orthogonality."""
from fractions import Fraction

import mpmath
import numpy as np
import pytest
import sympy as sp

import oracle
from hqr_inputs import random_case


def _charpoly_roots(A):
    n = A.shape[0]
    M = sp.Matrix(n, n, lambda i, j: sp.Rational(Fraction(float(A[i, j]))))
    coeffs = [sp.Rational(c) for c in M.charpoly().all_coeffs()]
    with mpmath.workdps(50):
        roots = mpmath.polyroots([mpmath.mpf(c.p) / c.q for c in coeffs], maxsteps=400, extraprec=400)
    return [complex(r) for r in roots]


def _match(a, b):
    a, b = list(a), list(b)
    worst = 0.0
    for z in a:
        k = int(np.argmin([abs(z - w) for w in b]))
        worst = max(worst, abs(z - b[k]) / max(1.0, abs(b[k])))
        b.pop(k)
    return worst


@pytest.mark.parametrize("seed,n", [(0, 3), (1, 5), (2, 7), (3, 8), (4, 8)])
def test_small_eig_vs_charpoly(seed, n):
    g = np.random.default_rng(700 + seed)
    A = np.triu(g.integers(-4, 5, (n, n)), -1).astype(float)
    A[np.arange(1, n), np.arange(n - 1)] = g.integers(1, 4, n - 1)
    wr, wi, info = oracle.small_eig(A)
    assert info == 0
    assert _match(wr + 1j * wi, _charpoly_roots(A)) <= 1e-12
    # conjugate pairs adjacent, positive imaginary part first
    for k in range(n):
        if wi[k] > 0:
            assert wr[k + 1] == wr[k] and wi[k + 1] == -wi[k]


@pytest.mark.parametrize("roots", [[1, 2, 3, 4, 5, 6], [-3, -1, 2, 2.5], [1 + 2j, 1 - 2j, -0.5, 3, 0.5j, -0.5j]])
def test_small_eig_companion_known_roots(roots):
    """Companion matrices (upper Hessenberg) of polynomials with the given roots."""
    c = np.real(np.poly(roots))
    n = len(roots)
    C = np.zeros((n, n))
    C[np.arange(1, n), np.arange(n - 1)] = 1.0
    C[:, -1] = -c[::-1][:n]
    wr, wi, info = oracle.small_eig(C)
    assert info == 0 and _match(wr + 1j * wi, roots) <= 1e-9


def test_small_eig_deflated_and_2x2_blocks():
    # block diagonal: exact zeros on the subdiagonal deflate at once; a rotation-like 2x2 block
    A = np.zeros((5, 5))
    A[0:2, 0:2] = [[1.0, -4.0], [1.0, 1.0]]      # eigenvalues 1 +- 2i
    A[2, 2] = 7.0
    A[3:5, 3:5] = [[2.0, 3.0], [1.0, 0.0]]        # eigenvalues 3, -1
    A[0, 4] = 5.0
    wr, wi, info = oracle.small_eig(A)
    assert info == 0 and _match(wr + 1j * wi, [1 + 2j, 1 - 2j, 7, 3, -1]) <= 1e-14


def _assert_real_schur(H, wr, wi):
    n = H.shape[0]
    sub = np.diag(H, -1)
    assert np.all(np.tril(H, -2) == 0.0)
    assert not np.any((sub[:-1] != 0.0) & (sub[1:] != 0.0))  # no 3x3 or larger blocks
    lam = []
    j = 0
    while j < n:
        if j + 1 < n and H[j + 1, j] != 0.0:
            lam += list(np.linalg.eigvals(H[j:j + 2, j:j + 2]))
            j += 2
        else:
            lam.append(H[j, j])
            j += 1
    assert _match(np.array(lam), wr + 1j * wi) <= 1e-9


@pytest.mark.parametrize("n,ns,nmin,seed", [(10, 2, 2, 5), (60, 8, 8, 6), (300, 16, 32, 7)])
def test_qr_iterate_eigenvalues_similarity(n, ns, nmin, seed):
    H0, Z0, _, _ = random_case(seed, n, 2, z0="orth")
    H, Z = H0.copy(order="F"), Z0.copy(order="F")
    wr, wi, rc, sweeps = oracle.qr_iterate(H, Z, 0, n - 1, ns, nmin=nmin)
    assert rc == 0 and sweeps >= 1
    lam = wr + 1j * wi
    if n <= 10:
        ref = _charpoly_roots(H0)
        assert _match(lam, ref) <= 1e-10
    assert abs(np.sum(wr) - np.trace(H0)) <= 1e-10 * n * np.linalg.norm(H0)
    assert np.linalg.norm(Z.T @ Z - np.eye(n)) <= 1e-13 * n
    assert np.linalg.norm(Z @ H @ Z.T - Z0 @ H0 @ Z0.T) <= 1e-13 * n * np.linalg.norm(H0)
    # H ends in real Schur form (R24): quasi-triangular, and the reported eigenvalues are those of
    # its 1x1 / 2x2 diagonal blocks
    _assert_real_schur(H, wr, wi)


# --------------------------------------------------------------------------------------------
# AED (reading R22)
# --------------------------------------------------------------------------------------------

@pytest.mark.parametrize("seed,n", [(10, 6), (11, 8), (12, 40)])
def test_schur_form(seed, n):
    A, _, _, _ = random_case(seed, n, 2)
    T, U, wr, wi, info = oracle.schur(A)
    assert info == 0
    assert np.linalg.norm(U.T @ U - np.eye(n)) <= 1e-13 * n
    assert np.linalg.norm(U.T @ A @ U - T) <= 1e-13 * n * np.linalg.norm(A)
    sub = np.diag(T, -1)
    assert np.all(np.tril(T, -2) == 0.0) and not np.any((sub[:-1] != 0) & (sub[1:] != 0))  # quasi-triangular
    if n <= 8:
        assert _match(wr + 1j * wi, _charpoly_roots(A)) <= 1e-12


def test_aed_deflates_below_a_tiny_spike():
    """A window whose coupling entry s is tiny: every spike entry s U(0, j) is below u ||H||_F, so
    the whole window deflates, its eigenvalues are those of the window, H stays similar."""
    from hqr_inputs import make_hess
    p = make_hess(60, 2)
    H0 = p.H.copy(order="F")
    k0, nw = 40, 20
    H0[k0, k0 - 1] = 1e-30
    W = H0[k0:, k0:].copy()
    H, Z = H0.copy(order="F"), np.asfortranarray(np.eye(60))
    thr = 2.0 ** -53 * np.linalg.norm(H0)
    nd, wr, wi, cand = oracle.aed(H, Z, 0, k0, nw, thr)
    assert nd == nw and len(cand) == 0
    assert _match(wr[k0:] + 1j * wi[k0:], np.linalg.eigvals(W)) <= 1e-10
    assert np.linalg.norm(Z @ H @ Z.T - H0) <= 1e-13 * 60 * np.linalg.norm(H0)
    assert np.all(H[k0:, k0 - 1] == 0.0) and np.all(np.tril(H, -2)[:, :k0] == 0.0)


@pytest.mark.parametrize("n,k0,nw,seed", [(80, 40, 40, 13), (120, 60, 60, 14)])
def test_aed_structure_and_similarity(n, k0, nw, seed):
    """After AED H is again upper Hessenberg, similar to H0 through Z, and the rows below
    n - nd are decoupled with the deflated eigenvalues their eigenvalues."""
    from hqr_inputs import make_hess
    p = make_hess(n, 2, z0="orth")
    H, Z = p.H.copy(order="F"), p.Z.copy(order="F")
    # a converged-looking tail: shrink the subdiagonal entries inside the window's bottom part
    for r in range(n - 6, n):
        H[r, r - 1] *= 1e-9
    H0, Z0 = H.copy(order="F"), Z.copy(order="F")
    thr = 2.0 ** -53 * np.linalg.norm(H0)
    nd, wr, wi, cand = oracle.aed(H, Z, 0, k0, nw, thr)
    assert np.linalg.norm(Z @ H @ Z.T - Z0 @ H0 @ Z0.T) <= 1e-13 * n * np.linalg.norm(H0)
    assert np.linalg.norm(Z.T @ Z - np.eye(n)) <= 1e-13 * n
    assert np.all(np.tril(H, -2) == 0.0)
    if nd > 0:
        assert H[n - nd, n - nd - 1] == 0.0
        tail = np.linalg.eigvals(H[n - nd:, n - nd:])
        assert _match(wr[n - nd:] + 1j * wi[n - nd:], tail) <= 1e-8


@pytest.mark.parametrize("n,ns,nw,nmin,seed", [(10, 2, 6, 2, 15), (300, 16, 48, 32, 16)])
def test_qr_iterate_aed(n, ns, nw, nmin, seed):
    from hqr_inputs import make_hess
    p = make_hess(n, 2, z0="orth")
    H, Z = p.H.copy(order="F"), p.Z.copy(order="F")
    wr, wi, rc, sweeps, naed, ndefl = oracle.qr_iterate_aed(H, Z, 0, n - 1, ns, nw=nw, nmin=nmin)
    assert rc == 0
    if n <= 10:
        assert _match(wr + 1j * wi, _charpoly_roots(p.H)) <= 1e-10
    hn = np.linalg.norm(p.H)
    assert np.linalg.norm(Z @ H @ Z.T - p.Z @ p.H @ p.Z.T) <= 1e-13 * n * hn
    assert abs(np.sum(wr) - np.trace(p.H)) <= 1e-10 * n * hn
    _assert_real_schur(H, wr, wi)
    if n >= 100:  # AED pays: fewer sweeps than the iteration without it, most eigenvalues by AED
        H2 = p.H.copy(order="F")
        _, _, _, sweeps_plain = oracle.qr_iterate(H2, None, 0, n - 1, ns, nmin=nmin)
        assert sweeps < sweeps_plain and ndefl > n // 2


# --------------------------------------------------------------------------------------------
# Eigenvalue reordering inside AED (reading R23)
# --------------------------------------------------------------------------------------------

def _quasi(rng, nw, blocks):
    """Quasi-triangular nw x nw T with the given diagonal block sizes (2x2 blocks complex)."""
    T = np.triu(rng.standard_normal((nw, nw)))
    j = 0
    for b in blocks:
        if b == 2:
            a = rng.standard_normal()
            T[j, j], T[j + 1, j + 1] = a, a
            T[j, j + 1] = abs(rng.standard_normal()) + 0.5
            T[j + 1, j] = -(abs(rng.standard_normal()) + 0.5)
        j += b
    return T


@pytest.mark.parametrize("p,q", [(1, 1), (2, 1), (1, 2), (2, 2)])
def test_swap_blocks(p, q):
    """The swap moves B's eigenvalues into the leading q x q block and A's into the next p x p block
    (eigenvalues from np.linalg.eigvals of the blocks), by an orthogonal similarity (U^T T0 U = T),
    leaving exact zeros below them and touching nothing outside rows / columns i..i+p+q-1 beyond U."""
    rng = np.random.default_rng(100 + 10 * p + q)
    i = 2
    layout = [1, 1, p, q, 1, 2]
    nw = sum(layout)
    T0 = np.asfortranarray(_quasi(rng, nw, layout))
    T, U = T0.copy(order="F"), np.asfortranarray(np.eye(nw))
    assert oracle.swap(T, U, i, p, q) == 0
    k = p + q
    assert np.linalg.norm(U.T @ U - np.eye(nw)) <= 1e-14 * nw
    assert np.linalg.norm(U @ T @ U.T - T0) <= 1e-14 * nw * np.linalg.norm(T0)
    ev = lambda M: np.sort_complex(np.linalg.eigvals(M))  # noqa: E731
    assert np.abs(ev(T[i:i + q, i:i + q]) - ev(T0[i + p:i + k, i + p:i + k])).max() <= 1e-13
    assert np.abs(ev(T[i + q:i + k, i + q:i + k]) - ev(T0[i:i + p, i:i + p])).max() <= 1e-13
    assert np.all(T[i + q:i + k, i:i + q] == 0.0)
    assert np.all(np.tril(T, -2) == 0.0)
    # outside the swapped rows / columns T is unchanged; U differs from I only in those columns
    rest = [r for r in range(nw) if not i <= r < i + k]
    assert np.array_equal(T[np.ix_(rest, rest)], T0[np.ix_(rest, rest)])
    assert np.array_equal(U[:, rest], np.eye(nw)[:, rest])


def test_swap_two_1x1_closed_form():
    """Two 1x1 blocks [[a, c], [0, b]]: the swap gives [[b, +-c], [0, a]] (a rotation keeps the
    Frobenius norm and the trace / determinant, so the off-diagonal entry keeps its modulus)."""
    for a, b, c in [(1.0, 2.0, 3.0), (-0.5, 4.0, 1e-3), (2.0, -2.0, 7.0)]:
        T = np.asfortranarray([[a, c], [0.0, b]])
        U = np.asfortranarray(np.eye(2))
        assert oracle.swap(T, U, 0, 1, 1) == 0
        assert abs(T[0, 0] - b) <= 1e-15 * 8 and abs(T[1, 1] - a) <= 1e-15 * 8 and T[1, 0] == 0.0
        assert abs(abs(T[0, 1]) - abs(c)) <= 1e-14 * 8
        # the first column of U is the eigenvector of b: (c, b - a) normalised
        x = np.array([c, b - a]) / np.hypot(c, b - a)
        assert abs(abs(U[:, 0] @ x) - 1.0) <= 1e-14


def test_swap_rejected_leaves_state_unchanged():
    """Badly scaled blocks (entries 1e-8 .. 1e8): a rejected swap returns 1 and leaves
    T and U bit-identical; an accepted one is an orthogonal similarity to working accuracy."""
    rng = np.random.default_rng(2)
    rejected = 0
    for _ in range(400):
        p, q = int(rng.integers(1, 3)), int(rng.integers(1, 3))
        k = p + q
        T0 = np.triu(rng.standard_normal((k, k)) * 10.0 ** rng.uniform(-8, 8, (k, k)))
        T0 = np.asfortranarray(T0)
        T, U = T0.copy(order="F"), np.asfortranarray(np.eye(k))
        rc = oracle.swap(T, U, 0, p, q)
        if rc:
            rejected += 1
            assert np.array_equal(T, T0) and np.array_equal(U, np.eye(k))
        else:
            assert np.linalg.norm(U @ T @ U.T - T0) <= 1e-13 * np.abs(T0).max()
    assert rejected >= 1


def test_aed_reordering_matches_the_predicted_deflations():
    """Windows whose bottom block fails the deflation check while blocks above it pass (no
    reordering would deflate nothing): the oracle's AED deflates exactly the eigenvalues predicted
    from the invariant subspaces of W (tests/aed_predict.py, LAPACK's ordered Schur form), H stays
    similar and Hessenberg."""
    from aed_predict import reorder_cases
    cases = list(reorder_cases(oracle.schur))
    assert len(cases) == 3
    above = 6
    rng = np.random.default_rng(3)
    for W, s, thr, defl, dec in cases:
        nw = W.shape[0]
        n = above + nw
        H0 = np.asfortranarray(np.triu(rng.standard_normal((n, n)), -1))
        H0[above:, above:] = W
        H0[above, above - 1] = s
        H, Z = H0.copy(order="F"), np.asfortranarray(np.eye(n))
        nd, wr, wi, cand = oracle.aed(H, Z, 0, above, nw, thr)
        assert nd == len(defl) and nd > 0 and not dec[0]
        got = wr[n - nd:] + 1j * wi[n - nd:]
        assert _match(got, defl) <= 1e-10 and _match(defl, got) <= 1e-10
        assert _match(cand, [l for l in np.linalg.eigvals(W) if min(abs(l - np.array(defl))) > 1e-8]) <= 1e-10
        # similar up to the zeroed spike entries (each <= thr: the deflation's backward error)
        assert np.linalg.norm(Z @ H @ Z.T - H0) <= np.sqrt(nd) * thr + 1e-13 * n * np.linalg.norm(H0)
        assert np.all(np.tril(H, -2) == 0.0) and H[n - nd, n - nd - 1] == 0.0
