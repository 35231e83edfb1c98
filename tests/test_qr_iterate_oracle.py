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
    # H is reduced to unreduced blocks of at most nmin rows
    zeros = [0] + [k for k in range(1, n) if H[k, k - 1] == 0.0] + [n]
    assert max(b - a for a, b in zip(zeros, zeros[1:])) <= nmin
