"""Pins for the generalized (QZ) sweep oracle (``-m "not gpu"``, PAPER.md
P:208-213): closed forms of the right-hand side reflector, the bulge vector against
exact rational arithmetic, the reduction to the standard QR sweep when T = I, the equivalence
(Q^T H0 Z, Q^T T0 Z), structure, LAPACK-free preservation of the generalized eigenvalues, and
perfect-shift deflation."""
from fractions import Fraction

import mpmath
import numpy as np
import pytest
import sympy as sp

import oracle
from hqr_inputs import make_qz, random_case

U = 2.0 ** -53


@pytest.mark.parametrize("r", [[1.0, 2.0, 2.0], [3.0, 4.0], [0.0, 0.0, 5.0], [-1.0, 2.0, 0.0], [2.0, -3.0, 6.0]])
def test_rhs_house_zeros_row(r):
    u, tau, beta = oracle.rhs_house(r)
    m = len(r)
    assert u[m - 1] == 1.0
    P = np.eye(m) - tau * np.outer(u, u)
    y = np.array(r) @ P
    nr = np.linalg.norm(r)
    assert np.all(np.abs(y[:-1]) <= 8 * U * nr) and abs(y[-1] - beta) <= 8 * U * nr
    assert abs(abs(beta) - nr) <= 4 * U * nr
    assert np.linalg.norm(P @ P.T - np.eye(m)) <= 16 * U


def test_rhs_house_exact_122():
    # reversed (2, 2, 1): beta = -3, tau = 5/3, v = (1, 2/5, 1/5) -> u = (1/5, 2/5, 1)
    u, tau, beta = oracle.rhs_house([1.0, 2.0, 2.0])
    assert beta == -3.0 and abs(tau - 5.0 / 3.0) <= 2 * U and np.allclose(u, [0.2, 0.4, 1.0], atol=U, rtol=0)


def _qz_first_col_exact(Hq, Tq, s1, s2):
    """(M - s1 I)(M - s2 I) e1 with M = H T^-1, exact rationals (T upper triangular)."""
    n = len(Hq)

    def tinv(vec):  # back substitution
        y = [Fraction(0)] * n
        for i in range(n - 1, -1, -1):
            y[i] = (vec[i] - sum(Tq[i][k] * y[k] for k in range(i + 1, n))) / Tq[i][i]
        return y

    def mv(vec, s):
        y = tinv(vec)
        return [sum(Hq[i][k] * y[k] for k in range(n)) - s * vec[i] for i in range(n)]

    e = [Fraction(int(i == 0)) for i in range(n)]
    return mv(mv(e, s2), s1)


@pytest.mark.parametrize("seed", range(8))
def test_qz_first_column_exact(seed):
    g = np.random.default_rng(500 + seed)
    n = 6
    Hi = np.triu(g.integers(-4, 5, (n, n)), -1).astype(float)
    Hi[np.arange(1, n), np.arange(n - 1)] = g.integers(1, 4, n - 1)
    Ti = np.triu(g.integers(-3, 4, (n, n))).astype(float)
    Ti[np.arange(n), np.arange(n)] = [1.0, 2.0, 4.0, 1.0, 2.0, 1.0]   # powers of two: exact quotients
    s1, s2 = Fraction(int(g.integers(-3, 4)), 2), Fraction(int(g.integers(-3, 4)), 4)
    Hq = [[Fraction(int(Hi[i, j])) for j in range(n)] for i in range(n)]
    Tq = [[Fraction(int(Ti[i, j])) for j in range(n)] for i in range(n)]
    exact = _qz_first_col_exact(Hq, Tq, s1, s2)
    x = oracle.qz_first_column(np.asfortranarray(Hi), np.asfortranarray(Ti), 0, (float(s1), float(s2)))
    assert all(Fraction(x[i]) == exact[i] for i in range(3))
    assert all(v == 0 for v in exact[3:])


def _qz_case(n, ns, seed, q0="orth", ilo=0, ihi=None):
    p = make_qz(n, ns, q0=q0, seed=seed)
    ihi = n - 1 if ihi is None else ihi
    if ilo > 0:
        p.H[ilo, ilo - 1] = 0.0
    if ihi < n - 1:
        p.H[ihi + 1, ihi] = 0.0
    return p, ilo, ihi


@pytest.mark.parametrize("n,ns,seed", [(6, 2, 0), (40, 8, 1), (120, 20, 2), (300, 40, 3)])
def test_qz_with_identity_T_is_the_qr_sweep(n, ns, seed):
    """T = I: the left reflectors are the QR sweep's; the right ones restore T = diag(+-1), so
    H' T'^-1 equals the QR oracle's H' and T' is diagonal +-1 (to rounding)."""
    H0, Z0, re_, im_ = random_case(seed, n, ns, z0="eye", shift_kind="disk2")
    Hq, Tq = H0.copy(order="F"), np.asfortranarray(np.eye(n))
    oracle.qz_sweep(Hq, Tq, None, None, 0, n - 1, re_, im_)
    Hr = H0.copy(order="F")
    oracle.sweep(Hr, None, 0, n - 1, re_, im_)
    d = np.diag(Tq)
    assert np.all(np.abs(np.abs(d) - 1.0) <= 1e-13 * n)
    assert np.linalg.norm(Tq - np.diag(d)) <= 1e-13 * n
    assert np.linalg.norm(Hq / d[None, :] - Hr) <= 1e-12 * n * np.linalg.norm(H0)


@pytest.mark.parametrize("n,ns,seed,ilo,ihi", [(50, 8, 4, 0, None), (150, 20, 5, 10, 140), (200, 40, 6, 0, None)])
def test_qz_equivalence_structure(n, ns, seed, ilo, ihi):
    p, ilo, ihi = _qz_case(n, ns, seed, q0="orth", ilo=ilo, ihi=ihi)
    H, T, Q, Z = (A.copy(order="F") for A in (p.H, p.T, p.Q, p.Z))
    oracle.qz_sweep(H, T, Q, Z, ilo, ihi, p.shifts_re, p.shifts_im)
    assert np.all(np.tril(H, -2) == 0.0) and np.all(np.tril(T, -1) == 0.0)
    assert np.array_equal(H[:ilo, :ilo], p.H[:ilo, :ilo]) and np.array_equal(T[:ilo, :ilo], p.T[:ilo, :ilo])
    assert np.array_equal(H[ihi + 1:, ihi + 1:], p.H[ihi + 1:, ihi + 1:])
    assert np.array_equal(T[ihi + 1:, ihi + 1:], p.T[ihi + 1:, ihi + 1:])
    I = np.eye(n)
    assert np.linalg.norm(Q.T @ Q - I) <= 1e-13 * n and np.linalg.norm(Z.T @ Z - I) <= 1e-13 * n
    # (Q0 H0 Z0^T, Q0 T0 Z0^T) = (Q H Z^T, Q T Z^T): the pencil is preserved
    for A0, A in ((p.H, H), (p.T, T)):
        lhs = p.Q @ A0 @ p.Z.T
        assert np.linalg.norm(Q @ A @ Z.T - lhs) <= 1e-13 * n * np.linalg.norm(A0)


def _gen_eigs(H, T):
    """LAPACK-free generalized eigenvalues: roots of det(H - lam T) (exact rationals, sympy) at
    50 digits (mpmath)."""
    n = H.shape[0]
    lam = sp.Symbol("lam")
    M = sp.Matrix(n, n, lambda i, j: sp.Rational(Fraction(float(H[i, j]))) - lam * sp.Rational(Fraction(float(T[i, j]))))
    poly = sp.Poly(M.det(method="berkowitz"), lam)
    coeffs = [sp.Rational(c) for c in poly.all_coeffs()]
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


@pytest.mark.parametrize("n,ns,seed", [(4, 2, 7), (5, 2, 8), (6, 4, 9)])
def test_qz_generalized_eigenvalues_preserved(n, ns, seed):
    p, ilo, ihi = _qz_case(n, ns, seed, q0="eye")
    H, T = p.H.copy(order="F"), p.T.copy(order="F")
    oracle.qz_sweep(H, T, None, None, 0, n - 1, p.shifts_re, p.shifts_im)
    assert _match(_gen_eigs(H, T), _gen_eigs(p.H, p.T)) <= 1e-11


@pytest.mark.parametrize("n,seed", [(6, 10), (8, 11), (12, 12)])
def test_qz_perfect_shifts(n, seed):
    """Shifts = two exact generalized eigenvalues: the trailing 2 x 2 pair decouples."""
    p, _, _ = _qz_case(n, 2, seed, q0="eye")
    lam = _gen_eigs(p.H, p.T)
    cpx = [z for z in lam if z.imag > 1e-8]
    if cpx:
        z = cpx[0]
        re_, im_ = [z.real, z.real], [abs(z.imag), -abs(z.imag)]
    else:
        rl = sorted(lam, key=lambda z: -abs(z))
        re_, im_ = [rl[0].real, rl[1].real], [0.0, 0.0]
    H, T = p.H.copy(order="F"), p.T.copy(order="F")
    oracle.qz_sweep(H, T, None, None, 0, n - 1, re_, im_)
    assert abs(H[n - 2, n - 3]) <= 1e-11 * np.linalg.norm(p.H)
    ev = _gen_eigs(H[n - 2:, n - 2:], T[n - 2:, n - 2:])
    assert _match(ev, [complex(re_[0], im_[0]), complex(re_[1], im_[1])]) <= 1e-9
