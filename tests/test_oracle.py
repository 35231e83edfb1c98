"""Pins for the CPU oracle (``-m "not gpu"``): the oracle is checked against things other than
itself -- closed forms, exact rational arithmetic, the implicit-Q theorem evaluated as a
50-digit QR factorisation of the shifted polynomial, perfect-shift deflation, invariants, and
eigenvalues from the exact characteristic polynomial (LAPACK-free, n <= 8).

Each test names the mistake it catches (dropped term, wrong sign / index, transposed operand).
"""
import json
import os
from fractions import Fraction

import mpmath
import numpy as np
import pytest
import sympy as sp

import oracle
from hqr_inputs import hessenberg, random_case, make

GOLD = os.path.join(os.path.dirname(__file__), "golden")
U = 2.0 ** -53


def F(s):
    return Fraction(s)


# --------------------------------------------------------------------------------------------
# house (reading R2)
# --------------------------------------------------------------------------------------------

def test_house_exact_rational_122():
    # x = (1,2,2): ||x|| = 3, beta = -3, tau = (beta-x0)/beta = 4/3, v = (1, 2/4, 2/4)
    v, tau, beta = oracle.house([1.0, 2.0, 2.0])
    assert beta == -3.0 and abs(tau - 4.0 / 3.0) <= 2 * U and np.array_equal(v, [1.0, 0.5, 0.5])
    P = np.eye(3) - tau * np.outer(v, v)
    assert np.allclose(P, np.array([[-1, -2, -2], [-2, 2, -1], [-2, -1, 2]]) / 3.0, atol=4 * U)


@pytest.mark.parametrize("x", [[1.0, 0.0, 0.0], [-2.0, 0.0], [0.0, 0.0], [0.0, 0.0, 0.0]])
def test_house_identity_cases(x):
    v, tau, beta = oracle.house(x)
    assert tau == 0.0 and beta == x[0] and v[0] == 1.0 and not np.any(v[1:])


def test_house_34_and_sign_of_zero():
    v, tau, beta = oracle.house([3.0, 4.0])          # |image| = 5
    assert beta == -5.0
    P = np.eye(2) - tau * np.outer(v, v)
    y = P @ np.array([3.0, 4.0])
    assert abs(y[0] + 5.0) <= 8 * U * 5 and abs(y[1]) <= 8 * U * 5
    v, tau, beta = oracle.house([0.0, 3.0, 4.0])     # sign(0) = +1 -> beta = -||x||
    assert beta == -5.0 and tau == 1.0


@pytest.mark.parametrize("k", [600, -600, 1000, -1000])
def test_house_scaled_extremes(k):
    # R15: |x| ~ 2^k (1e180 .. 1e-300): the unscaled x0^2 + tail^2 would overflow / underflow; the
    # reflector is the one of x = (1, 2, 2) exactly (tau, v identical; beta scaled by 2^k)
    v, tau, beta = oracle.house(np.ldexp([1.0, 2.0, 2.0], k))
    v0, tau0, beta0 = oracle.house([1.0, 2.0, 2.0])
    assert np.array_equal(v, v0) and tau == tau0 and beta == np.ldexp(beta0, k)
    v, tau, beta = oracle.house(np.ldexp([3.0, 4.0], k))
    assert beta == np.ldexp(-5.0, k) and np.isfinite(tau)
    # a tail far below the head but representable: still a (tiny) rotation, not the identity
    v, tau, beta = oracle.house([np.ldexp(1.0, k), np.ldexp(1.0, k - 200), 0.0])
    assert beta == -np.ldexp(1.0, k) and tau == 0.0 or abs(v[1]) <= 2.0 ** -199


@pytest.mark.parametrize("seed", range(20))
def test_house_random_maps_to_beta_e1(seed):
    g = np.random.default_rng(seed)
    x = g.standard_normal(3) * 10.0 ** g.integers(-3, 4)
    v, tau, beta = oracle.house(x)
    P = np.eye(3) - tau * np.outer(v, v)
    y = P @ x
    nx = np.linalg.norm(x)
    assert abs(y[0] - beta) <= 16 * U * nx and np.all(np.abs(y[1:]) <= 16 * U * nx)
    assert np.sign(beta) == -np.sign(x[0])
    assert np.linalg.norm(P @ P.T - np.eye(3)) <= 16 * U


# --------------------------------------------------------------------------------------------
# first column (reading R1): explicit product (H - s I)(H - s' I) e1 in exact rationals
# --------------------------------------------------------------------------------------------

def _shifted_first_col_exact(Hq, s1, s2, ilo):
    n = len(Hq)
    e = [Fraction(0)] * n
    e[ilo] = Fraction(1)

    def mv(vec, s):
        return [sum(Hq[i][k] * vec[k] for k in range(n)) - s * vec[i] for i in range(n)]

    return mv(mv(e, s2), s1)


@pytest.mark.parametrize("seed", range(10))
def test_first_column_matches_explicit_product(seed):
    g = np.random.default_rng(100 + seed)
    n, ilo = 7, int(g.integers(0, 3))
    Hi = np.triu(g.integers(-4, 5, (n, n)), -1).astype(float)
    Hi[np.arange(1, n), np.arange(n - 1)] = g.integers(1, 4, n - 1)
    s1, s2 = Fraction(int(g.integers(-3, 4)), 2), Fraction(int(g.integers(-3, 4)), 4)
    # the active block starts at ilo: (B - s1 I)(B - s2 I) e1 with B = H[ilo:, ilo:]
    Bq = [[Fraction(int(Hi[i, j])) for j in range(ilo, n)] for i in range(ilo, n)]
    exact = _shifted_first_col_exact(Bq, s1, s2, 0)
    x, e2 = oracle.first_column(np.asfortranarray(Hi), ilo, (float(s1), float(s2)))
    assert all(Fraction(x[i]) * Fraction(2) ** e2 == exact[i] for i in range(3))
    assert all(v == 0 for v in exact[3:])
    # scale invariance (R15): H and the shifts times 2^k give the same scaled vector, e2 + 2k; at
    # k = +-600 the unscaled products would overflow / underflow (|H| ~ 1e180 / 1e-180)
    for k in (600, -600, 7):
        xs, e2s = oracle.first_column(np.asfortranarray(np.ldexp(Hi, k)), ilo,
                                      (float(np.ldexp(float(s1), k)), float(np.ldexp(float(s2), k))))
        assert np.array_equal(xs, x) and e2s == e2 + 2 * k
    # a conjugate pair (a +- bi): pi = a^2 + b^2, sigma = 2a
    a, b = Fraction(int(g.integers(-3, 4)), 2), Fraction(int(g.integers(1, 4)), 2)
    Bc = [[Fraction(int(Hi[i, j])) for j in range(ilo, n)] for i in range(ilo, n)]
    e1 = [Fraction(int(i == 0)) for i in range(n - ilo)]
    mv = lambda v: [sum(Bc[i][k] * v[k] for k in range(n - ilo)) for i in range(n - ilo)]
    Hv, HHv = mv(e1), mv(mv(e1))
    exact_c = [HHv[i] - 2 * a * Hv[i] + (a * a + b * b) * e1[i] for i in range(n - ilo)]
    x, e2 = oracle.first_column(np.asfortranarray(Hi), ilo, (float(a), float(a)), (float(b), float(-b)))
    assert all(Fraction(x[i]) * Fraction(2) ** e2 == exact_c[i] for i in range(3))


# --------------------------------------------------------------------------------------------
# 6x6 worked example (tests/golden/francis_6x6.json)
# --------------------------------------------------------------------------------------------

def _gold():
    with open(os.path.join(GOLD, "francis_6x6.json")) as f:
        return json.load(f)


def test_worked_example_6x6_exact_values():
    g = _gold()
    H0 = np.asfortranarray(np.array(g["H_rows"], dtype=float))
    H, Z = H0.copy(order="F"), np.asfortranarray(np.eye(6))
    x, e2 = oracle.first_column(H0, 0, (1.0, 2.0))   # shifts 1, 2: sigma = 3, pi = 2
    assert [Fraction(t) * Fraction(2) ** e2 for t in x] == [F(s) for s in g["first_column"]]
    v, tau, beta = oracle.house(x)   # the reflector of the scaled vector; beta scales back by 2^e2
    assert Fraction(beta) * Fraction(2) ** e2 == F(g["house_beta"]) and abs(tau - float(F(g["house_tau"]))) <= 2 * U
    oracle.sweep(H, Z, 0, 5, g["shifts_re"], g["shifts_im"])
    assert abs(H[0, 0] - float(F(g["Hp00"]))) <= 8 * U * 4
    assert np.allclose(Z[:, 0], [float(F(s)) for s in g["Zp_col0"]], atol=4 * U, rtol=0)
    assert abs(np.trace(H) - float(F(g["trace"]))) <= 64 * U * 11
    assert np.all(np.tril(H, -2) == 0.0)
    # eigenvalues of H' are the roots of the exact characteristic polynomial of the integer H
    lam_ref = [complex(r) for r in mpmath.polyroots(g["charpoly_desc"], maxsteps=200, extraprec=200)]
    lam = _eig_charpoly(H)
    assert _match(lam, lam_ref) <= 1e-12


def _eig_charpoly(A):
    """LAPACK-free eigenvalues: exact rational characteristic polynomial of the float matrix
    (sympy), roots by mpmath at 50 digits."""
    n = A.shape[0]
    M = sp.Matrix(n, n, lambda i, j: sp.Rational(Fraction(float(A[i, j]))))
    coeffs = [sp.Rational(c) for c in M.charpoly().all_coeffs()]
    with mpmath.workdps(50):
        roots = mpmath.polyroots([mpmath.mpf(c.p) / c.q for c in coeffs], maxsteps=400, extraprec=400)
    return [complex(r) for r in roots]


def _match(a, b):
    a = list(a)
    b = list(b)
    worst = 0.0
    for z in a:
        k = int(np.argmin([abs(z - w) for w in b]))
        worst = max(worst, abs(z - b[k]) / max(1.0, abs(b[k])))
        b.pop(k)
    return worst


# --------------------------------------------------------------------------------------------
# Implicit-Q theorem: one sweep with shift pairs j = 0..nb-1 equals the QR step on the
# shifted polynomial M = prod_j (H^2 - sigma_j H + pi_j I) restricted to the active block:
# Z' = Z0 Q_M D and H' = D Q_M^T H Q_M D (D = diag(+-1)), Q_M from a 50-digit Gram-Schmidt QR.
# Catches: dropped/wrong term anywhere in left, right or Z updates, wrong row range of the
# right update (bulge entry missing), transposed reflector, wrong shift pairing.
# --------------------------------------------------------------------------------------------

def _implicit_q_reference(H, ilo, ihi, re, im):
    n = H.shape[0]
    N = ihi - ilo + 1
    with mpmath.workdps(50):
        B = mpmath.matrix(N, N)
        for i in range(N):
            for j in range(N):
                B[i, j] = mpmath.mpf(float(H[ilo + i, ilo + j]))
        M = mpmath.eye(N)
        for j in range(len(re) // 2):
            sigma = mpmath.mpf(re[2 * j]) + mpmath.mpf(re[2 * j + 1])
            pi = mpmath.mpf(re[2 * j]) * mpmath.mpf(re[2 * j + 1]) - mpmath.mpf(im[2 * j]) * mpmath.mpf(im[2 * j + 1])
            M = (B * B - sigma * B + pi * mpmath.eye(N)) * M
        Q = mpmath.matrix(N, N)
        for j in range(N):  # modified Gram-Schmidt (50 digits)
            w = M[:, j]
            for k in range(j):
                w = w - (Q[:, k].T * w)[0] * Q[:, k]
            Q[:, j] = w / mpmath.norm(w)
        Qf = np.array([[float(Q[i, j]) for j in range(N)] for i in range(N)])
        Hp = Q.T * B * Q
        Hpf = np.array([[float(Hp[i, j]) for j in range(N)] for i in range(N)])
    Qfull = np.eye(n)
    Qfull[ilo:ihi + 1, ilo:ihi + 1] = Qf
    Href = Qfull.T @ H @ Qfull
    Href[ilo:ihi + 1, ilo:ihi + 1] = Hpf
    return Qfull, Href


@pytest.mark.parametrize("case", [
    (0, 6, 2, 0, None, "eye"), (1, 9, 2, 0, None, "orth"), (2, 10, 4, 0, None, "eye"),
    (3, 12, 4, 2, 9, "orth"), (4, 11, 6, 1, None, "eye"), (5, 3, 2, 0, None, "eye"),
    (6, 4, 2, 0, None, "orth"), (7, 14, 8, 0, 12, "eye"),
])
def test_implicit_q_theorem(case):
    seed, n, ns, ilo, ihi, z0 = case
    ihi = n - 1 if ihi is None else ihi
    H0, Z0, re, im = random_case(seed, n, ns, ilo, ihi, upper="u11", z0=z0)
    H, Z = H0.copy(order="F"), Z0.copy(order="F")
    oracle.sweep(H, Z, ilo, ihi, re, im)
    Qfull, Href = _implicit_q_reference(H0, ilo, ihi, re, im)
    Zref = Z0 @ Qfull
    d = np.sign(np.sum(Z * Zref, axis=0))
    d[d == 0] = 1.0
    assert np.linalg.norm(Z - Zref * d) <= 1e-11 * np.sqrt(n)
    Hd = (Href * d).T * d
    Hd = Hd.T
    assert np.linalg.norm(H - Hd) <= 1e-11 * np.linalg.norm(H0)


# --------------------------------------------------------------------------------------------
# Perfect shifts: shifts = two exact eigenvalues => the trailing 2x2 decouples and carries them
# --------------------------------------------------------------------------------------------

@pytest.mark.parametrize("seed", range(6))
def test_perfect_shift_deflation(seed):
    n = 8
    g = np.random.default_rng(300 + seed)
    Hi = np.triu(g.integers(-3, 4, (n, n)), -1).astype(float)
    Hi[np.arange(1, n), np.arange(n - 1)] = g.integers(1, 3, n - 1)
    H0 = np.asfortranarray(Hi)
    lam = _eig_charpoly(H0)
    # pick a conjugate pair if present else the two largest real eigenvalues
    cpx = [z for z in lam if z.imag > 1e-8]
    if cpx:
        z = cpx[0]
        re, im = [z.real, z.real], [abs(z.imag), -abs(z.imag)]
    else:
        z1, z2 = lam[-1], lam[-2]
        re, im = [z1.real, z2.real], [0.0, 0.0]
    H, Z = H0.copy(order="F"), np.asfortranarray(np.eye(n))
    oracle.sweep(H, Z, 0, n - 1, re, im)
    hn = np.linalg.norm(H0)
    assert abs(H[n - 2, n - 3]) <= 1e-11 * hn
    T = H[n - 2:, n - 2:]
    tr, det = T[0, 0] + T[1, 1], T[0, 0] * T[1, 1] - T[0, 1] * T[1, 0]
    assert abs(tr - (re[0] + re[1])) <= 1e-10 * hn
    assert abs(det - (re[0] * re[1] - im[0] * im[1])) <= 1e-10 * hn * hn


@pytest.mark.parametrize("seed,n,ns", [(0, 5, 2), (1, 7, 4), (2, 8, 6), (3, 6, 4)])
def test_spectrum_preserved_charpoly(seed, n, ns):
    H0, Z0, re, im = random_case(40 + seed, n, ns, upper="u11")
    H = H0.copy(order="F")
    oracle.sweep(H, None, 0, n - 1, re, im)
    assert _match(_eig_charpoly(H), _eig_charpoly(H0)) <= 1e-11


# --------------------------------------------------------------------------------------------
# Structure and invariants at moderate n (BASELINE north_star checks)
# --------------------------------------------------------------------------------------------

@pytest.mark.parametrize("n,ns,ilo,ihi,z0", [(150, 12, 20, 120, "orth"), (256, 8, 0, 255, "eye"),
                                             (200, 30, 0, 199, "orth"), (64, 40, 3, 60, "eye")])
def test_structure_and_invariants(n, ns, ilo, ihi, z0):
    H0, Z0, re, im = random_case(n + ns, n, ns, ilo, ihi, z0=z0, shift_kind="disk2")
    H, Z = H0.copy(order="F"), Z0.copy(order="F")
    oracle.sweep(H, Z, ilo, ihi, re, im)
    assert np.all(np.tril(H, -2) == 0.0)
    # blocks outside the active window are bitwise untouched
    assert np.array_equal(H[:ilo, :ilo], H0[:ilo, :ilo])
    assert np.array_equal(H[ihi + 1:, ihi + 1:], H0[ihi + 1:, ihi + 1:])
    assert np.array_equal(H[ilo:ihi + 1, :ilo], H0[ilo:ihi + 1, :ilo])
    assert H[ilo, ilo - 1] == 0.0 if ilo > 0 else True
    assert np.linalg.norm(Z.T @ Z - np.eye(n)) <= 1e-13 * n
    hn = np.linalg.norm(H0)
    assert np.linalg.norm(Z @ H @ Z.T - Z0 @ H0 @ Z0.T) / hn <= 1e-13 * n
    assert abs(np.trace(H) - np.trace(H0)) <= 1e-13 * n * hn
    assert abs(np.linalg.norm(H) - hn) <= 1e-13 * n * hn


def test_config0_pipelined_vs_sequential_noise_floor():
    p = make(0)
    Hs, Zs = p.H.copy(order="F"), p.Z.copy(order="F")
    Hp, Zp = p.H.copy(order="F"), p.Z.copy(order="F")
    oracle.sweep(Hs, Zs, p.ilo, p.ihi, p.shifts_re, p.shifts_im, order="sequential")
    oracle.sweep(Hp, Zp, p.ilo, p.ihi, p.shifts_re, p.shifts_im, order="pipelined")
    n = p.H.shape[0]
    assert np.linalg.norm(Hs - Hp) / np.linalg.norm(p.H) <= 1e-12
    assert np.linalg.norm(Zs - Zp) <= 1e-12 * np.sqrt(n)
    assert not np.array_equal(Hs, Hp)  # two genuinely different rounding orders


def test_block_commutation():
    # two decoupled blocks (the BJ.configs[4] situation in miniature): order of blocks is rounding only
    n = 120
    H0 = hessenberg(n, "n01", 77)
    H0[60, 59] = 0.0
    from hqr_inputs import shifts
    re, im = shifts("disk2", 8, 77)
    Ha, Za = H0.copy(order="F"), np.asfortranarray(np.eye(n))
    Hb, Zb = H0.copy(order="F"), np.asfortranarray(np.eye(n))
    oracle.sweep(Ha, Za, 0, 59, re[:4], im[:4]); oracle.sweep(Ha, Za, 60, 119, re[4:], im[4:])
    oracle.sweep(Hb, Zb, 60, 119, re[4:], im[4:]); oracle.sweep(Hb, Zb, 0, 59, re[:4], im[:4])
    assert np.linalg.norm(Ha - Hb) <= 1e-13 * np.linalg.norm(H0)
    assert np.linalg.norm(Za - Zb) <= 1e-13 * np.sqrt(n)
    assert Ha[60, 59] == 0.0


def test_flops_formula_small():
    # F_alg by enumeration of (left columns + right rows + Z rows) per reflector, n = 10, 1 bulge
    n, ilo, ihi = 10, 0, 9
    tot = 0
    for p in range(ilo - 1, ihi - 1):
        m = 3 if p <= ihi - 3 else 2
        cols = n - (ilo if p == ilo - 1 else p + 1)
        rows = min(p + m + 1, ihi) + 1
        tot += (10 if m == 3 else 6) * (cols + rows + n)
    assert oracle.flops(n, ilo, ihi, 1) == tot
    assert oracle.flops(n, ilo, ihi, 3) == 3 * tot


def test_flops_match_survey_table():
    # F_alg of the BASELINE configs as tabulated in SURVEY.md §8(d) (derived there independently
    # of this code, 4 significant digits): catches a wrong term count or range in oracle_flops
    table = {0: (256, [(0, 255, 8)], 5.255e6), 1: (4000, [(0, 3999, 100)], 1.600e10),
             2: (10000, [(0, 9999, 256)], 2.560e11), 3: (20000, [(0, 19999, 512)], 2.048e12),
             4: (40000, [(b * 10000, b * 10000 + 9999, 512) for b in range(4)], 8.191e12)}
    for cfg, (n, blocks, want) in table.items():
        got = sum(oracle.flops(n, lo, hi, ns // 2) for lo, hi, ns in blocks)
        assert abs(got - want) <= 0.0005 * want, (cfg, got, want)


@pytest.mark.parametrize("k", [600, -600])
def test_sweep_scale_equivariance(k):
    # R15: scaling H and the shifts by 2^k scales H' by 2^k bit for bit and leaves Z' unchanged
    # (every step is linear in H or scale invariant); at k = +-600 the unscaled bulge vector
    # (~|H|^2) would overflow / underflow, so this also pins the scaled first column and house
    n, ns = 60, 10
    H0, Z0, re, im = random_case(91, n, ns, z0="orth", shift_kind="disk2")
    H, Z = H0.copy(order="F"), Z0.copy(order="F")
    oracle.sweep(H, Z, 0, n - 1, re, im)
    Hs, Zs = np.asfortranarray(np.ldexp(H0, k)), Z0.copy(order="F")
    oracle.sweep(Hs, Zs, 0, n - 1, np.ldexp(re, k), np.ldexp(im, k))
    assert np.all(np.isfinite(Hs)) and np.array_equal(Hs, np.ldexp(H, k)) and np.array_equal(Zs, Z)


def test_hess_n_workload_sweep_invariants():
    # NEXT-3 workload: graded chi^2 subdiagonal, shifts in the disk of radius sqrt(n)
    from hqr_inputs import make_hess
    p = make_hess(300, 40, z0="orth")
    sub = np.diag(p.H, -1)
    assert sub[0] > 10.0 and np.all(sub > 0) and np.all(np.tril(p.H, -2) == 0)
    H, Z = p.H.copy(order="F"), p.Z.copy(order="F")
    oracle.sweep(H, Z, 0, 299, p.shifts_re, p.shifts_im)
    n, hn = 300, np.linalg.norm(p.H)
    assert np.all(np.tril(H, -2) == 0.0)
    assert np.linalg.norm(Z.T @ Z - np.eye(n)) <= 1e-13 * n
    assert np.linalg.norm(Z @ H @ Z.T - p.Z @ p.H @ p.Z.T) / hn <= 1e-13 * n


# --------------------------------------------------------------------------------------------
# Subdiagonal scan (aftermath vector; reading R16)
# --------------------------------------------------------------------------------------------

def test_subdiag_scan_closed_cases():
    n = 10
    H = np.asfortranarray(np.triu(np.ones((n, n)), -1) * 2.0)
    H[3, 2] = 0.0                     # exact zero -> 2
    H[6, 5] = 2.0 ** -52 * 4.0        # = eps (|h55| + |h66|) exactly -> 1 (boundary included)
    H[8, 7] = np.nextafter(2.0 ** -52 * 4.0, 1.0)   # one ulp above -> 0
    f = oracle.subdiag_scan(H, [(0, n - 1)])
    want = np.zeros(n, dtype=np.int8)
    want[2], want[5], want[9] = 2, 1, -1  # row n-1 has no subdiagonal entry
    assert np.array_equal(f, want)
    # only rows ilo-1 .. ihi of each block are scanned; ilo-1 / ihi are the decoupling zeros
    H[4, 3] = 0.0
    f = oracle.subdiag_scan(H, [(4, 6)])
    assert list(f) == [-1, -1, -1, 2, 0, 1, 0, -1, -1, -1]
    f = oracle.subdiag_scan(H, [(0, 2), (3, 3 + 2)])
    assert list(f[:6]) == [0, 0, 2, 2, 0, 1]
