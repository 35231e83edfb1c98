"""GPU parity of the generalized (QZ) sweep: hqr_qz_sweep through the C ABI
against the QZ oracle (oracle/hqr_oracle.c oracle_qz_sweep) on the same seeded inputs.

Tolerance as the QR sweep (BASELINE north_star): ||dH'||_F/||H||_F, ||dT'||_F/||T||_F <= 1e-10,
||dQ||_F, ||dZ||_F <= 1e-10 sqrt(n); H' Hessenberg and T' triangular with exact zeros."""
import numpy as np
import pytest

import oracle
import paper_2007_03576_b200 as hq
from hqr_inputs import make_qz

pytestmark = pytest.mark.gpu

TOL = 1e-10


@pytest.fixture(scope="module", autouse=True)
def lib_setup():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    hq.setup(0)
    yield
    hq.teardown()


def _case(n, ns, seed, ilo=0, ihi=None, q0="orth"):
    p = make_qz(n, ns, q0=q0, seed=seed)
    ihi = n - 1 if ihi is None else ihi
    if ilo > 0:
        p.H[ilo, ilo - 1] = 0.0
    if ihi < n - 1:
        p.H[ihi + 1, ihi] = 0.0
    return p, ilo, ihi


def _run(p, ilo, ihi, win, with_qz=True):
    d = [hq.to_device(A) for A in (p.H, p.T, p.Q, p.Z)]
    hq.qz_sweep(d[0], d[1], d[2] if with_qz else None, d[3] if with_qz else None, ilo, ihi,
                p.shifts_re, p.shifts_im, win)
    return [hq.from_device(A) for A in d]


def _oracle(p, ilo, ihi):
    H, T, Q, Z = (A.copy(order="F") for A in (p.H, p.T, p.Q, p.Z))
    oracle.qz_sweep(H, T, Q, Z, ilo, ihi, p.shifts_re, p.shifts_im)
    return H, T, Q, Z


CASES = [  # (n, nshifts, seed, ilo, ihi, window)
    (6, 2, 0, 0, None, 8), (30, 4, 1, 0, None, 8), (64, 8, 2, 0, None, 64), (101, 12, 3, 3, 97, 24),
    (200, 20, 4, 0, None, 40), (400, 40, 5, 0, None, 64), (513, 60, 6, 10, 500, 80),
    (1000, 80, 7, 0, None, 80), (1600, 120, 8, 0, None, 64),
]


@pytest.mark.parametrize("case", CASES, ids=[f"n{c[0]}s{c[1]}w{c[5]}" for c in CASES])
def test_qz_parity(case):
    n, ns, seed, ilo, ihi, win = case
    p, ilo, ihi = _case(n, ns, seed, ilo, ihi)
    Hg, Tg, Qg, Zg = _run(p, ilo, ihi, win)
    Ho, To, Qo, Zo = _oracle(p, ilo, ihi)
    assert np.linalg.norm(Hg - Ho) / np.linalg.norm(p.H) <= TOL
    assert np.linalg.norm(Tg - To) / np.linalg.norm(p.T) <= TOL
    assert np.linalg.norm(Qg - Qo) <= TOL * np.sqrt(n)
    assert np.linalg.norm(Zg - Zo) <= TOL * np.sqrt(n)
    assert np.all(np.tril(Hg, -2) == 0.0) and np.all(np.tril(Tg, -1) == 0.0)
    assert np.array_equal(Hg[:ilo, :ilo], p.H[:ilo, :ilo]) and np.array_equal(Tg[:ilo, :ilo], p.T[:ilo, :ilo])
    assert np.array_equal(Hg[ihi + 1:, ihi + 1:], p.H[ihi + 1:, ihi + 1:])


def test_qz_without_accumulators_and_identity_T():
    n = 300
    p, ilo, ihi = _case(n, 24, 9)
    Hg, Tg, _, _ = _run(p, ilo, ihi, 64, with_qz=False)
    Hf, Tf, _, _ = _run(p, ilo, ihi, 64, with_qz=True)
    assert np.array_equal(Hg, Hf) and np.array_equal(Tg, Tf)   # Q / Z never feed back
    # T = I: H'T'^-1 is the QR sweep's H' (the QR kernels' result), T' = diag(+-1)
    p.T = np.asfortranarray(np.eye(n))
    Hq, Tq, _, _ = _run(p, 0, n - 1, 64, with_qz=False)
    d = np.diag(Tq)
    assert np.linalg.norm(Tq - np.diag(d)) <= 1e-12 and np.all(np.abs(np.abs(d) - 1) <= 1e-12)
    Hd, Zd = hq.to_device(p.H), None
    hq.sweep(Hd, Zd, 0, n - 1, p.shifts_re, p.shifts_im, 64)
    assert np.linalg.norm(Hq / d[None, :] - hq.from_device(Hd)) <= 1e-11 * np.linalg.norm(p.H)


def test_qz_error_codes():
    n = 50
    p, _, _ = _case(n, 4, 10)
    H, T = hq.to_device(p.H), hq.to_device(p.T)
    with pytest.raises(hq.HQRError) as e:
        hq.qz_sweep(H, T, None, None, 10, n - 1, p.shifts_re, p.shifts_im, 16)   # H[10, 9] != 0
    assert e.value.code == -10
    T0 = p.T.copy(order="F")
    T0[0, 0] = 0.0
    with pytest.raises(hq.HQRError) as e:
        hq.qz_sweep(H, hq.to_device(T0), None, None, 0, n - 1, p.shifts_re, p.shifts_im, 16)
    assert e.value.code == -2


def test_qz_parity_large():
    """n = 4000, 100 shifts, window 80 (the bench's QZ window): many chains and wavefront steps."""
    n = 4000
    p, ilo, ihi = _case(n, 100, 11)
    Hg, Tg, Qg, Zg = _run(p, ilo, ihi, 80)
    Ho, To, Qo, Zo = _oracle(p, ilo, ihi)
    assert np.linalg.norm(Hg - Ho) / np.linalg.norm(p.H) <= TOL
    assert np.linalg.norm(Tg - To) / np.linalg.norm(p.T) <= TOL
    assert np.linalg.norm(Qg - Qo) <= TOL * np.sqrt(n) and np.linalg.norm(Zg - Zo) <= TOL * np.sqrt(n)
    assert np.all(np.tril(Hg, -2) == 0.0) and np.all(np.tril(Tg, -1) == 0.0)
