"""CPU oracle for one multishift QR sweep -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  It shares no code with the CUDA product
path (``paper_2007_03576_b200``): the arithmetic lives in ``oracle/hqr_oracle.c`` (plain C,
fp64, OpenMP over independent rows/columns only), this module only marshals arguments.

Functions and the passages they follow (PAPER.md line numbers, see hqr_oracle.c):
  house(x)                 -- 3x3 / 2x2 Householder reflector, P:200 (reading R2 in DESIGN.md)
  first_column(H, ilo, ..) -- first column of (H - s I)(H - s' I), P:200 (reading R1), scaled
                              by a power of two (reading R15)
  sweep(H, Z, ...)         -- nshifts/2 sequential Francis double steps on the full matrix,
                              P:146-151, P:198-206, P:227-233
  flops(...)               -- F_alg, the work of applying every reflector directly
  subdiag_scan(H, ...)     -- the aftermath subdiagonal scan, P:379-381 (reading R16)
  rhs_house(r)             -- right-hand side reflector r P = beta e_m^T (reading R18)
  qz_first_column(H, T ..) -- (H T^-1 - s I)(H T^-1 - s' I) e1, P:209 (reading R17)
  qz_sweep(H, T, Q, Z, ..) -- nshifts/2 sequential double-shift QZ steps
  small_eig(A)             -- eigenvalues of a small Hessenberg matrix, Francis double-shift QR
                              (the small Schur task's role; reading R21)
  qr_iterate(H, Z, ..)     -- repeated sweeps with shifts from the trailing block and deflation
                              (NEXT-2 without AED; reading R21)
  schur(A) / aed(H, ..)    -- real Schur form with U; aggressive early deflation on a window
                              (reading R22) with the failed blocks
                              reordered to the top (reading R23)
  swap(T, U, i, p, q)      -- swap of two adjacent diagonal blocks of a quasi-triangular T
                              (the reordering kernel; reading R23)
  qr_iterate_aed(H, Z, ..) -- the QR iteration with AED (NEXT-2, R22)

Parity pins for every function are in tests/test_oracle.py (none is "parity unpinned").
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hqr_oracle.c")
_LIB_PATH = os.path.join(_HERE, "_build", "libhqr_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2 -fopenmp, no FMA contraction: reading R10)."""
    os.makedirs(os.path.dirname(_LIB_PATH), exist_ok=True)
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-ffp-contract=off", "-std=c11",
               "-o", _LIB_PATH, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        dp = ctypes.POINTER(ctypes.c_double)
        lib.oracle_house.argtypes = [ctypes.c_int, dp, dp, dp, dp]
        lib.oracle_house.restype = None
        lib.oracle_first_column.argtypes = [dp, ctypes.c_int64, ctypes.c_int64, ctypes.c_double,
                                            ctypes.c_double, ctypes.c_double, ctypes.c_double, dp,
                                            ctypes.POINTER(ctypes.c_int)]
        lib.oracle_first_column.restype = None
        lib.oracle_sweep.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                     ctypes.c_int64, dp, dp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_int]
        lib.oracle_sweep.restype = ctypes.c_int
        lib.oracle_flops.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                     ctypes.c_int]
        lib.oracle_flops.restype = ctypes.c_double
        lib.oracle_subdiag_scan.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                            ctypes.c_int64, ctypes.c_void_p]
        lib.oracle_subdiag_scan.restype = None
        lib.oracle_rhs_house.argtypes = [ctypes.c_int, dp, dp, dp, dp]
        lib.oracle_rhs_house.restype = None
        lib.oracle_qz_first_column.argtypes = [dp, dp, ctypes.c_int64, ctypes.c_int64, ctypes.c_double,
                                               ctypes.c_double, ctypes.c_double, ctypes.c_double, dp]
        lib.oracle_qz_first_column.restype = None
        lib.oracle_qz_sweep.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int64] * 3 + [dp, dp, ctypes.c_int,
                                                                                       ctypes.c_int]
        lib.oracle_qz_sweep.restype = ctypes.c_int
        lib.oracle_small_eig.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, dp, dp]
        lib.oracle_small_eig.restype = ctypes.c_int
        lib.oracle_qr_iterate.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                          ctypes.c_int64, ctypes.c_int, ctypes.c_int64, ctypes.c_int, dp, dp,
                                          ctypes.POINTER(ctypes.c_int)]
        lib.oracle_qr_iterate.restype = ctypes.c_int
        ip = ctypes.POINTER(ctypes.c_int)
        lib.oracle_schur.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                     dp, dp]
        lib.oracle_schur.restype = ctypes.c_int
        lib.oracle_swap.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                                    ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int]
        lib.oracle_swap.restype = ctypes.c_int
        lib.oracle_aed.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                   ctypes.c_int, ctypes.c_double, dp, dp, dp, dp, ip]
        lib.oracle_aed.restype = ctypes.c_int
        lib.oracle_qr_iterate_aed.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                              ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int,
                                              dp, dp, ip, ip, ip]
        lib.oracle_qr_iterate_aed.restype = ctypes.c_int
        _lib = lib
    return _lib


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def house(x):
    """Return (v, tau, beta) with (I - tau v v^T) x = beta e1 (reading R2)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    m = x.shape[0]
    v = np.zeros(m)
    tau = ctypes.c_double()
    beta = ctypes.c_double()
    _load().oracle_house(m, _dptr(x), _dptr(v), ctypes.byref(tau), ctypes.byref(beta))
    return v, tau.value, beta.value


def first_column(H: np.ndarray, ilo: int, re_pair, im_pair=(0.0, 0.0)):
    """(x, e2): the first column of (H - s I)(H - s' I) at rows ilo..ilo+2 is x * 2**e2 (x is
    computed on inputs scaled by a power of two, reading R15).  re_pair / im_pair: the shift pair
    (s, s') as real and imaginary parts."""
    H = _as_colmajor(H)
    x = np.zeros(3)
    e2 = ctypes.c_int()
    _load().oracle_first_column(_dptr(H), H.shape[0], ilo, float(re_pair[0]), float(re_pair[1]),
                                float(im_pair[0]), float(im_pair[1]), _dptr(x), ctypes.byref(e2))
    return x, e2.value


def _as_colmajor(a: np.ndarray) -> np.ndarray:
    if a.dtype != np.float64 or not a.flags.f_contiguous:
        raise TypeError("oracle expects float64 Fortran-ordered (column-major) arrays")
    return a


def sweep(H: np.ndarray, Z: np.ndarray | None, ilo: int, ihi: int, shifts_re, shifts_im,
          order: str = "sequential", bulges: tuple[int, int] | None = None) -> None:
    """In place: H <- Q^T H Q, Z <- Z Q for one multishift sweep.

    H, Z: n x n float64 Fortran-ordered.  order: "sequential" (the oracle) or "pipelined"
    (noise-floor measurement only).  bulges=(j0, j1) restricts to shift pairs j0..j1-1.
    """
    H = _as_colmajor(H)
    n = H.shape[0]
    if Z is not None:
        Z = _as_colmajor(Z)
        assert Z.shape == (n, n)
    sr = np.ascontiguousarray(shifts_re, dtype=np.float64)
    si = np.ascontiguousarray(shifts_im, dtype=np.float64)
    ns = sr.shape[0]
    nb = ns // 2
    j0, j1 = bulges if bulges is not None else (0, nb)
    o = {"sequential": 0, "pipelined": 1}[order]
    _load().oracle_sweep(H.ctypes.data, None if Z is None else Z.ctypes.data, n, ilo, ihi,
                         _dptr(sr), _dptr(si), ns, o, j0, j1)


def flops(n: int, ilo: int, ihi: int, nbulges: int, with_z: bool = True) -> float:
    return _load().oracle_flops(n, ilo, ihi, nbulges, 1 if with_z else 0)


def subdiag_scan(H: np.ndarray, blocks) -> np.ndarray:
    """Aftermath flags (int8, n entries) of H for the active blocks [(ilo, ihi), ...]: 2 exact
    zero, 1 negligible (|h| <= 2^-52 (|h_ii| + |h_i+1,i+1|)), 0 otherwise, -1 not scanned."""
    H = _as_colmajor(H)
    n = H.shape[0]
    flags = np.full(n, -1, dtype=np.int8)
    for ilo, ihi in blocks:
        _load().oracle_subdiag_scan(H.ctypes.data, n, ilo, ihi, flags.ctypes.data)
    return flags


def rhs_house(r):
    """(u, tau, beta) with r (I - tau u u^T) = beta e_m^T, u[m-1] = 1 (reading R18)."""
    r = np.ascontiguousarray(r, dtype=np.float64)
    m = r.shape[0]
    u = np.zeros(m)
    tau = ctypes.c_double()
    beta = ctypes.c_double()
    _load().oracle_rhs_house(m, _dptr(r), _dptr(u), ctypes.byref(tau), ctypes.byref(beta))
    return u, tau.value, beta.value


def qz_first_column(H, T, ilo, re_pair, im_pair=(0.0, 0.0)):
    H, T = _as_colmajor(H), _as_colmajor(T)
    x = np.zeros(3)
    _load().oracle_qz_first_column(_dptr(H), _dptr(T), H.shape[0], ilo, float(re_pair[0]),
                                   float(re_pair[1]), float(im_pair[0]), float(im_pair[1]), _dptr(x))
    return x


def qz_sweep(H, T, Q, Z, ilo, ihi, shifts_re, shifts_im, bulges=None):
    """In place: (H, T) <- Q_s^T (H, T) Z_s, Q <- Q Q_s, Z <- Z Z_s for one multishift QZ sweep
    (Q / Z may be None).  Column-major float64 arrays."""
    H, T = _as_colmajor(H), _as_colmajor(T)
    n = H.shape[0]
    for A in (Q, Z):
        if A is not None:
            _as_colmajor(A)
    sr = np.ascontiguousarray(shifts_re, dtype=np.float64)
    si = np.ascontiguousarray(shifts_im, dtype=np.float64)
    j0, j1 = bulges if bulges is not None else (0, sr.shape[0] // 2)
    _load().oracle_qz_sweep(H.ctypes.data, T.ctypes.data, None if Q is None else Q.ctypes.data,
                            None if Z is None else Z.ctypes.data, n, ilo, ihi, _dptr(sr), _dptr(si), j0, j1)


def small_eig(A):
    """Eigenvalues (wr, wi, info) of the small upper-Hessenberg matrix A (not modified)."""
    B = np.asfortranarray(np.array(A, dtype=np.float64))
    m = B.shape[0]
    wr, wi = np.zeros(m), np.zeros(m)
    info = _load().oracle_small_eig(B.ctypes.data, m, m, _dptr(wr), _dptr(wi))
    return wr, wi, info


def qr_iterate(H, Z, ilo, ihi, nshifts, nmin=64, max_sweeps=1000):
    """In place: the QR iteration of R21 on H (and Z).  Returns (wr, wi, rc, sweeps)."""
    H = _as_colmajor(H)
    n = H.shape[0]
    wr, wi = np.zeros(n), np.zeros(n)
    sw = ctypes.c_int()
    rc = _load().oracle_qr_iterate(H.ctypes.data, None if Z is None else _as_colmajor(Z).ctypes.data, n, ilo,
                                   ihi, nshifts, nmin, max_sweeps, _dptr(wr), _dptr(wi), ctypes.byref(sw))
    return wr, wi, rc, sw.value


def schur(A):
    """(T, U, wr, wi, info): real Schur form T = U^T A U of the small Hessenberg matrix A."""
    T = np.asfortranarray(np.array(A, dtype=np.float64))
    m = T.shape[0]
    U = np.asfortranarray(np.eye(m))
    wr, wi = np.zeros(m), np.zeros(m)
    info = _load().oracle_schur(T.ctypes.data, m, m, U.ctypes.data, m, _dptr(wr), _dptr(wi))
    return T, U, wr, wi, info


def swap(T, U, i, p, q):
    """In place: swap the diagonal blocks T(i:i+p) and T(i+p:i+p+q) (p, q in {1, 2}), U <- U Q.
    Returns 0, or 1 when the swap was rejected (T, U unchanged)."""
    T = _as_colmajor(T)
    U = _as_colmajor(U)
    nw = T.shape[0]
    return _load().oracle_swap(T.ctypes.data, nw, nw, U.ctypes.data, nw, i, p, q)


def aed(H, Z, ilo, k0, nw, thr):
    """In place AED on the window [k0, k0+nw) of H (block from ilo): (nd, wr, wi, shift candidates)."""
    H = _as_colmajor(H)
    n = H.shape[0]
    wr, wi = np.zeros(n), np.zeros(n)
    swr, swi = np.zeros(nw), np.zeros(nw)
    nund = ctypes.c_int()
    nd = _load().oracle_aed(H.ctypes.data, None if Z is None else _as_colmajor(Z).ctypes.data, n, ilo, k0, nw, thr,
                            _dptr(wr), _dptr(wi), _dptr(swr), _dptr(swi), ctypes.byref(nund))
    return nd, wr, wi, swr[:nund.value] + 1j * swi[:nund.value]


def qr_iterate_aed(H, Z, ilo, ihi, nshifts, nw=96, nmin=64, max_sweeps=1000):
    """In place: the QR iteration with AED (R22).  Returns (wr, wi, rc, sweeps, aed_steps, aed_deflated)."""
    H = _as_colmajor(H)
    n = H.shape[0]
    wr, wi = np.zeros(n), np.zeros(n)
    sw, na, nd = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    rc = _load().oracle_qr_iterate_aed(H.ctypes.data, None if Z is None else _as_colmajor(Z).ctypes.data, n, ilo,
                                       ihi, nshifts, nw, nmin, max_sweeps, _dptr(wr), _dptr(wi), ctypes.byref(sw),
                                       ctypes.byref(na), ctypes.byref(nd))
    return wr, wi, rc, sw.value, na.value, nd.value
