"""Seeded synthetic inputs for the multishift QR sweep (BASELINE.json ``configs``).

Shared by the oracle tests, the GPU parity tests and bench.py.  This module holds NONE of the
method's arithmetic (no reflectors, no shifts polynomials): it only draws random numbers.

Recipe:
  RNG: numpy Generator(PCG64(SeedSequence([2020, cfg, stream]))); 2020 is the paper's test
       seed.  Streams: 0 upper entries, 1 subdiagonal, 2 shifts, 3 Z0 Gaussian.
  H:   upper-triangle entries (i <= j) drawn column by column (column-major order), subdiagonal
       h[j+1, j] drawn in order j = 0..n-2; everything below the subdiagonal is exactly 0.
  Z0:  identity, or the Q factor of a Householder QR of an n x n N(0,1) matrix (stream 3).
  shifts: consecutive pairs; real pair = two reals, complex pair = (a+bi, a-bi) adjacent.

Arrays are float64 Fortran-ordered (column-major, ld = n), the layout of the C ABI.
These inputs stand in for the paper's syn_n / SuiteSparse matrices: a sweep only
ever sees an upper-Hessenberg matrix, so only its shape and value distribution matter.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

SEED = 2020


def rng(cfg: int, stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([SEED, cfg, stream])))


@dataclass
class Config:
    idx: int
    n: int
    upper: str            # "u11" = U[-1,1], "n01" = N(0,1)
    z0: str               # "eye" or "orth"
    shifts: str           # "mixed" (half real pairs, half conj pairs) or "disk2"
    nshifts: int
    window: int | None    # None = library default
    blocks: int = 1       # number of unreduced diagonal blocks (config 4)
    name: str = ""
    gpus: tuple = field(default_factory=lambda: (1,))


CONFIGS = {
    0: Config(0, 256, "u11", "eye", "mixed", 8, 24, name="cfg0_n256_s8_w24"),
    1: Config(1, 4000, "u11", "orth", "mixed", 100, 151, name="cfg1_n4000_s100_w151"),
    2: Config(2, 10000, "n01", "eye", "disk2", 256, None, name="cfg2_n10000_s256", gpus=(1, 2, 4, 8)),
    3: Config(3, 20000, "n01", "orth", "disk2", 512, None, name="cfg3_n20000_s512", gpus=(1, 2, 4, 8)),
    4: Config(4, 40000, "n01", "eye", "disk2", 512, None, blocks=4, name="cfg4_n40000_4x512",
              gpus=(8,)),
}


def hessenberg(n: int, upper: str, cfg: int, blocks: int = 1, col_chunk: int = 512,
               subdiag: str = "u0515") -> np.ndarray:
    """Random upper-Hessenberg H (Fortran order).  blocks > 1 zeroes h[b*n/blocks, b*n/blocks - 1].
    subdiag: "u0515" = U[0.5, 1.5] (BASELINE configs) or "chi2" = the paper's hess_n recipe
    (after Braman et al.): h_{i+1,i}^2 ~ chi^2(n - i) (1-based i), i.e.
    h[i+1, i] = sqrt(chi^2(n - 1 - i)) 0-based -- graded from ~sqrt(n) at the top to ~1 at the
    bottom (the Hessenberg form of a Ginibre matrix)."""
    H = np.zeros((n, n), dtype=np.float64, order="F")
    g = rng(cfg, 0)
    for c0 in range(0, n, col_chunk):
        c1 = min(n, c0 + col_chunk)
        cnt = (c1 * (c1 + 1) - c0 * (c0 + 1)) // 2
        if upper == "u11":
            vals = g.uniform(-1.0, 1.0, cnt)
        elif upper == "n01":
            vals = g.standard_normal(cnt)
        else:
            raise ValueError(upper)
        off = 0
        for j in range(c0, c1):
            H[: j + 1, j] = vals[off: off + j + 1]
            off += j + 1
    if subdiag == "u0515":
        sub = rng(cfg, 1).uniform(0.5, 1.5, max(n - 1, 0))
    elif subdiag == "chi2":
        sub = np.sqrt(rng(cfg, 1).chisquare(np.arange(n - 1, 0, -1, dtype=np.float64)))
    else:
        raise ValueError(subdiag)
    idx = np.arange(n - 1)
    H[idx + 1, idx] = sub
    if blocks > 1:
        bs = n // blocks
        for b in range(1, blocks):
            H[b * bs, b * bs - 1] = 0.0
    return H


def orthogonal(n: int, cfg: int, device: str = "cpu") -> np.ndarray:
    """Q factor of a Householder QR of an n x n N(0,1) matrix drawn from stream 3 (Fortran order)."""
    G = rng(cfg, 3).standard_normal((n, n))
    if device == "cpu":
        Q, _ = np.linalg.qr(G)
        return np.asfortranarray(Q)
    import torch  # input generation only; not the product path
    Qt, _ = torch.linalg.qr(torch.from_numpy(G).to(device))
    return np.asfortranarray(Qt.cpu().numpy())


def shifts(kind: str, nshifts: int, cfg: int, stream_offset: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """Shift set as (re, im) arrays of length nshifts, conjugates adjacent."""
    g = rng(cfg, 2 + 10 * stream_offset)
    npairs = nshifts // 2
    re = np.zeros(nshifts)
    im = np.zeros(nshifts)
    if kind == "mixed":
        nreal = npairs // 2
        for j in range(npairs):
            if j < nreal:
                re[2 * j: 2 * j + 2] = g.uniform(-1.0, 1.0, 2)
            else:
                a = g.uniform(-1.0, 1.0)
                b = g.uniform(0.1, 1.0)
                re[2 * j: 2 * j + 2] = a
                im[2 * j], im[2 * j + 1] = b, -b
    elif kind == "disk2":
        j = 0
        while j < npairs:
            a, b = g.uniform(-2.0, 2.0), g.uniform(0.0, 2.0)
            if a * a + b * b <= 4.0 and b > 0.0:
                re[2 * j: 2 * j + 2] = a
                im[2 * j], im[2 * j + 1] = b, -b
                j += 1
    elif kind == "ring68":
        # conjugate pairs on the annulus 6 <= |lambda| <= 8, upper half plane (angle U(0, pi)):
        # well outside the spectrum of the configs[2..4] matrices (spectral radius ~4), so no
        # subdiagonal converges during the sweep and the reflectors stay well conditioned -- the
        # full-size parity case whose rounding floor sits far below 1e-10 (R14)
        for j in range(npairs):
            r, t = g.uniform(6.0, 8.0), g.uniform(0.0, np.pi)
            b = r * np.sin(t)
            if b <= 0.0:
                b = 1e-3 * r
            re[2 * j: 2 * j + 2] = r * np.cos(t)
            im[2 * j], im[2 * j + 1] = b, -b
    elif kind.startswith("disk"):
        # "disk<R>": conjugate pairs uniform on the upper half disk of radius R (rejection), e.g.
        # hess_n shifts drawn from the region its spectrum fills (radius sqrt(n), Ginibre-like)
        R = float(kind[4:])
        j = 0
        while j < npairs:
            a, b = g.uniform(-R, R), g.uniform(0.0, R)
            if a * a + b * b <= R * R and b > 0.0:
                re[2 * j: 2 * j + 2] = a
                im[2 * j], im[2 * j + 1] = b, -b
                j += 1
    else:
        raise ValueError(kind)
    return re, im


@dataclass
class Problem:
    H: np.ndarray
    Z: np.ndarray | None
    ilo: int
    ihi: int
    shifts_re: np.ndarray
    shifts_im: np.ndarray
    window: int | None
    blocks: list  # [(ilo, ihi, shift slice start, shift count)]


def make(cfg_idx: int, z_device: str = "cpu", n_override: int | None = None,
         shift_kind: str | None = None) -> Problem:
    """Materialise BASELINE.json configs[cfg_idx] (optionally at a smaller n for tests, or with
    another shift distribution: shift_kind, e.g. "ring68")."""
    c = CONFIGS[cfg_idx]
    n = n_override or c.n
    H = hessenberg(n, c.upper, c.idx, blocks=c.blocks)
    Z = np.asfortranarray(np.eye(n)) if c.z0 == "eye" else orthogonal(n, c.idx, z_device)
    if c.blocks == 1:
        re, im = shifts(shift_kind or c.shifts, c.nshifts, c.idx)
        return Problem(H, Z, 0, n - 1, re, im, c.window, [(0, n - 1, 0, c.nshifts)])
    bs = n // c.blocks
    res, ims, blocks = [], [], []
    for b in range(c.blocks):
        re, im = shifts(c.shifts, c.nshifts, c.idx, stream_offset=b)
        res.append(re)
        ims.append(im)
        blocks.append((b * bs, b * bs + bs - 1, b * c.nshifts, c.nshifts))
    return Problem(H, Z, 0, n - 1, np.concatenate(res), np.concatenate(ims), c.window, blocks)


def config4_block(b: int, H: np.ndarray | None = None, shift_kind: str | None = None):
    """Diagonal block b of BASELINE configs[4] as a problem of its own: (H_bb copy, shifts_re,
    shifts_im, (lo, hi)).  The blocks are decoupled, so one sweep of the whole matrix acts on H_bb
    exactly as a sweep of H_bb alone with Z = I (Z(:, block) = its factor).  H: the full configs[4]
    matrix if already materialised (else it is generated); shift_kind: another shift distribution
    (e.g. "ring68") for every block."""
    c = CONFIGS[4]
    if H is None:
        H = hessenberg(c.n, c.upper, c.idx, blocks=c.blocks)
    bs = c.n // c.blocks
    lo, hi = b * bs, b * bs + bs - 1
    re, im = shifts(shift_kind or c.shifts, c.nshifts, c.idx, stream_offset=b)
    return np.asfortranarray(H[lo:hi + 1, lo:hi + 1]), re, im, (lo, hi)


HESS_CFG = 5  # seed-space id of the hess_n workload


def make_hess(n: int, nshifts: int, z0: str = "eye", z_device: str = "cpu") -> Problem:
    """hess_n: N(0,1) upper entries, sqrt(chi^2(n-i)) subdiagonal; shifts =
    conjugate pairs uniform on the upper half disk of radius sqrt(n) (the region a Ginibre-like
    spectrum fills: the shifts an AED window would return lie there); one sweep ilo=0, ihi=n-1."""
    H = hessenberg(n, "n01", HESS_CFG, subdiag="chi2")
    Z = np.asfortranarray(np.eye(n)) if z0 == "eye" else orthogonal(n, HESS_CFG, z_device)
    re, im = shifts("disk%.6g" % np.sqrt(n), nshifts, HESS_CFG)
    return Problem(H, Z, 0, n - 1, re, im, None, [(0, n - 1, 0, nshifts)])


QZ_CFG = 6  # seed-space id of the generalized (QZ) workload


def triangular(n: int, cfg: int) -> np.ndarray:
    """Random upper-triangular T (Fortran order) for the QZ workload: diagonal U[1, 2], strictly
    upper entries N(0, 1/n) drawn column by column (stream 4) -- nonsingular and well conditioned,
    so the pair has finite generalized eigenvalues near those of H (no infinite eigenvalues: the
    paper's push-infinities task, is out of scope)."""
    T = np.zeros((n, n), dtype=np.float64, order="F")
    g = rng(cfg, 4)
    for j in range(n):
        T[:j, j] = g.standard_normal(j) / np.sqrt(n)
    T[np.arange(n), np.arange(n)] = rng(cfg, 5).uniform(1.0, 2.0, n)
    return T


@dataclass
class QZProblem:
    H: np.ndarray
    T: np.ndarray
    Q: np.ndarray
    Z: np.ndarray
    ilo: int
    ihi: int
    shifts_re: np.ndarray
    shifts_im: np.ndarray


def make_qz(n: int, nshifts: int, q0: str = "eye", seed: int = 0, upper: str = "n01",
            shift_kind: str = "disk2") -> QZProblem:
    """Hessenberg-triangular pair (H as BASELINE configs[2..4]: N(0,1) upper, U[0.5,1.5]
    subdiagonal; T = triangular()), Q0 = Z0 = I or random orthogonal, conjugate-pair shifts."""
    cfg = QZ_CFG * 1000 + seed
    H = hessenberg(n, upper, cfg)
    T = triangular(n, cfg)
    if q0 == "eye":
        Q = np.asfortranarray(np.eye(n))
        Z = np.asfortranarray(np.eye(n))
    else:
        Q = orthogonal(n, cfg)
        Z = orthogonal(n, cfg + 500)
    re, im = shifts(shift_kind, nshifts, cfg)
    return QZProblem(H, T, Q, Z, 0, n - 1, re, im)


def random_case(seed: int, n: int, nshifts: int, ilo: int = 0, ihi: int | None = None,
                upper: str = "n01", z0: str = "eye", shift_kind: str = "mixed"):
    """Small random case for property tests: H decoupled at ilo/ihi, Z0 identity or orthogonal."""
    ihi = n - 1 if ihi is None else ihi
    H = hessenberg(n, upper, 1000 + seed)
    if ilo > 0:
        H[ilo, ilo - 1] = 0.0
    if ihi < n - 1:
        H[ihi + 1, ihi] = 0.0
    if z0 == "eye":
        Z = np.asfortranarray(np.eye(n))
    else:
        Z = orthogonal(n, 1000 + seed)
    re, im = shifts(shift_kind, nshifts, 1000 + seed)
    return H, Z, re, im
