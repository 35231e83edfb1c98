"""CPU tests of the product library without a GPU: the C ABI loads and exports every symbol
include/hqr.h declares, argument validation returns the documented codes, the wavefront planner's
invariants hold, and the planned schedule (emulated in numpy) reproduces the oracle."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
import paper_2007_03576_b200 as hq
from hqr_inputs import random_case, make
from schedule_emulator import emulate

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "hqr.h")).read()
    names = set(re.findall(r"^\s*(?:int|const char\*)\s+(hqr_\w+)\s*\(", hdr, re.M))
    assert names == set(hq.SYMBOLS)
    L = ctypes.CDLL(hq.lib()._name)
    for s in names:
        assert hasattr(L, s), s


def _call(n=16, ilo=0, ihi=15, ns=4, window=8, sr=None, si=None, H=True):
    sr = np.array([0.1, 0.2, 0.3, 0.3] if sr is None else sr, dtype=np.float64)
    si = np.array([0.0, 0.0, 0.5, -0.5] if si is None else si, dtype=np.float64)
    Hm = np.asfortranarray(np.eye(max(n, 1)))
    return hq.sweep_raw(Hm.ctypes.data if H else None, None, n, ilo, ihi, sr.ctypes.data,
                        si.ctypes.data, ns, window)


@pytest.mark.parametrize("kw,code", [
    (dict(H=False), -1), (dict(n=0), -3), (dict(ilo=-1), -4), (dict(ilo=5, ihi=4), -4),
    (dict(ihi=16), -5), (dict(ilo=3, ihi=4), -5), (dict(ns=3), -8), (dict(ns=0), -8),
    (dict(ns=4, n=16, ilo=0, ihi=2), -8), (dict(sr=[np.nan, 0.2, 0.3, 0.3]), -6),
    (dict(si=[0.0, 0.0, 0.5, 0.5]), -7), (dict(si=[0.1, 0.0, 0.5, -0.5]), -7),
    (dict(sr=[0.1, 0.2, 0.3, 0.31]), -7), (dict(window=0), -9), (dict(window=7), -9),
])
def test_invalid_arguments_exact_codes(kw, code):
    assert _call(**kw) == code


def test_not_set_up_code():
    hq.lib().hqr_teardown()
    assert _call() == -100


def test_error_strings():
    L = hq.lib()
    for c in (0, -1, -3, -4, -5, -6, -7, -8, -9, -10, -100, -101, 1002, 2001):
        assert L.hqr_error_string(c)


@pytest.mark.parametrize("n,ns,ilo,ihi,win", [
    (256, 8, 0, 255, 24), (20000, 512, 0, 19999, 96), (10000, 256, 0, 9999, 112),
    (4000, 100, 0, 3999, 151), (300, 20, 40, 259, 24), (9, 8, 0, 8, 8), (200, 60, 10, 190, 8),
    (5000, 1000, 100, 4899, 64),
])
def test_plan_invariants(n, ns, ilo, ihi, win):
    info, W = hq.plan_query(n, ilo, ihi, ns, win)
    N = ihi - ilo + 1
    k = info["k"]
    assert k == min(win, N, hq.MAX_WINDOW)
    nb = ns // 2
    # chains partition the bulges (remainders on the earliest chains), <= (k-2)/6 each
    # and <= 13 (the fused kernel's chase runs one warp per bulge, R5)
    chains = {}
    for w in W:
        chains.setdefault(int(w[1]), (int(w[6]), int(w[7])))
    b = 0
    for c in sorted(chains):
        b0, nbc = chains[c]
        assert b0 == b and (N <= k or nbc <= min((k - 2) // 6, 13))
        b += nbc
    if N > k:  # as few chains as the cap allows
        assert len(chains) == -(-nb // min((k - 2) // 6, 13))
    assert b == nb
    sizes = [chains[c][1] for c in sorted(chains)]
    assert sizes == sorted(sizes, reverse=True) and max(sizes) - min(sizes) <= 1
    for step in range(info["nsteps"]):
        sw = W[W[:, 0] == step]
        assert len(sw) >= 1
        # windows of a step are disjoint and listed top (highest chain) first
        for a_, b_ in zip(sw[:-1], sw[1:]):
            assert a_[3] < b_[2] and a_[1] > b_[1]
    for c in chains:
        cw = W[W[:, 1] == c]
        steps = cw[:, 0]
        assert np.all(np.diff(steps) == 1)                       # one window per step
        assert cw[0, 2] == ilo and cw[-1, 3] == ihi and cw[-1, 9] == 1
        assert np.all(cw[:, 3] - cw[:, 2] + 1 <= k)
        assert np.all(cw[1:, 4] == cw[:-1, 5] + 1)               # chain-local steps contiguous
        nbc = cw[0, 7]
        for w in cw:
            for t in (w[4], w[5]):
                for jj in range(nbc):
                    p = ilo - 1 + t - 3 * jj
                    if ilo - 1 <= p <= ihi - 2:
                        assert (p >= w[2]) or (p == ilo - 1 and w[2] == ilo)   # column p in window
                        assert min(p + 4, ihi) <= w[3]                          # bulge row inside
        # the top bulge leaves at p = ihi - 2 in the last step
        assert ilo - 1 + cw[-1, 5] - 3 * (nbc - 1) == ihi - 2
    # chain c+1 never overlaps chain c in the same step and starts `lag` steps later
    assert info["lag"] * info["s"] >= k or info["nchains"] == 1


@pytest.mark.parametrize("n,ns,ilo,ihi,win,z0", [
    (256, 8, 0, 255, 24, "eye"), (256, 8, 0, 255, 13, "orth"), (300, 20, 40, 259, 24, "orth"),
    (400, 40, 0, 399, 96, "eye"), (200, 60, 10, 190, 20, "eye"), (150, 100, 0, 149, 40, "orth"),
    (60, 12, 0, 59, 60, "eye"), (9, 8, 0, 8, 8, "eye"), (7, 4, 1, 5, 8, "orth"), (3, 2, 0, 2, 8, "eye"),
    (120, 24, 0, 119, 112, "orth"),
])
def test_schedule_emulation_matches_oracle(n, ns, ilo, ihi, win, z0):
    H0, Z0, re_, im_ = random_case(n + ns + win, n, ns, ilo, ihi, z0=z0)
    Ho, Zo = H0.copy(order="F"), Z0.copy(order="F")
    oracle.sweep(Ho, Zo, ilo, ihi, re_, im_)
    He, Ze = H0.copy(order="F"), Z0.copy(order="F")
    emulate(He, Ze, ilo, ihi, re_, im_, win)
    assert np.linalg.norm(He - Ho) / np.linalg.norm(H0) <= 1e-11
    assert np.linalg.norm(Ze - Zo) <= 1e-11 * np.sqrt(n)
    assert np.all(np.tril(He, -2) == 0.0)
    assert np.array_equal(He[:ilo, :ilo], H0[:ilo, :ilo])
    assert np.array_equal(He[ihi + 1:, ihi + 1:], H0[ihi + 1:, ihi + 1:])


@pytest.mark.parametrize("n,ns,win", [(600, 60, 96), (300, 40, 112), (200, 30, 40), (90, 40, 96)])
def test_window_factor_lower_bandwidth(n, ns, win):
    """update.cu skips Q_W[k][c] for k > c + 2*nbc: every bulge passing a row extends the row's
    support at most 2 columns to the left.  Check it on every window of emulated sweeps."""
    H0, Z0, re_, im_ = random_case(n + ns, n, ns)
    worst = []

    def chk(nbc, Q):
        r, c = np.nonzero(Q)
        worst.append(int((r - c).max()) - 2 * nbc)

    emulate(H0.copy(order="F"), None, 0, n - 1, re_, im_, win, on_window=chk)
    assert worst and max(worst) <= 0


def _blocks_case(n, sizes, ns_each, seed):
    """decoupled blocks of the given sizes covering [0, n)"""
    H0, Z0, _, _ = random_case(seed, n, 2, z0="orth")
    from hqr_inputs import shifts
    blocks, res, ims = [], [], []
    lo = 0
    for b, (sz, ns) in enumerate(zip(sizes, ns_each)):
        hi = lo + sz - 1
        if lo > 0:
            H0[lo, lo - 1] = 0.0
        re_, im_ = shifts("disk2", ns, seed, stream_offset=b + 1)
        blocks.append((lo, hi, ns)); res.append(re_); ims.append(im_)
        lo = hi + 1
    return H0, Z0, blocks, np.concatenate(res), np.concatenate(ims)


@pytest.mark.parametrize("n,sizes,ns_each,win", [
    (400, [100, 100, 100, 100], [16, 16, 16, 16], 24), (300, [150, 150], [40, 20], 48),
    (250, [40, 10, 200], [8, 4, 60], 96), (200, [200], [30], 32),
])
def test_multi_block_emulation_matches_oracle(n, sizes, ns_each, win):
    H0, Z0, blocks, re_, im_ = _blocks_case(n, sizes, ns_each, 7)
    Ho, Zo = H0.copy(order="F"), Z0.copy(order="F")
    off = 0
    for lo, hi, ns in blocks:                      # the oracle sweeps the blocks one after another
        oracle.sweep(Ho, Zo, lo, hi, re_[off:off + ns], im_[off:off + ns])
        off += ns
    He, Ze = H0.copy(order="F"), Z0.copy(order="F")
    info = emulate(He, Ze, 0, n - 1, re_, im_, win, blocks=blocks)
    assert np.linalg.norm(He - Ho) / np.linalg.norm(H0) <= 1e-11
    assert np.linalg.norm(Ze - Zo) <= 1e-11 * np.sqrt(n)
    for lo, hi, _ in blocks[1:]:
        assert He[lo, lo - 1] == 0.0
    # blocks share wavefront steps
    _, W = hq.plan_query_multi(n, blocks, win)
    if len(blocks) > 1:
        steps0 = set(W[W[:, 10] == blocks[0][0], 0])
        steps1 = set(W[W[:, 10] == blocks[1][0], 0])
        assert steps0 & steps1


def test_multi_block_validation():
    n = 100
    sr = np.array([0.1, 0.2] * 4); si = np.zeros(8)
    ilo = np.array([0, 40], dtype=np.int64); ihi = np.array([50, 99], dtype=np.int64)
    ns = np.array([4, 4], dtype=np.int32)
    H = np.asfortranarray(np.eye(n))
    L = hq.lib()
    args = lambda lo, hi: (H.ctypes.data, None, n, 2, lo.ctypes.data, hi.ctypes.data, sr.ctypes.data,
                          si.ctypes.data, ns.ctypes.data, 16)
    assert L.hqr_sweep_multi(*args(ilo, ihi)) == -4            # overlapping blocks
    ilo2 = np.array([60, 0], dtype=np.int64); ihi2 = np.array([99, 50], dtype=np.int64)
    assert L.hqr_sweep_multi(*args(ilo2, ihi2)) == -4          # unsorted
    ilo3 = np.array([0, 51], dtype=np.int64); ihi3 = np.array([50, 99], dtype=np.int64)
    assert L.hqr_sweep_multi(*args(ilo3, ihi3)) == -100        # valid, library not set up


@pytest.mark.parametrize("n,ilo,ihi,sweeps,win", [
    (400, 0, 399, [20, 20, 20], 40), (300, 10, 290, [24, 8, 40], 48), (120, 0, 119, [8, 8], 200),
    (500, 0, 499, [60, 60, 60, 60], 96),
])
def test_sweeps_emulation_matches_oracle(n, ilo, ihi, sweeps, win):
    """NEXT-1: overlapped sweeps (hqr_sweeps' plan) reproduce the oracle applying the sweeps one
    after another; every step's windows stay disjoint and all chains share one stride."""
    from hqr_inputs import shifts
    H0, Z0, _, _ = random_case(n + len(sweeps), n, 2, ilo, ihi, z0="orth")
    sets = [shifts("disk2", ns, 17, stream_offset=i + 1) for i, ns in enumerate(sweeps)]
    Ho, Zo = H0.copy(order="F"), Z0.copy(order="F")
    for re_, im_ in sets:
        oracle.sweep(Ho, Zo, ilo, ihi, re_, im_)
    sr = np.concatenate([r for r, _ in sets]); si = np.concatenate([i for _, i in sets])
    He, Ze = H0.copy(order="F"), Z0.copy(order="F")
    info = emulate(He, Ze, ilo, ihi, sr, si, win, sweeps=sweeps)
    assert np.linalg.norm(He - Ho) / np.linalg.norm(H0) <= 1e-11
    assert np.linalg.norm(Ze - Zo) <= 1e-11 * np.sqrt(n)
    _, W = hq.plan_query_sweeps(n, ilo, ihi, sweeps, win)
    for step in range(info["nsteps"]):
        sw = W[W[:, 0] == step]
        for a_, b_ in zip(sw[:-1], sw[1:]):
            assert a_[3] < b_[2]
    # the sweeps overlap: a later sweep's first window runs while an earlier sweep is still active
    first = {}
    for w in W:
        first.setdefault(int(w[6]), int(w[0]))
    if ihi - ilo + 1 > win:
        last_step_sweep0 = max(int(w[0]) for w in W if int(w[6]) < sweeps[0] // 2)
        b_sweep1 = sweeps[0] // 2
        assert min(int(w[0]) for w in W if int(w[6]) >= b_sweep1) < last_step_sweep0
