"""GPU parity: the CUDA sweep (through the C ABI) against the CPU oracle on the same seeded inputs.

Tolerance (BASELINE.json north_star): ||dH'||_F / ||H||_F <= 1e-10 and ||dZ||_F <= 1e-10 sqrt(n).
Integer / structural results are exact: entries below the subdiagonal are exactly 0.0, and blocks
outside the active window that the sweep must not touch are bitwise unchanged.
"""
import numpy as np
import pytest

import oracle
import paper_2007_03576_b200 as hq
from hqr_inputs import make, random_case

pytestmark = pytest.mark.gpu

TOL = 1e-10


@pytest.fixture(scope="module", autouse=True)
def lib_setup():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    hq.setup(0)
    yield
    hq.teardown()


def gpu_sweep(H0, Z0, ilo, ihi, re_, im_, window):
    Hd = hq.to_device(H0)
    Zd = hq.to_device(Z0) if Z0 is not None else None
    hq.sweep(Hd, Zd, ilo, ihi, re_, im_, window)
    return hq.from_device(Hd), (hq.from_device(Zd) if Zd is not None else None)


def oracle_sweep(H0, Z0, ilo, ihi, re_, im_):
    H, Z = H0.copy(order="F"), (Z0.copy(order="F") if Z0 is not None else None)
    oracle.sweep(H, Z, ilo, ihi, re_, im_)
    return H, Z


def check(Hg, Zg, Ho, Zo, H0, ilo, ihi, tol=TOL):
    n = H0.shape[0]
    dh = np.linalg.norm(Hg - Ho) / np.linalg.norm(H0)
    assert dh <= tol, dh
    if Zo is not None:
        dz = np.linalg.norm(Zg - Zo) / np.sqrt(n)
        assert dz <= tol, dz
    assert np.all(np.tril(Hg, -2) == 0.0)
    assert np.array_equal(Hg[:ilo, :ilo], H0[:ilo, :ilo])
    assert np.array_equal(Hg[ihi + 1:, ihi + 1:], H0[ihi + 1:, ihi + 1:])
    assert np.array_equal(Hg[ilo:ihi + 1, :ilo], H0[ilo:ihi + 1, :ilo])
    if ilo > 0:
        assert Hg[ilo, ilo - 1] == 0.0
    if ihi < n - 1:
        assert Hg[ihi + 1, ihi] == 0.0


def test_config0_full_parity():
    p = make(0)
    Hg, Zg = gpu_sweep(p.H, p.Z, p.ilo, p.ihi, p.shifts_re, p.shifts_im, p.window)
    Ho, Zo = oracle_sweep(p.H, p.Z, p.ilo, p.ihi, p.shifts_re, p.shifts_im)
    check(Hg, Zg, Ho, Zo, p.H, p.ilo, p.ihi)


CASES = [
    # (seed, n, nshifts, ilo, ihi, window, z0)
    (0, 3, 2, 0, 2, 8, "eye"), (1, 4, 2, 0, 3, 8, "orth"), (2, 6, 4, 0, 5, 24, "eye"),
    (3, 9, 8, 0, 8, 8, "eye"), (4, 17, 6, 2, 15, 8, "orth"), (5, 40, 8, 0, 39, 16, "eye"),
    (6, 64, 12, 0, 63, 32, "orth"), (7, 100, 20, 5, 90, 24, "eye"), (8, 129, 30, 0, 128, 40, "orth"),
    (9, 200, 60, 10, 190, 20, "eye"), (10, 257, 16, 0, 256, 96, "orth"), (11, 300, 40, 40, 259, 64, "eye"),
    (12, 333, 50, 0, 332, 112, "orth"), (13, 400, 80, 0, 399, 96, "eye"), (14, 150, 100, 0, 149, 40, "eye"),
    (15, 120, 24, 0, 119, 112, "orth"), (16, 511, 64, 100, 400, 48, "eye"), (17, 97, 2, 0, 96, 9, "eye"),
    (18, 250, 248, 0, 249, 112, "eye"), (19, 401, 30, 1, 399, 100, "orth"),
    # many chains over many wavefront steps: the next step's chases wait only for the near tiles of
    # the windows meeting them, so chain-to-chain interactions matter here
    (20, 1500, 200, 0, 1499, 48, "orth"), (21, 2000, 300, 7, 1990, 96, "eye"),
]


@pytest.mark.parametrize("case", CASES, ids=[f"n{c[1]}s{c[2]}w{c[5]}" for c in CASES])
def test_random_parity(case):
    seed, n, ns, ilo, ihi, win, z0 = case
    H0, Z0, re_, im_ = random_case(seed, n, ns, ilo, ihi, z0=z0, shift_kind="mixed" if seed % 2 else "disk2")
    Hg, Zg = gpu_sweep(H0, Z0, ilo, ihi, re_, im_, win)
    Ho, Zo = oracle_sweep(H0, Z0, ilo, ihi, re_, im_)
    check(Hg, Zg, Ho, Zo, H0, ilo, ihi)


def test_no_z_and_host_pointer_path():
    H0, Z0, re_, im_ = random_case(50, 180, 20, 3, 170, z0="orth")
    Hg, _ = gpu_sweep(H0, None, 3, 170, re_, im_, 32)
    Hg2, Zg2 = gpu_sweep(H0, Z0, 3, 170, re_, im_, 32)
    assert np.array_equal(Hg, Hg2)               # Z does not influence H
    Hh, Zh = H0.copy(order="F"), Z0.copy(order="F")
    hq.sweep(Hh, Zh, 3, 170, re_, im_, 32)         # host buffers: staged through the library
    assert np.array_equal(Hh, Hg2) and np.array_equal(Zh, Zg2)
    st = hq.stats()
    assert st["h2d_bytes"] == 2 * 180 * 180 * 8 and st["d2h_bytes"] == 2 * 180 * 180 * 8


@pytest.mark.parametrize("mode", ["both_host", "h_host", "z_host"])
def test_host_buffers_overlapped_copies(mode):
    """Host H / Z: the copies run in column chunks overlapped with the steps (IoPlan in
    hqr_api.cu); several chunks and an interior active block.  Bitwise equal to device buffers."""
    n, ilo, ihi = 2400, 37, 2290
    H0, Z0, re_, im_ = random_case(53, n, 64, ilo, ihi, z0="orth")
    Hg, Zg = gpu_sweep(H0, Z0, ilo, ihi, re_, im_, 96)
    Hh, Zh = H0.copy(order="F"), Z0.copy(order="F")
    Hd, Zd = hq.to_device(H0), hq.to_device(Z0)
    if mode == "both_host":
        hq.sweep(Hh, Zh, ilo, ihi, re_, im_, 96)
        Hr, Zr = Hh, Zh
    elif mode == "h_host":
        hq.sweep(Hh, Zd, ilo, ihi, re_, im_, 96)
        Hr, Zr = Hh, hq.from_device(Zd)
    else:
        hq.sweep(Hd, Zh, ilo, ihi, re_, im_, 96)
        Hr, Zr = hq.from_device(Hd), Zh
    assert np.array_equal(Hr, Hg) and np.array_equal(Zr, Zg)
    st = hq.stats()
    nb = n * n * 8
    # H goes up by row chunks of 512, each from column c - 1 on (the Hessenberg part); Z whole
    h_up = sum(min(512, n - c) * (n - max(c - 1, 0)) * 8 for c in range(0, n, 512))
    assert st["h2d_bytes"] == (h_up if mode != "z_host" else 0) + (nb if mode != "h_host" else 0)
    # Z comes back whole; of H only the rows the sweep can change (rows <= c + 1 of column c: the
    # rest of a Hessenberg matrix is zero in and out), about half
    z_back = nb if mode != "h_host" else 0
    h_back = st["d2h_bytes"] - z_back
    if mode == "z_host":
        assert h_back == 0
    else:
        assert 0.45 * nb < h_back <= nb


def _band_units(Q, KP=96):
    """Executed DMMA work units of one window factor, written out from the kernel's contract
    (gemm_tile.cuh consume_tile): 8-column blocks' nonzero row ranges rounded to 4, quarters of
    KP/32 blocks, K segments with their active blocks."""
    kw = Q.shape[0]
    ext = []
    for b in range(KP // 8):
        cols = [c for c in range(8 * b, 8 * b + 8) if c < kw]
        rows = [r for c in cols for r in np.nonzero(Q[:, c])[0]]
        ext.append((min(rows) // 4 * 4, (max(rows) + 4) // 4 * 4) if rows else (KP, 0))
    nb, u = KP // 32, 0
    for q in range(4):
        e = ext[q * nb:(q + 1) * nb]
        cuts = sorted({v for lo, hi in e if hi > lo for v in (lo, hi)})
        for k0, k1 in zip(cuts, cuts[1:]):
            act = [i for i, (lo, hi) in enumerate(e) if lo <= k0 < hi]
            if act:
                u += 8 * (max(act) - min(act) + 1) * (k1 - k0)
    return u


def test_executed_dmma_flops_match_band_model():
    """hqr_stats.flops_dmma (the roofline numerator, recorded by the chase per window) equals the
    executed work rebuilt from the windows' factors Q_W computed independently by the numpy
    schedule emulator (same plan, same reflectors; exact zeros are structural)."""
    import schedule_emulator as em
    n, ns = 600, 60
    H0, Z0, re_, im_ = random_case(61, n, ns, z0="orth", shift_kind="disk2")
    gpu_sweep(H0, Z0, 0, n - 1, re_, im_, 96)
    got = hq.stats()["flops_dmma"]
    info, wins = hq.plan_query(n, 0, n - 1, ns, 96)
    units = []
    em.emulate(H0.copy(), None, 0, n - 1, re_, im_, 96, on_window=lambda nbc, Q: units.append(_band_units(Q)))
    assert len(units) == len(wins)
    want = sum(2.0 * u * ((n - 1 - int(w[3])) + int(w[2]) + n) for u, w in zip(units, wins))
    assert abs(got - want) <= 1e-12 * want, (got, want)
    dense = sum(2.0 * (int(w[3]) - int(w[2]) + 1) ** 2 * ((n - 1 - int(w[3])) + int(w[2]) + n) for w in wins)
    assert 0.5 * dense < got < dense


def test_graph_and_direct_launch_bitwise_equal():
    H0, Z0, re_, im_ = random_case(51, 300, 32, 0, 299, z0="orth")
    Hg, Zg = gpu_sweep(H0, Z0, 0, 299, re_, im_, 64)
    hq.teardown()
    hq.setup(0, flags=hq.FLAG_NO_GRAPH)
    try:
        Hd, Zd = gpu_sweep(H0, Z0, 0, 299, re_, im_, 64)
    finally:
        hq.teardown()
        hq.setup(0)
    assert np.array_equal(Hg, Hd) and np.array_equal(Zg, Zd)


def test_decoupling_error_code():
    H0, Z0, re_, im_ = random_case(52, 50, 4, 0, 49)
    Hd = hq.to_device(H0)
    with pytest.raises(hq.HQRError) as e:
        hq.sweep(Hd, None, 10, 49, re_, im_, 16)      # H[10, 9] != 0
    assert e.value.code == -10
    with pytest.raises(hq.HQRError) as e:
        hq.sweep(Hd, None, 0, 30, re_, im_, 16)       # H[31, 30] != 0
    assert e.value.code == -10


def test_repeat_determinism():
    H0, Z0, re_, im_ = random_case(53, 400, 40, 0, 399, z0="orth")
    a = gpu_sweep(H0, Z0, 0, 399, re_, im_, 96)
    b = gpu_sweep(H0, Z0, 0, 399, re_, im_, 96)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_config1_full_parity():
    p = make(1)
    Hg, Zg = gpu_sweep(p.H, p.Z, p.ilo, p.ihi, p.shifts_re, p.shifts_im, p.window)
    Ho, Zo = oracle_sweep(p.H, p.Z, p.ilo, p.ihi, p.shifts_re, p.shifts_im)
    check(Hg, Zg, Ho, Zo, p.H, p.ilo, p.ihi)


def _multi_case(n, sizes, ns_each, seed):
    from hqr_inputs import shifts
    H0, Z0, _, _ = random_case(seed, n, 2, z0="orth")
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
    (400, [100, 100, 100, 100], [16, 16, 16, 16], 24), (1000, [250] * 4, [40] * 4, 96),
    (601, [300, 301], [40, 30], 64), (250, [40, 10, 200], [8, 4, 60], 96),
])
def test_multi_block_parity(n, sizes, ns_each, win):
    """BASELINE configs[4] in miniature: several decoupled blocks swept concurrently."""
    H0, Z0, blocks, re_, im_ = _multi_case(n, sizes, ns_each, 11)
    Hd, Zd = hq.to_device(H0), hq.to_device(Z0)
    hq.sweep_multi(Hd, Zd, blocks, re_, im_, win)
    Hg, Zg = hq.from_device(Hd), hq.from_device(Zd)
    Ho, Zo = H0.copy(order="F"), Z0.copy(order="F")
    off = 0
    for lo, hi, ns in blocks:
        oracle.sweep(Ho, Zo, lo, hi, re_[off:off + ns], im_[off:off + ns])
        off += ns
    check(Hg, Zg, Ho, Zo, H0, 0, n - 1)
    for lo, _, _ in blocks[1:]:
        assert Hg[lo, lo - 1] == 0.0


def _gpu_invariants(Hd, Zd, H0d, Z0d, n):
    """Properties that hold at any size, computed on the GPU (torch matmul is test infrastructure)."""
    import torch
    H, Z, H0, Z0 = Hd.t(), Zd.t(), H0d.t(), Z0d.t()   # row-major views of the transposes
    low = torch.tril(Hd, -2)
    assert int(torch.count_nonzero(low)) == 0
    I = torch.eye(n, dtype=torch.float64, device=Hd.device)
    orth = torch.linalg.norm(Zd.T @ Zd - I).item()
    assert orth <= 1e-13 * n, orth
    sim = (torch.linalg.norm(Zd @ Hd @ Zd.T - Z0d @ H0d @ Z0d.T) / torch.linalg.norm(H0d)).item()
    assert sim <= 1e-13 * n, sim
    return orth, sim


def _record_parity(key, rec):
    """Append one full-size parity record to gpurun_out/parity_r02.json (copied to profiles/)."""
    import json
    import os
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
    os.makedirs(out, exist_ok=True)
    path = os.path.join(out, "parity_r02.json")
    d = json.load(open(path)) if os.path.exists(path) else {}
    d[key] = rec
    with open(path, "w") as f:
        json.dump(d, f, indent=1)


def _floor(key):
    import json
    import os
    floor = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "noise_floor.json")))
    return floor["configs"].get(key)


FULL = [  # (record key, BASELINE config, shift kind override, tolerance rule)
    ("2", 2, None, "1e-10"),
    ("3", 3, None, "R14"),
    ("3:ring68", 3, "ring68", "1e-10"),
]


@pytest.mark.parametrize("key,cfg,kind,rule", FULL, ids=[f[0] for f in FULL])
def test_full_size_parity_against_oracle(key, cfg, kind, rule):
    """BASELINE configs[2] (n = 10000) and configs[3] (n = 20000, 512 shifts) in the bench's launch
    configuration (default window), element by element against the oracle run on the host cores,
    plus the invariants computed on the GPU.  The measured differences and the oracle's own
    two-order noise floor are recorded (gpurun_out/parity_r02.json -> profiles/).

    Tolerance: the north_star's 1e-10, except configs[3] with its own shifts (rule R14):
    there two valid orders of the oracle itself differ by 5.3e-10 (tests/golden/noise_floor.json,
    tools/noise_floor.py, oracle/ only) -- the 512 shifts lie inside the spectrum, a subdiagonal
    converges to 1e-11 during the sweep and bulges crossing it lose accuracy locally -- so there
    the GPU must sit within 1.2 x that floor.  The same matrix with shifts outside the spectrum
    ("3:ring68", floor far below 1e-10) is held at 1e-10."""
    p = make(cfg, z_device="cuda", shift_kind=kind)
    n = p.H.shape[0]
    H0d, Z0d = hq.to_device(p.H), hq.to_device(p.Z)
    Hd = hq.to_device(p.H)
    Zd = hq.to_device(p.Z)
    hq.sweep(Hd, Zd, p.ilo, p.ihi, p.shifts_re, p.shifts_im, hq.DEFAULT_WINDOW)
    orth, sim = _gpu_invariants(Hd, Zd, H0d, Z0d, n)
    Hg, Zg = hq.from_device(Hd), hq.from_device(Zd)
    del Hd, Zd, H0d, Z0d
    Ho, Zo = oracle_sweep(p.H, p.Z, p.ilo, p.ihi, p.shifts_re, p.shifts_im)
    dh = float(np.linalg.norm(Hg - Ho) / np.linalg.norm(p.H))
    dz = float(np.linalg.norm(Zg - Zo) / np.sqrt(n))
    fl = _floor(key)
    floor = max(fl["dH_rel_fro"], fl["dZ_fro_over_sqrt_n"]) if fl else None
    tol = TOL if rule == "1e-10" else max(TOL, 1.2 * floor)
    _record_parity(key, {"n": n, "nshifts": len(p.shifts_re), "window": hq.DEFAULT_WINDOW,
                         "dH_rel_fro": dh, "dZ_fro_over_sqrt_n": dz, "dH_max": float(np.abs(Hg - Ho).max()),
                         "oracle_floor": fl, "tolerance": tol, "rule": rule,
                         "orth_ZtZ_minus_I": orth, "similarity_rel": sim,
                         "min_abs_subdiag_gpu": float(np.abs(np.diag(Hg, -1)).min())})
    check(Hg, Zg, Ho, Zo, p.H, p.ilo, p.ihi, tol=tol)


FULL4 = [  # (record key, shift kind override, tolerance rule)
    ("4:b2", None, "R14"),
    ("4:b2:ring68", "ring68", "1e-10"),
]


@pytest.mark.parametrize("key,kind,rule", FULL4, ids=[f[0] for f in FULL4])
def test_config4_full_size_block_against_oracle(key, kind, rule):
    """BASELINE configs[4] at full size (n = 40000, four decoupled 10000 blocks, 512 shifts each) swept
    together in the bench's launch configuration (hqr_sweep_multi, default window).  The blocks are
    decoupled, so H(b, b) and Z(b, b) after the sweep equal a sweep of H0(b, b) alone with Z = I:
    block 2 is compared element by element with the oracle doing exactly that (the other three
    blocks would cost another ~10 min of oracle time; they share every code path).  For all blocks,
    properties that hold at any size, on the GPU: Z is zero outside its diagonal blocks and each
    Q_b = Z(b, b) is orthogonal, H is zero below the subdiagonal and at the decoupling entries, and
    every block above the diagonal is H(b, c) = Q_b^T H0(b, c) Q_c (the left / right updates agree
    with the accumulated factors).

    Tolerance: with the config's own shifts (inside the spectrum; a subdiagonal of block 2 converges
    to 2e-14 during the sweep) the oracle in its two valid reflector orders differs by 5.0e-10
    (tests/golden/noise_floor.json "4:b2"); the GPU is a third valid order, so it is held to twice
    that floor (rule R14); with HQR_PARITY_BOTH_ORDERS set its distance to the oracle's other order
    is recorded too (profiles/parity_r02.json: 1.04e-9).  The same blocks with
    shifts outside the spectrum ("ring68") are held at the north_star's 1e-10."""
    import os

    import torch
    from hqr_inputs import CONFIGS, config4_block, hessenberg, shifts

    c = CONFIGS[4]
    n, nb, bs = c.n, c.blocks, c.n // c.blocks
    H0 = hessenberg(n, c.upper, c.idx, blocks=nb)
    sr, si, blocks = [], [], []
    for b in range(nb):
        re_, im_ = shifts(kind or c.shifts, c.nshifts, c.idx, stream_offset=b)
        sr.append(re_)
        si.append(im_)
        blocks.append((b * bs, b * bs + bs - 1, c.nshifts))
    H0d = hq.to_device(H0)
    Hd = hq.to_device(H0)
    Zd = torch.eye(n, dtype=torch.float64, device="cuda").t()  # column-major view of I
    hq.sweep_multi(Hd, Zd, blocks, np.concatenate(sr), np.concatenate(si), hq.DEFAULT_WINDOW)
    torch.cuda.synchronize()
    # structure: below the subdiagonal, decoupling entries, Z outside the diagonal blocks
    for b in range(nb):
        lo = b * bs
        cols = Hd[:, lo:lo + bs]
        assert int(torch.count_nonzero(torch.tril(cols, -2 - lo))) == 0
        if b > 0:
            assert Hd[lo, lo - 1].item() == 0.0
        zc = Zd[:, lo:lo + bs]
        assert int(torch.count_nonzero(zc[:lo])) == 0 and int(torch.count_nonzero(zc[lo + bs:])) == 0
    Q = [Zd[b * bs:(b + 1) * bs, b * bs:(b + 1) * bs] for b in range(nb)]
    I = torch.eye(bs, dtype=torch.float64, device="cuda")
    orth = [torch.linalg.norm(q.T @ q - I).item() for q in Q]
    assert max(orth) <= 1e-13 * bs, orth
    offd = {}
    for b in range(nb):
        for cc in range(b + 1, nb):
            rb, rc = slice(b * bs, (b + 1) * bs), slice(cc * bs, (cc + 1) * bs)
            ref = Q[b].T @ H0d[rb, rc] @ Q[cc]
            offd[f"{b}{cc}"] = (torch.linalg.norm(Hd[rb, rc] - ref) / torch.linalg.norm(H0d[rb, rc])).item()
    assert max(offd.values()) <= TOL, offd
    # block 2 against the oracle
    b = 2
    lo = b * bs
    Hg = hq.from_device(Hd[lo:lo + bs, lo:lo + bs])
    Zg = hq.from_device(Zd[lo:lo + bs, lo:lo + bs])
    del Hd, Zd, H0d, Q
    torch.cuda.empty_cache()
    Hb, re_, im_, _ = config4_block(b, H0, shift_kind=kind)
    del H0
    Ho, Zo = oracle_sweep(Hb, np.asfortranarray(np.eye(bs)), 0, bs - 1, re_, im_)
    dh = float(np.linalg.norm(Hg - Ho) / np.linalg.norm(Hb))
    dz = float(np.linalg.norm(Zg - Zo) / np.sqrt(bs))
    rec = {"n": n, "block": [lo, lo + bs - 1], "nshifts_per_block": c.nshifts, "window": hq.DEFAULT_WINDOW,
           "dH_rel_fro": dh, "dZ_fro_over_sqrt_n": dz, "dH_max": float(np.abs(Hg - Ho).max()),
           "orth_QtQ_minus_I": orth, "offdiag_rel": offd, "rule": rule}
    if rule == "R14":
        fl = _floor(key)
        rec["oracle_floor"] = fl
        tol = max(TOL, 2.0 * max(fl["dH_rel_fro"], fl["dZ_fro_over_sqrt_n"]))
        if os.environ.get("HQR_PARITY_BOTH_ORDERS"):  # evidence run (profiles/parity_r02.json): ~2.5 min more
            Hp, Zp = Hb.copy(order="F"), np.asfortranarray(np.eye(bs))
            oracle.sweep(Hp, Zp, 0, bs - 1, re_, im_, order="pipelined")  # the other valid order
            rec["vs_pipelined_oracle"] = {"dH_rel_fro": float(np.linalg.norm(Hg - Hp) / np.linalg.norm(Hb)),
                                          "dZ_fro_over_sqrt_n": float(np.linalg.norm(Zg - Zp) / np.sqrt(bs))}
    else:
        tol = TOL
    rec["tolerance"] = tol
    _record_parity(key, rec)
    check(Hg, Zg, Ho, Zo, Hb, 0, bs - 1, tol=tol)


@pytest.mark.parametrize("vworld,case", [(1, (60, 1000, 40, 96)), (2, (61, 1200, 60, 64)),
                                         (4, (62, 2000, 80, 96)), (8, (63, 2400, 64, 96)),
                                         (3, (64, 1501, 30, 40))])
def test_sharded_virtual_ranks(vworld, case):
    """The multi-GPU algorithm (H column shards with lent slabs, Z row shards, per-rank kernels) with
    vworld virtual ranks on this GPU (hqr_sweep_virtual) against the oracle."""
    seed, n, ns, win = case
    H0, Z0, re_, im_ = random_case(seed, n, ns, z0="orth", shift_kind="disk2")
    Hd, Zd = hq.to_device(H0), hq.to_device(Z0)
    hq.sweep_virtual(Hd, Zd, 0, n - 1, re_, im_, win, vworld)
    Hg, Zg = hq.from_device(Hd), hq.from_device(Zd)
    Ho, Zo = oracle_sweep(H0, Z0, 0, n - 1, re_, im_)
    check(Hg, Zg, Ho, Zo, H0, 0, n - 1)


@pytest.mark.parametrize("vworld,sizes,ns_each,win", [(2, [600, 600], [40, 40], 96),
                                                      (4, [1000, 1000, 1000, 1000], [60, 60, 60, 60], 96),
                                                      (8, [1500, 1500], [80, 60], 64)])
def test_sharded_virtual_multi_block(vworld, sizes, ns_each, win):
    """BASELINE configs[4] in miniature on the sharded path: several decoupled blocks, every
    block's windows sharing the steps and the shard roles (hqr_sweep_virtual_multi)."""
    n = sum(sizes)
    H0, Z0, blocks, re_, im_ = _multi_case(n, sizes, ns_each, 13)
    Hd, Zd = hq.to_device(H0), hq.to_device(Z0)
    hq.sweep_virtual_multi(Hd, Zd, blocks, re_, im_, win, vworld)
    Hg, Zg = hq.from_device(Hd), hq.from_device(Zd)
    Ho, Zo = H0.copy(order="F"), Z0.copy(order="F")
    off = 0
    for lo, hi, ns in blocks:
        oracle.sweep(Ho, Zo, lo, hi, re_[off:off + ns], im_[off:off + ns])
        off += ns
    check(Hg, Zg, Ho, Zo, H0, 0, n - 1)


def test_sharded_nccl_transport_one_rank():
    """hqr_sweep_dist with its NCCL transport executed (HQR_FLAG_NCCL_SELF: a one-rank communicator
    on this GPU): the grouped ncclBroadcast of every step's factors on the comm stream, the event
    gating of the two compute streams -- against the oracle, on the local shard (= the matrix)."""
    import torch
    n, ns, win = 1200, 80, 96
    H0, Z0, re_, im_ = random_case(66, n, ns, z0="orth", shift_kind="disk2")
    cb, rb, halo = hq.dist_layout(n, 1)
    hq.teardown()
    hq.setup(0, flags=hq.FLAG_NCCL_SELF)
    try:
        Hl = torch.zeros((n + halo, n), dtype=torch.float64, device="cuda")   # rows = local columns
        Hl[:n].copy_(torch.from_numpy(np.ascontiguousarray(H0.T)))
        Zl = torch.from_numpy(np.ascontiguousarray(Z0.T)).cuda()
        hq.sweep_dist(Hl.data_ptr(), Zl.data_ptr(), n, 0, n - 1, re_, im_, win)
        torch.cuda.synchronize()
        Hg = np.asfortranarray(Hl[:n].cpu().numpy().T)
        Zg = np.asfortranarray(Zl.cpu().numpy().T)
    finally:
        hq.teardown()
        hq.setup(0)
    Ho, Zo = oracle_sweep(H0, Z0, 0, n - 1, re_, im_)
    check(Hg, Zg, Ho, Zo, H0, 0, n - 1)


def test_sharded_virtual_deferred_long_lag():
    """Many chains crossing every boundary of 8 virtual ranks: the deferred far-right / Z work
    (low-priority stream) trails the chases by many steps and is drained at every lend."""
    seed, n, ns, win = 65, 3000, 200, 96
    H0, Z0, re_, im_ = random_case(seed, n, ns, z0="orth", shift_kind="disk2")
    Hd, Zd = hq.to_device(H0), hq.to_device(Z0)
    hq.sweep_virtual(Hd, Zd, 0, n - 1, re_, im_, win, 8)
    Hg, Zg = hq.from_device(Hd), hq.from_device(Zd)
    Ho, Zo = oracle_sweep(H0, Z0, 0, n - 1, re_, im_)
    check(Hg, Zg, Ho, Zo, H0, 0, n - 1)


@pytest.mark.parametrize("case", [(70, 600, 60, 96), (71, 1000, 100, 64), (72, 400, 40, 112)])
def test_fused_step_kernel_matches_separate_launches(case):
    """The fused step kernel (prioritised task queue, chase of step g+1 inside step g's launch) and
    the separate chase / left / right launches compute every element with the same operations in
    the same order: bitwise equal."""
    seed, n, ns, win = case
    H0, Z0, re_, im_ = random_case(seed, n, ns, z0="orth", shift_kind="disk2")
    Hf, Zf = gpu_sweep(H0, Z0, 0, n - 1, re_, im_, win)
    hq.teardown()
    hq.setup(0, flags=hq.FLAG_NO_FUSE)
    try:
        Hs, Zs = gpu_sweep(H0, Z0, 0, n - 1, re_, im_, win)
    finally:
        hq.teardown()
        hq.setup(0)
    assert np.array_equal(Hf, Hs) and np.array_equal(Zf, Zs)


# ------------------------------------------------------------------------------------------------
# round 2: aftermath scan (a9), scaled inputs (R15), degenerate reflectors, hess_n, entry ordering
# ------------------------------------------------------------------------------------------------

@pytest.mark.parametrize("case", [(80, 500, 40, 0, 499, 64), (81, 700, 60, 30, 650, 96),
                                  (82, 60, 8, 5, 50, 112)])
def test_aftermath_scan_bit_exact(case):
    """a9: the flags the last chain's chases compute equal the oracle's scan of the
    GPU's own H' bit for bit (same criterion, same precision), and the scan of the oracle's H'."""
    seed, n, ns, ilo, ihi, win = case
    H0, Z0, re_, im_ = random_case(seed, n, ns, ilo, ihi, z0="orth", shift_kind="disk2")
    Hg, Zg = gpu_sweep(H0, Z0, ilo, ihi, re_, im_, win)
    f = hq.aftermath(n)
    assert np.array_equal(f, oracle.subdiag_scan(Hg, [(ilo, ihi)]))
    Ho, _ = oracle_sweep(H0, Z0, ilo, ihi, re_, im_)
    assert np.array_equal(f, oracle.subdiag_scan(Ho, [(ilo, ihi)]))
    if ilo > 0:
        assert f[ilo - 1] == 2 and np.all(f[:ilo - 1] == -1)
    if ihi < n - 1:
        assert f[ihi] == 2 and np.all(f[ihi + 1:] == -1)


def test_aftermath_multi_block_and_small_entries():
    """Several blocks: the decoupling zeros between them are flagged 2; an entry made negligible
    (but nonzero) in a block that is not swept is left unscanned (-1), one right at a block edge
    is scanned."""
    H0, Z0, blocks, re_, im_ = _multi_case(600, [150, 150, 300], [16, 16, 40], 12)
    Hd, Zd = hq.to_device(H0), hq.to_device(Z0)
    hq.sweep_multi(Hd, Zd, blocks, re_, im_, 48)
    Hg = hq.from_device(Hd)
    f = hq.aftermath(600)
    want = oracle.subdiag_scan(Hg, [(lo, hi) for lo, hi, _ in blocks])
    assert np.array_equal(f, want)
    assert f[149] == 2 and f[299] == 2 and f[599] == -1


@pytest.mark.parametrize("k", [600, -600])
def test_scaled_matrix_parity_and_equivariance(k):
    """R15: H and the shifts times 2^k (|H| ~ 1e180 / 1e-180: the unscaled bulge vector and
    house() would overflow / underflow): finite, equal to 2^k times the unscaled GPU sweep bit for
    bit (every kernel step is linear in H or scale invariant), and within tolerance of the oracle."""
    n, ns, win = 400, 40, 64
    H0, Z0, re_, im_ = random_case(85, n, ns, z0="orth", shift_kind="disk2")
    Hg, Zg = gpu_sweep(H0, Z0, 0, n - 1, re_, im_, win)
    Hs0 = np.asfortranarray(np.ldexp(H0, k))
    Hgs, Zgs = gpu_sweep(Hs0, Z0, 0, n - 1, np.ldexp(re_, k), np.ldexp(im_, k), win)
    assert np.all(np.isfinite(Hgs))
    assert np.array_equal(Hgs, np.ldexp(Hg, k)) and np.array_equal(Zgs, Zg)
    Ho, Zo = oracle_sweep(Hs0, Z0, 0, n - 1, np.ldexp(re_, k), np.ldexp(im_, k))
    # norms of 2^+-600-sized entries over/underflow: compare scaled back (exact)
    check(np.ldexp(Hgs, -k), Zgs, np.ldexp(Ho, -k), Zo, H0, 0, n - 1)


def test_decimal_extreme_scales():
    """|H| ~ 1e200 and 1e-200 (not powers of two): the sweep stays finite and matches the oracle."""
    n, ns = 300, 24
    H0, Z0, re_, im_ = random_case(86, n, ns, z0="orth", shift_kind="disk2")
    for sc in (1e200, 1e-200):
        Hs0 = np.asfortranarray(H0 * sc)
        Hg, Zg = gpu_sweep(Hs0, Z0, 0, n - 1, re_ * sc, im_ * sc, 48)
        Ho, Zo = oracle_sweep(Hs0, Z0, 0, n - 1, re_ * sc, im_ * sc)
        assert np.all(np.isfinite(Hg)) and np.all(np.isfinite(Zg))
        check(Hg / sc, Zg, Ho / sc, Zo, Hs0 / sc, 0, n - 1)   # norms of 1e+-200 entries over/underflow


@pytest.mark.parametrize("n,win", [(40, 16), (300, 64)])
def test_zero_tail_reflectors_identity(n, win):
    """tau = 0 path (R2: zero tail -> identity): with h(ilo+1, ilo) = 0 every bulge vector has a
    zero tail (x1 = h10 (...), x2 = h10 h21) and every later reflector acts on an exactly zero
    column, so the sweep is the identity -- bitwise, on H and Z, as in the oracle."""
    H0, Z0, re_, im_ = random_case(87, n, 8, z0="orth", shift_kind="disk2")
    H0[1, 0] = 0.0
    Hg, Zg = gpu_sweep(H0, Z0, 0, n - 1, re_, im_, win)
    Ho, Zo = oracle_sweep(H0, Z0, 0, n - 1, re_, im_)
    assert np.array_equal(Ho, H0) and np.array_equal(Zo, Z0)
    assert np.array_equal(Hg, H0) and np.array_equal(Zg, Z0)
    assert hq.aftermath(n)[0] == 2


@pytest.mark.parametrize("n,ns,win", [(8, 2, 8), (12, 4, 12), (24, 4, 10), (30, 2, 8)])
def test_perfect_shifts(n, ns, win):
    """Shifts = exact eigenvalues (conjugate pairs exact): the trailing m x m block (m = ns)
    decouples on the GPU as in the oracle (small n only: over long chases the bulges lose the
    shift information -- forward instability -- and the oracle itself decouples only to ~1e-2 at
    n = 150; windows smaller than n make the chase cross windows).  Its internal basis is then fixed only by rounding (the
    last reflectors act on a collapsed bulge), so there the two are compared through invariants --
    the spectrum of the trailing block, the subspace of the last m columns of Z, the row norms of
    the coupling block -- and everything else element by element."""
    H0, Z0, _, _ = random_case(88 + n, n, 2, z0="orth")
    lam = np.linalg.eigvals(H0)   # test infrastructure: the shifts are inputs
    cpx = sorted([z for z in lam if z.imag > 1e-9], key=lambda z: -abs(z))[: ns // 2]
    rl = sorted([z.real for z in lam if abs(z.imag) <= 1e-9], key=lambda x: -abs(x))
    re_, im_ = [], []
    for z in cpx:
        re_ += [z.real, z.real]
        im_ += [abs(z.imag), -abs(z.imag)]
    while len(re_) < ns and len(rl) >= 2:   # not enough conjugate pairs: real pairs
        re_ += [rl.pop(0), rl.pop(0)]
        im_ += [0.0, 0.0]
    assert len(re_) == ns
    re_, im_ = np.array(re_), np.array(im_)
    Hg, Zg = gpu_sweep(H0, Z0, 0, n - 1, re_, im_, win)
    Ho, Zo = oracle_sweep(H0, Z0, 0, n - 1, re_, im_)
    m, hn = ns, np.linalg.norm(H0)
    assert abs(Hg[n - m, n - m - 1]) <= 1e-9 * hn and abs(Ho[n - m, n - m - 1]) <= 1e-9 * hn
    assert np.all(np.tril(Hg, -2) == 0.0)
    k = n - m
    assert np.linalg.norm(Hg[:k, :k] - Ho[:k, :k]) <= TOL * hn
    assert np.linalg.norm(Zg[:, :k] - Zo[:, :k]) <= TOL * np.sqrt(n)
    assert np.allclose(np.linalg.norm(Hg[:k, k:], axis=1), np.linalg.norm(Ho[:k, k:], axis=1),
                       rtol=0, atol=1e-10 * hn)
    Pg, Po = Zg[:, k:] @ Zg[:, k:].T, Zo[:, k:] @ Zo[:, k:].T
    assert np.linalg.norm(Pg - Po) <= 1e-10 * np.sqrt(n)
    eg = np.sort_complex(np.linalg.eigvals(Hg[k:, k:]))
    eo = np.sort_complex(np.linalg.eigvals(Ho[k:, k:]))
    assert np.allclose(eg, eo, rtol=0, atol=1e-9 * hn)
    assert np.allclose(np.sort_complex(re_ + 1j * im_), eg, rtol=0, atol=1e-7 * hn)


@pytest.mark.parametrize("n,ns", [(1000, 100), (4000, 200)])
def test_hess_n_parity(n, ns):
    """NEXT-3 workload hess_n: graded chi^2 subdiagonal, shifts in the disk of
    radius sqrt(n), random orthogonal Z."""
    from hqr_inputs import make_hess
    p = make_hess(n, ns, z0="orth")
    Hg, Zg = gpu_sweep(p.H, p.Z, 0, n - 1, p.shifts_re, p.shifts_im, hq.DEFAULT_WINDOW)
    Ho, Zo = oracle_sweep(p.H, p.Z, 0, n - 1, p.shifts_re, p.shifts_im)
    check(Hg, Zg, Ho, Zo, p.H, 0, n - 1)


def test_entry_waits_for_default_stream():
    """the sweep must see H / Z writes the caller queued on the default stream just
    before the call (the library stream waits for the legacy stream at entry)."""
    import torch
    n = 1200
    H0, Z0, re_, im_ = random_case(89, n, 40, z0="orth", shift_kind="disk2")
    Href, Zref = gpu_sweep(H0, Z0, 0, n - 1, re_, im_, 96)
    src_h, src_z = hq.to_device(H0), hq.to_device(Z0)
    Hd = torch.zeros_like(src_h.t()).t()
    Zd = torch.zeros_like(src_z.t()).t()
    torch.cuda.synchronize()
    torch.cuda._sleep(200_000_000)   # ~0.1 s of queued work ahead of the copies
    Hd.t().copy_(src_h.t())
    Zd.t().copy_(src_z.t())
    hq.sweep(Hd, Zd, 0, n - 1, re_, im_, 96)
    assert np.array_equal(hq.from_device(Hd), Href) and np.array_equal(hq.from_device(Zd), Zref)


def test_window_max_config():
    """hqr_config.window_max caps the effective window (SURVEY §8(b) "max window")."""
    n = 500
    H0, Z0, re_, im_ = random_case(90, n, 40, z0="orth", shift_kind="disk2")
    hq.teardown()
    hq.setup(0, window_max=48)
    try:
        Hg, Zg = gpu_sweep(H0, Z0, 0, n - 1, re_, im_, 96)
        assert hq.stats()["window_eff"] == 48
    finally:
        hq.teardown()
        hq.setup(0)
    Ho, Zo = oracle_sweep(H0, Z0, 0, n - 1, re_, im_)
    check(Hg, Zg, Ho, Zo, H0, 0, n - 1)


@pytest.mark.parametrize("n,ilo,ihi,sweeps,win", [(1500, 0, 1499, [100, 100, 100], 96),
                                                  (900, 20, 880, [40, 16, 64], 64),
                                                  (100, 0, 99, [8, 8], 112)])
def test_overlapped_sweeps_parity(n, ilo, ihi, sweeps, win):
    """NEXT-1: hqr_sweeps equals the oracle applying the sweeps one after another;
    the aftermath scan of the last sweep matches the oracle's scan of the GPU's H'."""
    from hqr_inputs import shifts
    H0, Z0, _, _ = random_case(95, n, 2, ilo, ihi, z0="orth")
    sets = [shifts("disk2", ns, 18, stream_offset=i + 1) for i, ns in enumerate(sweeps)]
    Hd, Zd = hq.to_device(H0), hq.to_device(Z0)
    hq.sweeps(Hd, Zd, ilo, ihi, sets, win)
    Hg, Zg = hq.from_device(Hd), hq.from_device(Zd)
    Ho, Zo = H0.copy(order="F"), Z0.copy(order="F")
    for re_, im_ in sets:
        oracle.sweep(Ho, Zo, ilo, ihi, re_, im_)
    check(Hg, Zg, Ho, Zo, H0, ilo, ihi)
    assert np.array_equal(hq.aftermath(n), oracle.subdiag_scan(Hg, [(ilo, ihi)]))


@pytest.mark.parametrize("n,ns,crit", [(1500, 64, True), (2000, 600, False)])
def test_critical_queue_and_single_queue_parity(n, ns, crit):
    """The persistent launch's two task-claiming modes (DESIGN.md §6 "Critical SMs"): a chase-bound
    sweep serves chases and their near tiles from a dedicated critical queue on 2*nchains+2 CTAs
    (hqr_stats.crit_sms > 0), a GEMM-bound one keeps one queue (0); both match the oracle.  (Shifts
    from a small disk: many shifts near the spectrum converge subdiagonals during the sweep and put
    the oracle's own floor above 1e-10, reading R14.)"""
    H0, Z0, re_, im_ = random_case(93, n, ns, z0="orth", shift_kind="disk2")
    Hg, Zg = gpu_sweep(H0, Z0, 0, n - 1, re_, im_, 96)
    st = hq.stats()
    assert (st["crit_sms"] > 0) == crit, st["crit_sms"]
    Ho, Zo = oracle_sweep(H0, Z0, 0, n - 1, re_, im_)
    check(Hg, Zg, Ho, Zo, H0, 0, n - 1)
