"""paper_2007_03576_b200 -- B200-native multishift QR sweep (thin Python binding over libhqr_b200.so).

Argument marshalling only: every step of the sweep runs in the sm_100a kernels behind the C ABI
declared in ``include/hqr.h`` (hqr_setup / hqr_sweep / hqr_teardown, plus hqr_plan_query and
hqr_get_stats).  There is no CPU fallback: if the shared library or a CUDA device is missing the
calls raise.

Matrices are fp64, n x n, column-major (leading dimension n):
  * device: a ``torch.float64`` CUDA tensor with ``stride() == (1, n)`` (e.g. ``T.t()`` of a
    contiguous tensor T holding the transpose), see :func:`to_device` / :func:`from_device`;
  * host: a numpy float64 Fortran-ordered array (the library stages it; copies are in the call).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import build as _build

_lib = None

ERRORS = {
    -1: "H is NULL / invalid config", -3: "n < 1", -4: "ilo < 0 or ilo > ihi",
    -5: "ihi >= n or active block shorter than 3", -6: "non-finite shift",
    -7: "shift pair not two reals / exact conjugates", -8: "nshifts odd, < 2 or > N",
    -9: "window out of range", -10: "active block not decoupled", -100: "not set up",
    -101: "no usable sm_100 CUDA device", -11: "matrix too small for the shard count",
    -2: "T is NULL or singular at the top of the block (QZ)",
}

FLAG_NO_GRAPH = 1
FLAG_PROFILE = 2
FLAG_NO_FUSE = 4
FLAG_NCCL_SELF = 8
MAX_WINDOW = 112
DEFAULT_WINDOW = 96


class HQRError(RuntimeError):
    def __init__(self, code: int, where: str):
        self.code = code
        msg = ERRORS.get(code) or ("CUDA error %d" % (code - 1000) if 1000 <= code < 2000 else
                                   "NCCL error %d" % (code - 2000) if code >= 2000 else "error")
        super().__init__(f"{where} returned {code}: {msg}")


class _Config(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("rank", ctypes.c_int), ("world", ctypes.c_int),
                ("nccl_id", ctypes.c_void_p), ("n_max", ctypes.c_int64), ("flags", ctypes.c_int),
                ("col_bounds", ctypes.c_void_p), ("row_bounds", ctypes.c_void_p),
                ("window_max", ctypes.c_int)]


class Stats(ctypes.Structure):
    _fields_ = [("kernels_launched", ctypes.c_int64), ("steps", ctypes.c_int64),
                ("windows", ctypes.c_int64), ("flops_update", ctypes.c_double),
                ("flops_chase", ctypes.c_double), ("bytes_update", ctypes.c_double),
                ("ms_chase", ctypes.c_double), ("ms_left", ctypes.c_double),
                ("ms_right", ctypes.c_double), ("ms_step", ctypes.c_double), ("ms_total", ctypes.c_double),
                ("h2d_bytes", ctypes.c_int64), ("d2h_bytes", ctypes.c_int64),
                ("launches_left", ctypes.c_int), ("launches_right", ctypes.c_int),
                ("launches_chase", ctypes.c_int), ("window_eff", ctypes.c_int),
                ("flops_dmma", ctypes.c_double), ("flops_alg", ctypes.c_double),
                ("crit_sms", ctypes.c_int), ("pad_", ctypes.c_int)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


SYMBOLS = ["hqr_setup", "hqr_sweep", "hqr_sweep_multi", "hqr_teardown", "hqr_plan_query",
           "hqr_plan_query_multi", "hqr_get_stats", "hqr_error_string", "hqr_dist_layout",
           "hqr_dist_query", "hqr_nccl_unique_id", "hqr_sweep_dist", "hqr_sweep_virtual",
           "hqr_get_aftermath", "hqr_sweeps", "hqr_plan_query_sweeps", "hqr_qz_sweep", "hqr_qr_iterate",
           "hqr_sweep_dist_multi", "hqr_sweep_virtual_multi", "hqr_aed"]


def lib():
    """Load (building first if stale) libhqr_b200.so.  Raises if it cannot be loaded."""
    global _lib
    if _lib is None:
        path = os.environ.get("HQR_LIB")  # debugging: an alternative build of the same library
        if not path:
            path = _build.LIB
            if not os.path.exists(path) or _build._stale():
                _build.build()
        L = ctypes.CDLL(path)
        L.hqr_setup.argtypes = [ctypes.POINTER(_Config)]
        L.hqr_setup.restype = ctypes.c_int
        L.hqr_sweep.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                ctypes.c_int]
        L.hqr_sweep.restype = ctypes.c_int
        L.hqr_sweep_multi.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        L.hqr_sweep_multi.restype = ctypes.c_int
        L.hqr_plan_query_multi.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
        L.hqr_plan_query_multi.restype = ctypes.c_int
        L.hqr_dist_layout.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.c_void_p]
        L.hqr_dist_layout.restype = ctypes.c_int
        L.hqr_dist_query.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                     ctypes.c_int64]
        L.hqr_dist_query.restype = ctypes.c_int
        L.hqr_nccl_unique_id.argtypes = [ctypes.c_void_p]
        L.hqr_nccl_unique_id.restype = ctypes.c_int
        L.hqr_sweep_dist.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                     ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                     ctypes.c_int]
        L.hqr_sweep_dist.restype = ctypes.c_int
        L.hqr_sweep_virtual.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                        ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.hqr_sweep_virtual.restype = ctypes.c_int
        L.hqr_teardown.argtypes = []
        L.hqr_teardown.restype = ctypes.c_int
        L.hqr_plan_query.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
        L.hqr_plan_query.restype = ctypes.c_int
        L.hqr_sweeps.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                 ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                 ctypes.c_void_p, ctypes.c_int]
        L.hqr_sweeps.restype = ctypes.c_int
        L.hqr_plan_query_sweeps.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                            ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                            ctypes.c_void_p, ctypes.c_int64]
        L.hqr_plan_query_sweeps.restype = ctypes.c_int
        L.hqr_qz_sweep.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int64] * 3 + [
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
        L.hqr_qz_sweep.restype = ctypes.c_int
        L.hqr_qr_iterate.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                     ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.hqr_qr_iterate.restype = ctypes.c_int
        L.hqr_aed.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                              ctypes.c_int, ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                              ctypes.c_void_p]
        L.hqr_aed.restype = ctypes.c_int
        for nm in ("hqr_sweep_dist_multi", "hqr_sweep_virtual_multi"):
            fn = getattr(L, nm)
            fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p,
                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int] + (
                [ctypes.c_int] if nm.endswith("virtual_multi") else [])
            fn.restype = ctypes.c_int
        L.hqr_get_aftermath.argtypes = [ctypes.c_void_p, ctypes.c_int64]
        L.hqr_get_aftermath.restype = ctypes.c_int
        L.hqr_get_stats.argtypes = [ctypes.POINTER(Stats)]
        L.hqr_get_stats.restype = ctypes.c_int
        L.hqr_error_string.argtypes = [ctypes.c_int]
        L.hqr_error_string.restype = ctypes.c_char_p
        _lib = L
    return _lib


def setup(device: int = 0, flags: int = 0, rank: int = 0, world: int = 1, nccl_id: bytes | None = None,
          n_max: int = 0, col_bounds=None, row_bounds=None, window_max: int = 0) -> None:
    buf = None
    cfg = _Config(device, rank, world, None, n_max, flags, None, None, window_max)
    if nccl_id is not None:
        buf = ctypes.create_string_buffer(bytes(nccl_id), len(nccl_id))
        cfg.nccl_id = ctypes.cast(buf, ctypes.c_void_p)
    cbs = rbs = None
    if col_bounds is not None:
        cbs = np.ascontiguousarray(col_bounds, dtype=np.int64)
        cfg.col_bounds = cbs.ctypes.data
    if row_bounds is not None:
        rbs = np.ascontiguousarray(row_bounds, dtype=np.int64)
        cfg.row_bounds = rbs.ctypes.data
    rc = lib().hqr_setup(ctypes.byref(cfg))
    if rc:
        raise HQRError(rc, "hqr_setup")


def teardown() -> None:
    rc = lib().hqr_teardown()
    if rc:
        raise HQRError(rc, "hqr_teardown")


def _ptr_n(A):
    """(pointer, n) of a column-major fp64 matrix given as a torch CUDA view or numpy F-array."""
    if A is None:
        return None, None
    if isinstance(A, np.ndarray):
        if A.dtype != np.float64 or A.ndim != 2 or A.shape[0] != A.shape[1] or not A.flags.f_contiguous:
            raise TypeError("host matrices must be square float64 Fortran-ordered numpy arrays")
        return A.ctypes.data, A.shape[0]
    import torch
    if not isinstance(A, torch.Tensor) or A.dtype != torch.float64 or A.dim() != 2:
        raise TypeError("device matrices must be 2-D torch.float64 tensors")
    n = A.shape[0]
    if A.shape[1] != n or A.stride() != (1, n):
        raise TypeError("device matrices must be column-major views (stride (1, n)); see to_device()")
    return A.data_ptr(), n


def sweep(H, Z, ilo: int, ihi: int, shifts_re, shifts_im, window: int = DEFAULT_WINDOW) -> None:
    """One multishift QR sweep in place: H <- Q^T H Q, Z <- Z Q (include/hqr.h hqr_sweep)."""
    hp, n = _ptr_n(H)
    zp, nz = _ptr_n(Z)
    if hp is None:
        raise HQRError(-1, "hqr_sweep")
    if zp is not None and nz != n:
        raise ValueError("H and Z must have the same order")
    sr = np.ascontiguousarray(shifts_re, dtype=np.float64)
    si = np.ascontiguousarray(shifts_im, dtype=np.float64)
    if sr.shape != si.shape:
        raise ValueError("shifts_re and shifts_im must have the same length")
    rc = lib().hqr_sweep(hp, zp, n, ilo, ihi, sr.ctypes.data, si.ctypes.data, int(sr.shape[0]),
                         int(window))
    if rc:
        raise HQRError(rc, "hqr_sweep")


def sweep_multi(H, Z, blocks, shifts_re, shifts_im, window: int = DEFAULT_WINDOW) -> None:
    """One sweep over several decoupled active blocks: blocks = [(ilo, ihi, nshifts), ...]
    (ascending, disjoint); shifts of block i follow those of blocks 0..i-1 (hqr_sweep_multi)."""
    hp, n = _ptr_n(H)
    zp, nz = _ptr_n(Z)
    if hp is None:
        raise HQRError(-1, "hqr_sweep_multi")
    if zp is not None and nz != n:
        raise ValueError("H and Z must have the same order")
    ilo = np.array([b[0] for b in blocks], dtype=np.int64)
    ihi = np.array([b[1] for b in blocks], dtype=np.int64)
    ns = np.array([b[2] for b in blocks], dtype=np.int32)
    sr = np.ascontiguousarray(shifts_re, dtype=np.float64)
    si = np.ascontiguousarray(shifts_im, dtype=np.float64)
    if sr.shape != si.shape or sr.shape[0] != int(ns.sum()):
        raise ValueError("shift arrays must hold sum(nshifts) entries")
    rc = lib().hqr_sweep_multi(hp, zp, n, len(blocks), ilo.ctypes.data, ihi.ctypes.data,
                               sr.ctypes.data, si.ctypes.data, ns.ctypes.data, int(window))
    if rc:
        raise HQRError(rc, "hqr_sweep_multi")


def sweeps(H, Z, ilo: int, ihi: int, shift_sets, window: int = DEFAULT_WINDOW) -> None:
    """Several sweeps of one block, overlapped (hqr_sweeps): shift_sets = [(re, im), ...], applied
    in order; the result is sweep() called once per set."""
    hp, n = _ptr_n(H)
    zp, nz = _ptr_n(Z)
    if hp is None:
        raise HQRError(-1, "hqr_sweeps")
    if zp is not None and nz != n:
        raise ValueError("H and Z must have the same order")
    sr = np.ascontiguousarray(np.concatenate([np.asarray(r, dtype=np.float64) for r, _ in shift_sets]))
    si = np.ascontiguousarray(np.concatenate([np.asarray(i, dtype=np.float64) for _, i in shift_sets]))
    ns = np.array([len(r) for r, _ in shift_sets], dtype=np.int32)
    if sr.shape != si.shape:
        raise ValueError("re / im lengths differ")
    rc = lib().hqr_sweeps(hp, zp, n, ilo, ihi, len(shift_sets), sr.ctypes.data, si.ctypes.data,
                          ns.ctypes.data, int(window))
    if rc:
        raise HQRError(rc, "hqr_sweeps")


def plan_query_sweeps(n: int, ilo: int, ihi: int, nshifts_list, window: int):
    """plan_query for hqr_sweeps: (info dict, windows int32 [nw, 12])."""
    ns = np.array(nshifts_list, dtype=np.int32)
    info = np.zeros(10, dtype=np.int32)
    args = (n, ilo, ihi, len(ns), ns.ctypes.data, window)
    rc = lib().hqr_plan_query_sweeps(*args, info.ctypes.data, None, 0)
    if rc:
        raise HQRError(rc, "hqr_plan_query_sweeps")
    nw = int(info[6])
    wins = np.zeros((nw, 12), dtype=np.int32)
    rc = lib().hqr_plan_query_sweeps(*args, info.ctypes.data, wins.ctypes.data, nw)
    if rc:
        raise HQRError(rc, "hqr_plan_query_sweeps")
    keys = ["k", "nbc_max", "s", "lag", "nchains", "nsteps", "nwindows", "max_kw", "max_nbc", "nb"]
    return dict(zip(keys, (int(v) for v in info))), wins


def qz_sweep(H, T, Q, Z, ilo: int, ihi: int, shifts_re, shifts_im, window: int = 64) -> None:
    """Generalized (QZ) multishift sweep in place on device matrices (include/hqr.h hqr_qz_sweep):
    (H, T) <- Q_s^T (H, T) Z_s, Q <- Q Q_s, Z <- Z Z_s (Q / Z may be None)."""
    hp, n = _ptr_n(H)
    tp, nt = _ptr_n(T)
    qp, nq = _ptr_n(Q)
    zp, nz = _ptr_n(Z)
    if hp is None:
        raise HQRError(-1, "hqr_qz_sweep")
    if tp is None:
        raise HQRError(-2, "hqr_qz_sweep")
    if nt != n or (qp is not None and nq != n) or (zp is not None and nz != n):
        raise ValueError("H, T, Q, Z must have the same order")
    sr = np.ascontiguousarray(shifts_re, dtype=np.float64)
    si = np.ascontiguousarray(shifts_im, dtype=np.float64)
    rc = lib().hqr_qz_sweep(hp, tp, qp, zp, n, ilo, ihi, sr.ctypes.data, si.ctypes.data, int(sr.shape[0]),
                            int(window))
    if rc:
        raise HQRError(rc, "hqr_qz_sweep")


def qr_iterate(H, Z, ilo: int, ihi: int, nshifts: int = 32, window: int = DEFAULT_WINDOW, nmin: int = 64,
               max_sweeps: int = 10000, aed_window: int = 0):
    """QR iteration (include/hqr.h hqr_qr_iterate) on device H (and Z): returns (wr, wi, info,
    sweeps) with the eigenvalues of rows ilo..ihi in wr / wi.  aed_window > 0: AED (R22)."""
    hp, n = _ptr_n(H)
    zp, _ = _ptr_n(Z)
    wr, wi = np.zeros(n), np.zeros(n)
    sw = ctypes.c_int()
    rc = lib().hqr_qr_iterate(hp, zp, n, ilo, ihi, int(nshifts), int(window), int(nmin), int(aed_window),
                              int(max_sweeps), wr.ctypes.data, wi.ctypes.data, ctypes.byref(sw))
    if rc < 0:
        raise HQRError(rc, "hqr_qr_iterate")
    return wr, wi, rc, sw.value


def aed(H, Z, ilo: int, k0: int, nw: int, thr: float):
    """One AED step (include/hqr.h hqr_aed, R22 / R23) on the window [k0, k0+nw) of device H (and Z):
    returns (nd, eigenvalues of the final window blocks as complex, nw entries in window order; the
    first nw - nd are the undeflated candidates)."""
    hp, n = _ptr_n(H)
    zp, _ = _ptr_n(Z)
    ew, ei = np.zeros(nw), np.zeros(nw)
    nd, m = ctypes.c_int(), ctypes.c_int()
    rc = lib().hqr_aed(hp, zp, n, int(ilo), int(k0), int(nw), ctypes.c_double(thr), ew.ctypes.data,
                       ei.ctypes.data, ctypes.byref(nd), ctypes.byref(m))
    if rc:
        raise HQRError(rc, "hqr_aed")
    return nd.value, ew + 1j * ei


def dist_layout(n: int, world: int):
    """(col_bounds, row_bounds, halo) of the sharded layout (include/hqr.h hqr_dist_layout)."""
    cb = np.zeros(world + 1, dtype=np.int64)
    rb = np.zeros(world + 1, dtype=np.int64)
    halo = ctypes.c_int()
    rc = lib().hqr_dist_layout(n, world, cb.ctypes.data, rb.ctypes.data, ctypes.byref(halo))
    if rc:
        raise HQRError(rc, "hqr_dist_layout")
    return cb, rb, halo.value


def dist_query(n, ilo, ihi, nshifts, window, world, rank) -> np.ndarray:
    """Per-step rank roles: rows {step, lend_out, lend_in, lc0, lc1, n_owned}."""
    steps = lib().hqr_dist_query(n, ilo, ihi, nshifts, window, world, rank, None, 0)
    if steps < 0:
        raise HQRError(steps, "hqr_dist_query")
    out = np.zeros((steps, 6), dtype=np.int64)
    rc = lib().hqr_dist_query(n, ilo, ihi, nshifts, window, world, rank, out.ctypes.data, steps)
    if rc:
        raise HQRError(rc, "hqr_dist_query")
    return out


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    rc = lib().hqr_nccl_unique_id(buf)
    if rc:
        raise HQRError(rc, "hqr_nccl_unique_id")
    return buf.raw


def sweep_dist(H_local_ptr: int, Z_local_ptr, n, ilo, ihi, shifts_re, shifts_im, window) -> None:
    """Collective sharded sweep on this rank's shards (raw device pointers, hqr_dist_layout)."""
    sr = np.ascontiguousarray(shifts_re, dtype=np.float64)
    si = np.ascontiguousarray(shifts_im, dtype=np.float64)
    rc = lib().hqr_sweep_dist(H_local_ptr, Z_local_ptr, n, ilo, ihi, sr.ctypes.data, si.ctypes.data,
                              int(sr.shape[0]), int(window))
    if rc:
        raise HQRError(rc, "hqr_sweep_dist")


def sweep_virtual(H, Z, ilo, ihi, shifts_re, shifts_im, window, vworld: int) -> None:
    """The sharded algorithm with `vworld` virtual ranks on one GPU (device H, Z as in sweep)."""
    hp, n = _ptr_n(H)
    zp, _ = _ptr_n(Z)
    sr = np.ascontiguousarray(shifts_re, dtype=np.float64)
    si = np.ascontiguousarray(shifts_im, dtype=np.float64)
    rc = lib().hqr_sweep_virtual(hp, zp, n, ilo, ihi, sr.ctypes.data, si.ctypes.data, int(sr.shape[0]),
                                 int(window), int(vworld))
    if rc:
        raise HQRError(rc, "hqr_sweep_virtual")


def sweep_virtual_multi(H, Z, blocks, shifts_re, shifts_im, window, vworld: int) -> None:
    """The sharded algorithm over several decoupled blocks with vworld virtual ranks on one GPU."""
    hp, n = _ptr_n(H)
    zp, _ = _ptr_n(Z)
    ilo = np.array([b[0] for b in blocks], dtype=np.int64)
    ihi = np.array([b[1] for b in blocks], dtype=np.int64)
    ns = np.array([b[2] for b in blocks], dtype=np.int32)
    sr = np.ascontiguousarray(shifts_re, dtype=np.float64)
    si = np.ascontiguousarray(shifts_im, dtype=np.float64)
    rc = lib().hqr_sweep_virtual_multi(hp, zp, n, len(blocks), ilo.ctypes.data, ihi.ctypes.data, sr.ctypes.data,
                                       si.ctypes.data, ns.ctypes.data, int(window), int(vworld))
    if rc:
        raise HQRError(rc, "hqr_sweep_virtual_multi")


def sweep_dist_multi(H_local_ptr: int, Z_local_ptr, n, blocks, shifts_re, shifts_im, window) -> None:
    """Collective sharded sweep over several decoupled blocks on this rank's shards."""
    ilo = np.array([b[0] for b in blocks], dtype=np.int64)
    ihi = np.array([b[1] for b in blocks], dtype=np.int64)
    ns = np.array([b[2] for b in blocks], dtype=np.int32)
    sr = np.ascontiguousarray(shifts_re, dtype=np.float64)
    si = np.ascontiguousarray(shifts_im, dtype=np.float64)
    rc = lib().hqr_sweep_dist_multi(H_local_ptr, Z_local_ptr, n, len(blocks), ilo.ctypes.data, ihi.ctypes.data,
                                    sr.ctypes.data, si.ctypes.data, ns.ctypes.data, int(window))
    if rc:
        raise HQRError(rc, "hqr_sweep_dist_multi")


def sweep_raw(H_ptr, Z_ptr, n, ilo, ihi, sr_ptr, si_ptr, nshifts, window) -> int:
    """Direct ABI call (tests of the error codes); returns the C return code."""
    return lib().hqr_sweep(H_ptr, Z_ptr, n, ilo, ihi, sr_ptr, si_ptr, nshifts, window)


def plan_query(n: int, ilo: int, ihi: int, nshifts: int, window: int):
    """Host-only plan introspection: (info dict, windows int32 array [nw, 12]) or raises.
    Window columns: step, chain, w0, w1, t0, t1, b0, nbc, slot, last, ilo, ihi."""
    return plan_query_multi(n, [(ilo, ihi, nshifts)], window)


def plan_query_multi(n: int, blocks, window: int):
    """plan_query for several decoupled active blocks [(ilo, ihi, nshifts), ...]."""
    ilo = np.array([b[0] for b in blocks], dtype=np.int64)
    ihi = np.array([b[1] for b in blocks], dtype=np.int64)
    ns = np.array([b[2] for b in blocks], dtype=np.int32)
    info = np.zeros(10, dtype=np.int32)
    args = (n, len(blocks), ilo.ctypes.data, ihi.ctypes.data, ns.ctypes.data, window)
    rc = lib().hqr_plan_query_multi(*args, info.ctypes.data, None, 0)
    if rc:
        raise HQRError(rc, "hqr_plan_query_multi")
    nw = int(info[6])
    wins = np.zeros((nw, 12), dtype=np.int32)
    rc = lib().hqr_plan_query_multi(*args, info.ctypes.data, wins.ctypes.data, nw)
    if rc:
        raise HQRError(rc, "hqr_plan_query_multi")
    keys = ["k", "nbc_max", "s", "lag", "nchains", "nsteps", "nwindows", "max_kw", "max_nbc", "nb"]
    return dict(zip(keys, (int(v) for v in info))), wins


def aftermath(n: int) -> np.ndarray:
    """Aftermath flags (int8 per row) of the last single-GPU sweep (include/hqr.h
    hqr_get_aftermath): 2 exact zero subdiagonal, 1 negligible, 0 not small, -1 not scanned."""
    out = np.empty(n, dtype=np.int8)
    rc = lib().hqr_get_aftermath(out.ctypes.data, n)
    if rc:
        raise HQRError(rc, "hqr_get_aftermath")
    return out


def stats() -> dict:
    st = Stats()
    lib().hqr_get_stats(ctypes.byref(st))
    return st.as_dict()


def to_device(A: np.ndarray, device: str = "cuda"):
    """numpy Fortran array -> torch CUDA column-major view (stride (1, n))."""
    import torch
    return torch.from_numpy(np.ascontiguousarray(A.T)).to(device).t()


def from_device(T) -> np.ndarray:
    """torch column-major view -> numpy Fortran array."""
    return np.asfortranarray(T.t().contiguous().cpu().numpy().T)
