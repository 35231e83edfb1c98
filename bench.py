"""bench.py -- one multishift QR sweep per step on B200 (BASELINE.json metric), JSON line on rank 0.

python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--window 96] [--impl ours|reference]

A "step" is one full sweep (every SURVEY §8(a) row: shift pairing, bulge introduction, in-window
chase, left / right / Z updates) over the seeded synthetic BASELINE.json configs[--config]
(default configs[3]: n = 20000, 512 shifts, Z = random orthogonal -- the largest configuration that
fits one GPU and the one the north_star target is quoted on).  H and Z are restored from pristine
device copies before every step (untimed); each sweep is timed with CUDA events on the library's
stream boundary (synchronize on both sides).  Inputs (2 x 3.2 GB) are far larger than L2.

value = F_alg / t  (fp64 GFLOP/s; F_alg = flops of applying every reflector directly, SURVEY
Appendix B, design independent).  Also reported: seconds/sweep, executed GEMM flops and their
fraction of the measured FP64 DMMA peak (profiles/fp64_peaks_r01.json), the update kernel's
roofline, the oracle's CPU baseline on a bounded sample, and the end-to-end number with host
buffers (pinned host memory, host<->device copies inside the C-ABI call).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_PEAK_FILE = os.path.join(ROOT, "profiles", "fp64_peaks_r01.json")
METRIC = "seconds/sweep & fp64 GFLOP/s (frac of FP64 TC peak), n=10k/20k, 1/2/4/8 B200"


def ncu_traffic(persistent, workload, sweeps):
    """DRAM bytes per fused-kernel launch from the committed ncu captures (profiles/): the
    persistent launch (one per sweep) from the launch list, or one step's launch. Only the workload
    the capture was taken on (its "workload" key, one sweep per launch) gets a number; every other
    workload reports traffic null (no capture of it)."""
    path = os.path.join(ROOT, "profiles", "ncu_step_summary.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        d = json.load(f)
    if persistent:
        if "persistent_launch" not in d:
            return None
        d = d["persistent_launch"]
    if d.get("workload") != workload or sweeps != 1:
        return None
    return {"bytes_per_launch": d["dram_bytes_read"] + d["dram_bytes_write"], "source": d["source"]}


def gpu_local_cpus(dev):
    """Restrict this process to the host CPUs NVML reports as local to GPU `dev` (so pinned buffers
    allocated next land on its NUMA node); returns the previous affinity, or None if unavailable."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(dev)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        cpus = {64 * i + b for i, w in enumerate(words) for b in range(64) if (w >> b) & 1}
        cpus &= set(os.sched_getaffinity(0))
        if not cpus:
            return None
        prev = os.sched_getaffinity(0)
        os.sched_setaffinity(0, cpus)
        return prev
    except Exception:
        return None


def fp64_peak():
    with open(FP64_PEAK_FILE) as f:
        d = json.load(f)
    return d["dmma_sustained_tflops"], d["dmma_burst_tflops"]


def dgemm_peak():
    with open(FP64_PEAK_FILE) as f:
        d = json.load(f)
    return d.get("cublas_dgemm_8192_sustained_tflops")


class Clocks:
    """SM clock and throttle-reason sampling during the timed region (B200_PROFILING.md clocks
    line): an NVML thread polling every 10 ms (enough samples in a sub-second region), else
    `nvidia-smi -lms 200`."""

    _REASON_BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
                    "hw_thermal_slowdown": 0x40}

    def __init__(self, index=0):
        self.p = None
        self.thread = None
        self.sm, self.smax, self.reasons = [], None, set()
        try:
            import threading
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.smax = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            get_reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
            self.stop_evt = threading.Event()

            def poll():
                while True:
                    self.sm.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                    bits = get_reasons(h)
                    for nm, b in self._REASON_BITS.items():
                        if bits & b:
                            self.reasons.add(nm)
                    if self.stop_evt.wait(0.01):
                        return

            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            return
        except Exception:
            self.thread = None
        self.path = f"/tmp/bench_clocks_{os.getpid()}.csv"
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.thread is not None:
            self.stop_evt.set()
            self.thread.join()
            sm, smax, reasons, how = self.sm, self.smax, self.reasons, "nvml 10 ms"
        elif self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        else:
            self.p.terminate()
            self.p.wait()
            self.f.close()
            sm, smax, reasons, how = [], None, set(), "nvidia-smi 200 ms"
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            for line in open(self.path):
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    smax = float(parts[2])
                except ValueError:
                    continue
                for nm, v in zip(names, parts[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
        loaded = [s for s in sm if smax and s > 0.5 * smax] or sm
        return {"sm_mhz": float(np.median(loaded)) if loaded else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm), "sampler": how}


def host_info():
    """CPU model, OpenMP threads and affinity of the host the oracle runs on."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    aff = sorted(os.sched_getaffinity(0))
    return {"cpu_model": model, "omp_num_threads": os.environ.get("OMP_NUM_THREADS"),
            "affinity_cpus": len(aff), "nproc": os.cpu_count()}


def cpu_baseline(prob, bulges, n, ilo, ihi):
    """The oracle as it stands on this host's cores, on a bounded sample: the first `bulges`
    shift pairs on the full matrix (F_alg per pair is the same for every pair)."""
    import oracle
    H = prob.H.copy(order="F")
    Z = prob.Z.copy(order="F") if prob.Z is not None else None
    t = time.perf_counter()
    oracle.sweep(H, Z, ilo, ihi, prob.shifts_re, prob.shifts_im, bulges=(0, bulges))
    dt = time.perf_counter() - t
    f = oracle.flops(n, ilo, ihi, bulges, Z is not None)
    cores = int(os.environ.get("OMP_NUM_THREADS", len(os.sched_getaffinity(0))))
    return {"value": f / dt / 1e9, "unit": "GFLOP/s", "cores": cores, "kind": "oracle",
            "sample": f"first {bulges} of {len(prob.shifts_re) // 2} shift pairs on the full "
                      f"n={n} matrix ({dt:.1f} s; F_alg {f:.3e})",
            "seconds_per_sweep_extrapolated": dt * (len(prob.shifts_re) // 2) / bulges,
            "host": host_info()}


def f_alg(n, ilo, ihi, nb, with_z):
    # SURVEY Appendix B (same closed form the oracle reports; recomputed here without oracle/)
    tot = 0.0
    p = np.arange(ilo - 1, ihi - 1, dtype=np.float64)
    m3 = p <= ihi - 3
    c0 = np.where(p == ilo - 1, ilo, p + 1)
    r1 = np.minimum(p + np.where(m3, 3, 2) + 1, ihi)
    per = np.where(m3, 10.0, 6.0)
    tot = np.sum(per * ((n - c0) + (r1 + 1) + (n if with_z else 0)))
    return float(tot) * nb


def f_alg_qz(n, ilo, ihi, nb):
    """Flops of applying every QZ reflector directly (the QZ oracle's work): per position p a left
    m-reflector on H columns, T columns and all Q rows, then right reflectors (3- and 2-element,
    or one 2-element at the end) on H rows <= min(p+4, ihi), T rows <= the zeroed row, all Z rows."""
    tot = 0.0
    for p in range(ilo - 1, ihi - 1):
        m = 3 if p <= ihi - 3 else 2
        per = 10.0 if m == 3 else 6.0
        c0 = ilo if p == ilo - 1 else p + 1
        tot += per * ((n - c0) + (n - (p + 1)) + n)
        hr = min(p + 4, ihi)
        for mm in range(m, 1, -1):
            tot += (10.0 if mm == 3 else 6.0) * ((hr + 1) + (p + mm + 1) + n)
    return tot * nb


def run_qz(args):
    """--workload qz: one generalized multishift sweep (hqr_qz_sweep) per step, single GPU."""
    import torch
    import paper_2007_03576_b200 as hq
    from hqr_inputs import make_qz
    n = args.n or 10000
    ns = 256
    win = min(args.window, 80)
    t0 = time.time()
    p = make_qz(n, ns, q0="eye")
    gen_s = time.time() - t0
    hq.setup(0)
    dev = torch.device("cuda", 0)
    src = [hq.to_device(A, dev) for A in (p.H, p.T, p.Q, p.Z)]
    work = [torch.empty_like(A.t()).t() for A in src]

    def restore():
        for w, s0 in zip(work, src):
            w.t().copy_(s0.t())

    def one():
        hq.qz_sweep(work[0], work[1], work[2], work[3], 0, n - 1, p.shifts_re, p.shifts_im, win)

    for _ in range(args.warmup):
        restore()
        one()
    torch.cuda.synchronize()
    clk = Clocks(0)
    times, launches = [], 0
    for _ in range(args.steps):
        restore()
        torch.cuda.synchronize()
        one()
        st = hq.stats()
        times.append(st["ms_total"])
        launches += st["kernels_launched"]
    clocks = clk.stop()
    ms = float(np.mean(times))
    fa = f_alg_qz(n, 0, n - 1, ns // 2)
    peak_sus, _ = fp64_peak()
    dense = st["flops_update"] / (ms * 1e-3) / 1e12
    hq.teardown()
    line = {"metric": METRIC, "value": fa / (ms * 1e-3) / 1e9, "unit": "GFLOP/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded: H as configs[2], T upper triangular diag U[1,2] + N(0,1/n))",
            "config": {"workload": f"QZ sweep (NEXT-4) on (H, T), n={n}, {ns} shifts", "n": n, "nshifts": ns,
                       "window": st["window_eff"], "q0_z0": "identity", "parallelism": "1 GPU",
                       "l2": "inputs (4 x %.1f GB) larger than L2" % (n * n * 8 / 1e9)},
            "seconds_per_sweep": ms * 1e-3, "gflops_alg": fa / (ms * 1e-3) / 1e9,
            "roofline": {"bound": "tensor", "kernel": "whole sweep: QZ chase + update.cu DMMA GEMMs (separate "
                         "launches)", "achieved": dense, "peak": peak_sus, "unit": "TFLOP/s",
                         "frac": dense / peak_sus, "achieved_what": "dense update GEMM flops (2 m n k) / sweep time",
                         "traffic": None},
            "clocks": clocks, "gpu_launches": launches, "steps_per_sweep": st["steps"], "input_gen_s": gen_s,
            "cpu_baseline": None, "e2e": None}
    print(json.dumps(line), flush=True)


def run_qriter(args):
    """--workload qriter: hqr_qr_iterate to all eigenvalues (one call per step), single GPU."""
    import torch
    import paper_2007_03576_b200 as hq
    from hqr_inputs import hessenberg, orthogonal
    n = args.n or 4000
    ns, nmin = 64, 96
    from hqr_inputs import make_hess
    H0 = make_hess(n, 2).H   # hess_n: Ginibre-like, eigenvalues well conditioned
    Z0 = np.asfortranarray(np.eye(n))
    hq.setup(0)
    src = [hq.to_device(A) for A in (H0, Z0)]
    work = [torch.empty_like(A.t()).t() for A in src]

    def restore():
        for w, s0 in zip(work, src):
            w.t().copy_(s0.t())

    aed = 96
    for _ in range(args.warmup):
        restore()
        hq.qr_iterate(work[0], work[1], 0, n - 1, nshifts=ns, window=args.window, nmin=nmin, aed_window=aed)
    torch.cuda.synchronize()
    clk = Clocks(0)
    wall, dev, sweeps, falg, naed, ndefl = [], [], [], [], [], []
    for _ in range(args.steps):
        restore()
        torch.cuda.synchronize()
        t = time.perf_counter()
        wr, wi, rc, sw = hq.qr_iterate(work[0], work[1], 0, n - 1, nshifts=ns, window=args.window, nmin=nmin,
                                       aed_window=aed)
        wall.append(time.perf_counter() - t)
        st = hq.stats()
        dev.append(st["ms_total"])
        sweeps.append(sw)
        falg.append(st["flops_alg"])
        naed.append(st["launches_chase"])
        ndefl.append(st["window_eff"])
        assert rc == 0
    clocks = clk.stop()
    # the same iteration without AED (shifts from the trailing block, R21), for comparison
    restore()
    torch.cuda.synchronize()
    t = time.perf_counter()
    _, _, rc0, sw0 = hq.qr_iterate(work[0], work[1], 0, n - 1, nshifts=ns, window=args.window, nmin=nmin)
    wall0 = time.perf_counter() - t
    hq.teardown()
    ms = float(np.mean(dev))
    line = {"metric": METRIC, "value": float(np.mean(falg)) / (ms * 1e-3) / 1e9, "unit": "GFLOP/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded hess_n, PAPER.md P:1061-1068: N(0,1) upper entries, sqrt(chi^2(n-i)) subdiagonal)",
            "config": {"workload": f"QR iteration with AED (NEXT-2, window {aed}) to all eigenvalues, n={n}, up to "
                                   f"{ns} shifts per sweep, blocks <= {nmin} by the one-CTA solver", "n": n,
                       "nshifts": ns, "aed_window": aed, "window": args.window, "parallelism": "1 GPU"},
            "seconds_to_eigenvalues_wall": float(np.mean(wall)), "sweeps": float(np.mean(sweeps)),
            "aed_steps": float(np.mean(naed)), "eigenvalues_deflated_by_aed": float(np.mean(ndefl)),
            "without_aed": {"seconds_wall": wall0, "sweeps": sw0},
            "gflops_alg_over_sweeps": float(np.mean(falg)) / (ms * 1e-3) / 1e9,
            "roofline": None, "clocks": clocks, "cpu_baseline": None, "e2e": None, "gpu_launches": None}
    print(json.dumps(line), flush=True)


def chase_line(hq, n, prob, nshifts, args, ms_chase, clocks, sweep_ms):
    """The chase kernel's own figures (north_star: its achieved HBM GB/s): step 0's windows run in a
    standalone chase launch (timed with CUDA events under FLAG_PROFILE); every later window is chased
    inside the persistent kernel with the same code.  Algorithmic bytes per window: H(W,W) in and out
    plus Q_W out, 3 k^2 doubles."""
    if args.sweeps > 1 or ms_chase <= 0:
        return None
    try:
        info, wins = hq.plan_query(n, prob.ilo, prob.ihi, nshifts, args.window)
    except Exception:  # multi-block configs: no single plan
        return None
    first = wins[wins[:, 0] == 0]
    if len(first) == 0:
        return None
    kw_all = (wins[:, 3] - wins[:, 2] + 1).astype(np.float64)
    sweep_bytes = float(np.sum(3.0 * kw_all * kw_all * 8.0))
    kw = (first[:, 3] - first[:, 2] + 1).astype(np.float64)
    steps = (first[:, 5] - first[:, 4] + 1).astype(np.float64)
    nbytes = float(np.sum(3.0 * kw * kw * 8.0))
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "MEASURED_PEAKS.json")))
    gbs = nbytes / (ms_chase * 1e-3) / 1e9
    mhz = (clocks or {}).get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
    return {"kernel": "chase kernel, step 0's windows (one standalone launch; later windows inside the "
                      "persistent kernel, same code)",
            "windows": int(len(first)), "ms": ms_chase, "us_per_window": ms_chase * 1e3 / len(first),
            "bulge_steps_per_window": float(steps.mean()),
            "cycles_per_bulge_step": ms_chase * 1e-3 * mhz * 1e6 / float(steps.max()),
            "algorithmic_bytes": nbytes, "achieved_gbs": gbs, "peak_gbs": peaks["hbm_gbs"],
            "frac_hbm": gbs / peaks["hbm_gbs"],
            "sweep_windows": int(len(wins)), "sweep_chase_bytes": sweep_bytes,
            "sweep_chase_gbs_over_sweep_time": sweep_bytes / (sweep_ms * 1e-3) / 1e9,
            "bound": "latency: the reflector chain and SMEM traffic of the in-window chase (DESIGN.md §6), "
                     "not HBM; the windows of a step run concurrently, one CTA each"}


def run_reference(args, cfg_idx):
    """--impl reference: the oracle timed as it stands on the host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from hqr_inputs import make
    prob = make(cfg_idx)
    n = prob.H.shape[0]
    steps = []
    cb = None
    for i in range(args.warmup + args.steps):
        cb = cpu_baseline(prob, args.ref_bulges, n, prob.ilo, prob.ihi)
        if i >= args.warmup:
            steps.append(cb["value"])
    v = float(np.mean(steps))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "GFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": None, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded, BASELINE.json configs)",
            "config": {"workload": f"configs[{cfg_idx}]", "n": n, "nshifts": len(prob.shifts_re)},
            "cpu_baseline": {"value": v, "unit": "GFLOP/s", "cores": cb["cores"], "kind": "oracle",
                             "sample": cb["sample"]},
            "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--window", type=int, default=None,
                    help="window side (default: the config's window when BASELINE.json gives one -- configs[0] 24, "
                         "configs[1] 151 -- else 96); the library's effective side is min(window, N, 112)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-bulges", type=int, default=32, help="oracle sample size (shift pairs)")
    ap.add_argument("--ref-bulges", type=int, default=16)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--n", type=int, default=None, help="override n (debug)")
    ap.add_argument("--sweeps", type=int, default=1,
                    help="NEXT-1: this many overlapped sweeps per step (hqr_sweeps), shift set 0 = the "
                         "config's, the others drawn from the same distribution")
    ap.add_argument("--workload", default="config", choices=["config", "hess", "qz", "qriter"],
                    help="hess: the paper's hess_n matrix (NEXT-3) at --n (default 10000), 256 shifts; "
                         "qz: the generalized sweep (NEXT-4) on a Hessenberg-triangular pair at --n "
                         "(default 10000), 256 shifts, window 80; qriter: the QR iteration (NEXT-2 without AED) "
                         "to all eigenvalues of a random Hessenberg matrix at --n (default 4000), 64 shifts "
                         "per sweep")
    args = ap.parse_args()

    if args.impl == "reference":
        run_reference(args, args.config)
        return

    import torch
    import paper_2007_03576_b200 as hq
    from hqr_inputs import make

    window_requested = args.window
    if args.workload == "qz":
        args.window = args.window or 80
        run_qz(args)
        return
    if args.workload == "qriter":
        args.window = args.window or 96
        run_qriter(args)
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    t0 = time.time()
    if args.workload == "hess":
        from hqr_inputs import make_hess
        prob = make_hess(args.n or 10000, 256, z0="orth", z_device="cuda" if torch.cuda.is_available() else "cpu")
        workload = f"hess_n (P:1061-1068), n={prob.H.shape[0]}, 256 shifts (NEXT-3)"
    else:
        prob = make(args.config, z_device="cuda" if torch.cuda.is_available() else "cpu", n_override=args.n)
        workload = f"configs[{args.config}]"
    n = prob.H.shape[0]
    gen_s = time.time() - t0
    nshifts = len(prob.shifts_re)
    window_note = None
    if args.window is None:  # the config's window, else the default 96
        args.window = prob.window if prob.window else 96
        if args.window > 112:  # configs[1]'s 3 nshifts/2 + 1 = 151 exceeds the library's 112 (SMEM)
            window_note = (f"config window {args.window} exceeds the maximum 112 (R5 / DESIGN.md); the default 96 "
                           f"is used (112: slower)")
            args.window = 96
    shift_sets = None
    if args.sweeps > 1:  # NEXT-1: further shift sets from the same distribution (stream offsets)
        from hqr_inputs import CONFIGS, shifts as draw_shifts
        c = CONFIGS[args.config]
        shift_sets = [(prob.shifts_re, prob.shifts_im)] + [
            draw_shifts(c.shifts, c.nshifts, c.idx, stream_offset=i) for i in range(1, args.sweeps)]
        workload += f" x {args.sweeps} overlapped sweeps (hqr_sweeps, NEXT-1)"

    if world == 1:
        hq.setup(local)
        H0 = hq.to_device(prob.H, dev)
        Z0 = hq.to_device(prob.Z, dev)
        H = torch.empty_like(H0.t()).t()
        Z = torch.empty_like(Z0.t()).t()

        def restore():
            H.t().copy_(H0.t())
            Z.t().copy_(Z0.t())

        if len(prob.blocks) > 1:  # configs[4]: decoupled blocks swept together (hqr_sweep_multi)
            blocks = [(b[0], b[1], b[3]) for b in prob.blocks]

            def call(Hx, Zx):
                hq.sweep_multi(Hx, Zx, blocks, prob.shifts_re, prob.shifts_im, args.window)
        elif shift_sets is not None:
            def call(Hx, Zx):
                hq.sweeps(Hx, Zx, prob.ilo, prob.ihi, shift_sets, args.window)
        else:
            def call(Hx, Zx):
                hq.sweep(Hx, Zx, prob.ilo, prob.ihi, prob.shifts_re, prob.shifts_im, args.window)

        def one():
            call(H, Z)
    else:
        # sharded sweep: this rank's H column shard (+ halo) and Z row shard
        import torch.distributed as dist
        uid = [hq.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        hq.setup(local, rank=rank, world=world, nccl_id=uid[0])
        cb, rb, halo = hq.dist_layout(n, world)
        c0, c1, r0, r1 = int(cb[rank]), int(cb[rank + 1]), int(rb[rank]), int(rb[rank + 1])
        # column-major shards as row-major tensors of their transposes: row j = local column j
        H0 = torch.zeros((c1 - c0 + halo, n), dtype=torch.float64, device=dev)
        H0[:c1 - c0].copy_(torch.from_numpy(np.ascontiguousarray(prob.H[:, c0:c1].T)))
        Z0 = torch.from_numpy(np.ascontiguousarray(prob.Z[r0:r1, :].T)).to(dev)
        H = torch.empty_like(H0)
        Z = torch.empty_like(Z0)

        def restore():
            H.copy_(H0)
            Z.copy_(Z0)

        if len(prob.blocks) > 1:  # configs[4]: decoupled blocks, sharded (hqr_sweep_dist_multi)
            blocks = [(b[0], b[1], b[3]) for b in prob.blocks]

            def one():
                hq.sweep_dist_multi(H.data_ptr(), Z.data_ptr(), n, blocks, prob.shifts_re, prob.shifts_im,
                                    args.window)
        else:
            def one():
                hq.sweep_dist(H.data_ptr(), Z.data_ptr(), n, prob.ilo, prob.ihi, prob.shifts_re,
                              prob.shifts_im, args.window)

    for _ in range(args.warmup):
        restore()
        one()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clk = Clocks(local)
    times = []
    outer = []
    launches = 0
    for _ in range(args.steps):
        restore()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        one()   # synchronous: returns after the library stream finished
        e1.record()
        torch.cuda.synchronize()
        st = hq.stats()
        # ms_total: CUDA events recorded by the library on its own (launching) stream around the
        # sweep; the torch-stream events around the blocking call are a cross-check
        times.append(st["ms_total"] if st["ms_total"] > 0 else e0.elapsed_time(e1))
        outer.append(e0.elapsed_time(e1))
        launches += st["kernels_launched"]
    clocks = clk.stop()
    ms = float(np.mean(times))
    if world > 1:
        t = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    st = hq.stats()
    fa = sum(f_alg(n, b[0], b[1], b[3] // 2, True) for b in prob.blocks) * max(1, args.sweeps)
    sequential_ms = None
    if shift_sets is not None and world == 1:
        # the same shift sets as separate hqr_sweep calls (device-timed), for the overlap's gain
        seq = []
        for _ in range(2):
            restore()
            torch.cuda.synchronize()
            tot = 0.0
            for sre, sim in shift_sets:
                hq.sweep(H, Z, prob.ilo, prob.ihi, sre, sim, args.window)
                tot += hq.stats()["ms_total"]
            seq.append(tot)
        sequential_ms = min(seq)
    value = fa / (ms * 1e-3) / 1e9   # one sweep (strong scaling: the same sweep on every N)
    peak_sus, peak_burst = fp64_peak()
    gflops_exec = (st["flops_update"] + st["flops_chase"]) / (ms * 1e-3) / 1e9

    chase = None
    if world == 1:
        # per-kernel CUDA-event times: the same sweep in profiling mode (events around every launch)
        hq.teardown()
        hq.setup(local, flags=hq.FLAG_PROFILE)
        prof = []
        for _ in range(max(1, min(args.steps, 2))):
            restore()
            torch.cuda.synchronize()
            one()
            prof.append(hq.stats())
        hq.teardown()
        ps = prof[-1]
        if ps["ms_step"] > 0:   # fused step kernels: updates of step g + chase of step g+1
            upd_ms = ps["ms_step"]
            upd_launches = ps["launches_left"]
            kern = ("fused step kernel (left/right/Z DMMA GEMM tiles + the chases), one persistent launch "
                    "per sweep" if ps["launches_left"] == 1 else
                    "fused step kernel (left/right/Z DMMA GEMM tiles + next chase), one launch per step")
        else:
            upd_ms = ps["ms_left"] + ps["ms_right"]
            upd_launches = ps["launches_left"] + ps["launches_right"]
            kern = "update (left + right/Z DMMA GEMM)"
        # executed tensor-core work: the update GEMMs restricted to the Q_W band extents the kernels
        # actually multiply (hqr_stats.flops_dmma, recorded per window by the chase); the dense
        # 2*m*n*k count of the same GEMMs is reported beside it
        achieved = ps["flops_dmma"] / (upd_ms * 1e-3) / 1e12
        traffic = ncu_traffic(ps["launches_left"] == 1, workload, args.sweeps)
        dg = dgemm_peak()
        roofline = {"bound": "tensor", "kernel": kern,
                    "achieved": achieved, "peak": peak_sus, "unit": "TFLOP/s", "frac": achieved / peak_sus,
                    "frac_of_cublas_dgemm": achieved / dg if dg else None, "cublas_dgemm_tflops": dg,
                    "traffic": traffic["bytes_per_launch"] if traffic else None,
                    "traffic_source": traffic["source"] if traffic else
                        "no ncu capture of this workload (the committed one is configs[3], one sweep)",
                    "achieved_what": "executed FP64 DMMA flops (band-trimmed update GEMMs) per launch / "
                                     "mean CUDA-event launch time",
                    "peak_source": "measured FP64 DMMA sustained, profiles/fp64_peaks_r01.json "
                                   "(MEASURED_PEAKS.json has no fp64 entry)",
                    "flops_per_launch": ps["flops_dmma"] / max(1, upd_launches),
                    "dense_gemm_flops_per_launch": ps["flops_update"] / max(1, upd_launches),
                    "alg_panel_bytes_per_launch": ps["bytes_update"] / max(1, upd_launches),
                    "avg_launch_ms": upd_ms / max(1, upd_launches),
                    "share_of_step": upd_ms / max(1e-9, ps["ms_chase"] + upd_ms),
                    "ms_chase_only_launches": ps["ms_chase"], "ms_kernel_total": upd_ms}
        chase = chase_line(hq, n, prob, nshifts, args, ps["ms_chase"], clocks, ms)
    else:
        # per-rank GEMM flops over the whole sweep time (lower bound of the kernels' own rate)
        fl = torch.tensor([st["flops_update"]], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(fl, op=torch.distributed.ReduceOp.MAX)
        achieved = float(fl.item()) / (ms * 1e-3) / 1e12
        roofline = {"bound": "tensor", "kernel": "update GEMMs of the busiest rank over the sweep",
                    "achieved": achieved, "peak": peak_sus, "unit": "TFLOP/s", "frac": achieved / peak_sus,
                    "traffic": None, "peak_source": "measured FP64 DMMA sustained, profiles/fp64_peaks_r01.json"}
        hq.teardown()

    e2e = None
    if not args.no_e2e and rank == 0 and world == 1:
        hq.setup(local)
        aff0 = gpu_local_cpus(local)  # pinned buffers on the GPU's NUMA node, as a user would place them
        Hh = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
        Zh = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
        Hp = np.asfortranarray(prob.H)
        e2e_t = []
        for i in range(4):  # wall clock over PCIe copies varies ~20% call to call: the best of four
            Hh.copy_(torch.from_numpy(Hp.T.copy()))
            Zh.copy_(torch.from_numpy(np.ascontiguousarray(prob.Z.T)))
            rc_t = time.perf_counter()
            call(Hh.t(), Zh.t())   # pinned HOST buffers: the library stages them (copies in the call)
            dt = time.perf_counter() - rc_t
            e2e_t.append(dt)
        st2 = hq.stats()
        hq.teardown()
        if aff0 is not None:
            os.sched_setaffinity(0, aff0)
        e2e = {"value": fa / min(e2e_t) / 1e9, "unit": "GFLOP/s",
               "seconds_per_sweep": min(e2e_t),
               "h2d_bytes_per_step": st2["h2d_bytes"], "d2h_bytes_per_step": st2["d2h_bytes"],
               "how": "the same C-ABI call with pinned host H and Z (wall clock around it)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(prob, args.cpu_bulges, n, prob.ilo, prob.ihi)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE.json configs)",
            "config": {"workload": workload, "n": n, "nshifts": nshifts,
                       "sweeps_per_step": args.sweeps,
                       "window": st["window_eff"], "window_requested": window_requested or args.window,
                       **({"window_note": window_note} if window_note else {}),
                       "z": "random orthogonal" if (args.config in (1, 3) or args.workload == "hess") else "identity",
                       "parallelism": (f"{world} GPUs: H block-column (sqrt-balanced), Z block-row, "
                                       "per-window Q ncclBroadcast, lent slabs") if world > 1 else "1 GPU",
                       "l2": "inputs (2 x %.1f GB) larger than L2" % (n * n * 8 / 1e9),
                       "restore": "H, Z restored from pristine device copies before each step (untimed)"},
            "seconds_per_sweep": ms * 1e-3,
            "ms_outer_events": float(np.mean(outer)),
            "gflops_alg": value, "gflops_dense_equiv": gflops_exec,
            "frac_fp64_peak_dense_equiv": gflops_exec / 1e3 / peak_sus,
            "gflops_dmma": st["flops_dmma"] / (ms * 1e-3) / 1e9 if world == 1 else None,
            "frac_fp64_peak_dmma": st["flops_dmma"] / (ms * 1e-3) / 1e12 / peak_sus if world == 1 else None,
            "flops_dense_over_alg": (st["flops_update"] + st["flops_chase"]) / fa,
            "roofline": roofline, "chase": chase, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
            "gpu_launches": launches, "steps_per_sweep": st["steps"], "windows_per_sweep": st["windows"],
            "input_gen_s": gen_s,
            "sequential_sweeps_ms": sequential_ms,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
