"""CPU test of the multi-GPU sharded sweep protocol with world_size 2 and 3 (torch.distributed gloo,
127.0.0.1), no GPU: each process holds only its H column shard (+ halo) and Z row shard, takes its
per-step role from the C++ library (hqr_dist_layout / hqr_dist_query / hqr_plan_query: ownership,
lent column slabs, left-update column range), and executes the protocol of hqr_sweep_dist in numpy
with gloo in place of NCCL:
  (1) lend straddling slabs (send/recv of whole columns; the lender first drains its deferred
  work), (2) chase owned windows, (3) broadcast every window's factor from its owner, (4) left
  update on the held columns and near-right update (rows [sp, w0)) of the owned windows, (5) the
  deferred work -- far-right rows [0, sp) of the owned windows (straddling ones: at once) and the
  Z update of the local rows -- queued and applied up to LAG steps late, as the low-priority
  stream of hqr_sweep_dist may, (6) return the slabs.
Rank 0 gathers the result and compares it with the CPU oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_2007_03576_b200 as hq
from hqr_inputs import random_case
from schedule_emulator import chase_window, shift_coefs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


LAG = 7  # deferred (far-right / Z) work applied this many steps late


def _split_rows(W, nsteps, n):
    """sp(s): the smallest first row of any window of a later step, rounded down to even (the
    library's near / far split of the right updates)."""
    sp = [0] * nsteps
    run = n
    for s in range(nsteps - 1, -1, -1):
        sp[s] = run & ~1
        run = min(run, int(W[W[:, 0] == s][:, 2].min()))
    return sp


def _worker(rank, world, port, case, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        seed, n, ns, win = case
        H0, Z0, sr, si = random_case(seed, n, ns, z0="orth", shift_kind="disk2")
        cb, rb, halo = hq.dist_layout(n, world)
        info, W = hq.plan_query(n, 0, n - 1, ns, win)
        roles = hq.dist_query(n, 0, n - 1, ns, win, world, rank)
        sig, pis = shift_coefs(sr, si)
        c0, c1 = int(cb[rank]), int(cb[rank + 1])
        r0, r1 = int(rb[rank]), int(rb[rank + 1])
        # local shards: H columns [c0, c1 + halo) (halo columns are work space), Z rows [r0, r1)
        Hl = np.zeros((n, c1 - c0 + halo))
        Hl[:, :c1 - c0] = H0[:, c0:c1]
        Zl = Z0[r0:r1, :].copy()

        def owner(col):
            return int(np.searchsorted(cb, col, side="right") - 1)

        def cols(j0, j1):  # local view of global columns [j0, j1)
            return Hl[:, j0 - c0:j1 - c0]

        sp = _split_rows(W, info["nsteps"], n)
        deferred = []  # (step, fn) of the low-priority work, applied in order

        def drain(upto):
            while deferred and deferred[0][0] <= upto:
                deferred.pop(0)[1]()

        for s in range(info["nsteps"]):
            _, lend_out, lend_in, lc0, lc1, nown = (int(v) for v in roles[s])
            sw = W[W[:, 0] == s]
            drain(s - LAG)
            # (1) lend: my leading lend_out columns -> rank-1's halo; rank+1's -> my halo
            if lend_out or lend_in:
                # the lender's deferred work may still touch the lent columns; the borrower applies
                # its straddling window's whole right update at once, after its earlier deferred
                # far-right rows on the same columns
                drain(s)
            if lend_out:
                dist.send(torch.from_numpy(np.ascontiguousarray(cols(c0, c0 + lend_out))), rank - 1)
            if lend_in:
                buf = torch.empty((n, lend_in), dtype=torch.float64)
                dist.recv(buf, rank + 1)
                cols(c1, c1 + lend_in)[:] = buf.numpy()
            # (2) chase owned windows
            Q = {}
            owned = [w for w in sw if owner(int(w[2])) == rank]
            assert len(owned) == nown
            for w in owned:
                w0, w1 = int(w[2]), int(w[3])
                Hw = cols(w0, w1 + 1)[w0:w1 + 1].copy()
                Q[w0] = chase_window(Hw, w, sig, pis)
                cols(w0, w1 + 1)[w0:w1 + 1] = Hw
            # (3) broadcast every factor from its owner
            for w in sw:
                w0, w1 = int(w[2]), int(w[3])
                t = torch.from_numpy(Q[w0]) if w0 in Q else torch.empty((w1 - w0 + 1,) * 2, dtype=torch.float64)
                dist.broadcast(t, owner(w0))
                Q[w0] = t.numpy()
            # (4) left update of every window on the held columns [lc0, lc1)
            for w in sw:
                w0, w1 = int(w[2]), int(w[3])
                a = max(w1 + 1, lc0)
                if a < lc1:
                    blk = cols(a, lc1)
                    blk[w0:w1 + 1] = Q[w0].T @ blk[w0:w1 + 1]
            # (4) near-right rows [sp, w0) of the owned windows (all rows if the rank straddles)
            for w in owned:
                w0, w1 = int(w[2]), int(w[3])
                blk = cols(w0, w1 + 1)
                lo = 0 if lend_in else min(sp[s], w0)
                blk[lo:w0] = blk[lo:w0] @ Q[w0]
                if not lend_in and lo > 0:  # (5) far-right rows [0, sp), deferred
                    deferred.append((s, lambda w0=w0, w1=w1, lo=lo, Qw=Q[w0]:
                                     cols(w0, w1 + 1).__setitem__(slice(0, lo), cols(w0, w1 + 1)[:lo] @ Qw)))
            for w in sw:  # (5) Z of the local rows, deferred
                w0, w1 = int(w[2]), int(w[3])
                deferred.append((s, lambda w0=w0, w1=w1, Qw=Q[w0]:
                                 Zl.__setitem__((slice(None), slice(w0, w1 + 1)), Zl[:, w0:w1 + 1] @ Qw)))
            # (6) return the lent slabs
            if lend_in:
                dist.send(torch.from_numpy(np.ascontiguousarray(cols(c1, c1 + lend_in))), rank + 1)
            if lend_out:
                buf = torch.empty((n, lend_out), dtype=torch.float64)
                dist.recv(buf, rank - 1)
                cols(c0, c0 + lend_out)[:] = buf.numpy()
        drain(info["nsteps"])
        # gather on rank 0
        Hs = [torch.empty((n, int(cb[r + 1] - cb[r])), dtype=torch.float64) for r in range(world)]
        Zs = [torch.empty((int(rb[r + 1] - rb[r]), n), dtype=torch.float64) for r in range(world)]
        mine_h = torch.from_numpy(np.ascontiguousarray(Hl[:, :c1 - c0]))
        mine_z = torch.from_numpy(Zl)
        if rank == 0:
            for r in range(1, world):
                dist.recv(Hs[r], r)
                dist.recv(Zs[r], r)
            Hs[0], Zs[0] = mine_h, mine_z
            H = np.asfortranarray(np.concatenate([h.numpy() for h in Hs], axis=1))
            Z = np.asfortranarray(np.concatenate([z.numpy() for z in Zs], axis=0))
            Ho, Zo = H0.copy(order="F"), Z0.copy(order="F")
            oracle.sweep(Ho, Zo, 0, n - 1, sr, si)
            dh = np.linalg.norm(H - Ho) / np.linalg.norm(H0)
            dz = np.linalg.norm(Z - Zo) / np.sqrt(n)
            lent = int(sum(roles[:, 1].sum() for _ in [0]))
            q.put(("ok", dh, dz, bool(np.all(np.tril(H, -2) == 0.0))))
        else:
            dist.send(mine_h, 0)
            dist.send(mine_z, 0)
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put(("err", traceback.format_exc(), 0, False))


@pytest.mark.parametrize("world,case", [(2, (5, 600, 24, 24)), (3, (6, 900, 30, 32)),
                                        (2, (7, 700, 60, 96))])
def test_sharded_protocol_gloo(world, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
    assert res[0] == "ok", res[1]
    _, dh, dz, zeros = res
    assert dh <= 1e-11 and dz <= 1e-11 and zeros, (dh, dz)


def test_layout_properties():
    for n, world in [(20000, 8), (10000, 4), (600, 2), (4000, 8)]:
        cb, rb, halo = hq.dist_layout(n, world)
        assert cb[0] == 0 and cb[-1] == n and rb[0] == 0 and rb[-1] == n
        assert np.all(cb[1:-1] % 2 == 0) and np.all(rb[1:-1] % 2 == 0)
        assert np.all(np.diff(cb) >= hq.MAX_WINDOW + 8) and halo >= hq.MAX_WINDOW
        # H work grows linearly with the column index: sqrt boundaries give equal integrals
        work = np.diff(cb.astype(float) ** 2)
        assert work.max() / work.min() < 1.02
    with pytest.raises(hq.HQRError) as e:
        hq.dist_layout(500, 8)
    assert e.value.code == -11


def test_roles_consistent_across_ranks():
    n, ns, win, world = 5000, 120, 96, 4
    info, W = hq.plan_query(n, 0, n - 1, ns, win)
    cb, _, _ = hq.dist_layout(n, world)
    R = [hq.dist_query(n, 0, n - 1, ns, win, world, r) for r in range(world)]
    for s in range(info["nsteps"]):
        assert sum(R[r][s, 5] for r in range(world)) == np.count_nonzero(W[:, 0] == s)
        for r in range(world - 1):
            assert R[r][s, 2] == R[r + 1][s, 1]          # lent in == lent out of the neighbour
            assert R[r][s, 4] == R[r + 1][s, 3]          # held ranges tile [0, n)
        assert R[0][s, 3] == 0 and R[world - 1][s, 4] == n
    assert sum(R[r][:, 1].sum() for r in range(world)) > 0    # chains cross shard boundaries
