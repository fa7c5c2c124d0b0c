"""CPU: host logic of the z-slab decomposition (north_star (6)).

* the slab plan exported by the C ABI (pure host function);
* a world_size-2 (and 3) gloo run of the ghost-plane exchange schedule and
  of the agglomeration gather, on the plan's windows: after one exchange
  every rank's window must equal the global field on all stored planes.
The device transport (NVLink copies / NCCL) moves exactly these plane ranges
(csrc/ehmg_slab.cuh: exchange(), the agglomeration branch of cycle()).
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2307_03242_b200 as E


@pytest.mark.parametrize("n2,nl,ns,agg", [(256, 5, 8, 64), (256, 5, 4, 64), (64, 4, 2, 8), (96, 3, 3, 16),
                                          (32, 3, 2, 4), (513 - 1, 6, 8, 64)])
def test_slab_plan_invariants(n2, nl, ns, agg):
    la, z0 = E.slab_plan(n2, nl, ns, agg)
    assert 1 <= la <= nl - 1
    assert z0[0] == 0 and z0[-1] == n2 and len(z0) == ns + 1
    for q in range(ns):
        assert z0[q] % (1 << la) == 0
        for lv in range(la):
            assert (z0[q + 1] >> lv) - (z0[q] >> lv) >= 4
    # agglomerate levels whose z extent is <= agg (unless the partition forbids)
    assert la == 1 or (n2 >> (la - 1)) > agg


def test_slab_plan_bench_layout():
    la, z0 = E.slab_plan(256, 5, 8, 64)
    assert la == 2  # 256^3 and 128^3 sharded, 64^3 and below agglomerated
    assert z0 == [0, 32, 64, 96, 128, 160, 192, 224, 256]


def test_slab_plan_rejects_thin_grids():
    with pytest.raises(ValueError):
        E.slab_plan(8, 3, 4, 2)


# ---------------------------------------------------------------- gloo
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _comp_planes(n0, n1, nz, k):
    """(planes, plane size) of component k on a window of nz cell planes."""
    ps = (n0 + (k == 0)) * (n1 + (k == 1))
    return nz + (k == 2), ps


def _worker(rank, ws, port, n0, n1, n2, nl, agg, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import torch
    try:
        wins = E.slab_windows(n2, nl, ws, agg, level=0)
        Z0, Z1, W0, W1 = wins[rank]
        rng = np.random.default_rng(0)
        glob = [rng.standard_normal(_comp_planes(n0, n1, n2, k)) for k in range(4)]
        # window with owned planes filled, ghosts poisoned
        win = []
        for k in range(4):
            planes, ps = _comp_planes(n0, n1, W1 - W0, k)
            a = np.full((planes, ps), np.nan)
            top = Z1 + (1 if (k == 2 and rank == ws - 1) else 0)
            a[Z0 - W0:top - W0] = glob[k][Z0:top]
            win.append(a)
        # exchange schedule of ehmg_slab.cuh exchange(): per boundary zb,
        # up = cells/faces [W0_hi, zb); down = cells [zb, W1_lo), faces [zb, W1_lo]
        for b in range(ws - 1):
            lo, hi = wins[b], wins[b + 1]
            zb = lo[1]
            for k in range(4):
                up = (hi[2], zb)
                down = (zb, lo[3] + (1 if k == 2 else 0))
                if rank == b:
                    dist.send(torch.from_numpy(np.ascontiguousarray(win[k][up[0] - W0:up[1] - W0])), b + 1)
                    buf = torch.empty((down[1] - down[0], win[k].shape[1]), dtype=torch.float64)
                    dist.recv(buf, b + 1)
                    win[k][down[0] - W0:down[1] - W0] = buf.numpy()
                elif rank == b + 1:
                    buf = torch.empty((up[1] - up[0], win[k].shape[1]), dtype=torch.float64)
                    dist.recv(buf, b)
                    win[k][up[0] - W0:up[1] - W0] = buf.numpy()
                    dist.send(torch.from_numpy(np.ascontiguousarray(win[k][down[0] - W0:down[1] - W0])), b)
        ok = all(np.array_equal(win[k], glob[k][W0:W0 + win[k].shape[0]]) for k in range(4))
        # agglomeration: gather owned planes into the full array on every rank
        full_ok = True
        for k in range(4):
            top = Z1 + (1 if (k == 2 and rank == ws - 1) else 0)
            mine = torch.from_numpy(np.ascontiguousarray(win[k][Z0 - W0:top - W0]))
            sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(ws)]
            dist.all_gather(sizes, torch.tensor([mine.shape[0]]))
            mx = max(int(s) for s in sizes)
            pad = torch.zeros((mx, mine.shape[1]), dtype=torch.float64)
            pad[:mine.shape[0]] = mine
            parts = [torch.zeros_like(pad) for _ in range(ws)]
            dist.all_gather(parts, pad)
            full = np.concatenate([p.numpy()[:int(s)] for p, s in zip(parts, sizes)])
            full_ok &= np.array_equal(full, glob[k])
        q.put((rank, bool(ok), bool(full_ok)))
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, False, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("ws,n2,nl,agg", [(2, 64, 4, 8), (3, 96, 3, 16)])
def test_ghost_exchange_and_gather_gloo(ws, n2, nl, agg):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, 6, 4, n2, nl, agg, q)) for r in range(ws)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(ws)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok and full for (_, ok, full) in res), res
