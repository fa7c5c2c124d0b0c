"""Exchange overhead of the one-slab-per-process path: 2 ranks sharing the
box's GPU (host barriers cannot deadlock; IPC-event waits are stream
semaphores, not spinning kernels), V(2,2) cycle time with the halo exchanges
ordered by CUDA IPC events vs by a stream drain + host barrier
(EHMG_EXCHANGE=event|host). Both ranks share one GPU, so the absolute times are
not a scaling measurement; the difference is the host round trips.

    python tools/dist_overhead.py [n_cells]
"""
import json
import os
import sys
import uuid

import numpy as np
import torch.multiprocessing as mp

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def rank_main(rank, ws, job, n, barrier, q):
    os.environ["EHMG_EXCHANGE"] = barrier
    try:
        import paper_2307_03242_b200 as E
        g = E.StaggeredGrid((n, n, n), 1.0 / n)
        med = E.MediaModel.homogeneous(g, 2.0, 1.0, 1.0, 0.01)
        med.gamma = E.build_attenuation_profile(g, 0.01, E.SpongeConfig(max(2, 24 * n // 256)))
        omega = 2 * np.pi * n / 10
        lv = max(2, int(round(np.log2(n))) - 3)
        opt = E.MgOptions(n_levels=lv, cycle="v", nu1=2, nu2=2, damping=0.25, vanka_mode="full",
                          sweep="red_black")
        d = E.DistributedSlabSolver(job, rank, ws, 0, g, med, E.OperatorParams(2 / 3, omega, 0.5), opt,
                                    agg_n2=max(8, n // 8))
        r = np.random.default_rng(3).standard_normal(g.n_dofs()) + 0j
        d.time_precondition(r, 3)
        ms = d.time_precondition(r, 10) / 10
        d.close()
        q.put((rank, ms, None))
    except Exception as e:
        q.put((rank, None, repr(e)))


def run(n, barrier, ws=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    job = f"ov{os.getpid()}_{uuid.uuid4().hex[:6]}"
    ps = [ctx.Process(target=rank_main, args=(k, ws, job, n, barrier, q)) for k in range(ws)]
    for p in ps:
        p.start()
    out = [q.get(timeout=900) for _ in range(ws)]
    for p in ps:
        p.join(timeout=60)
    errs = [e for _, _, e in out if e]
    if errs:
        raise RuntimeError(errs[0])
    return max(ms for _, ms, _ in out)


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    res = {"cells": n, "ranks_on_one_gpu": 2}
    for b in ("host", "event", "host", "event"):
        res.setdefault(b, []).append(round(run(n, b), 3))
    print(json.dumps(res))
