"""Time the preconditioner (graph-replayed V-cycle) and an FGMRES solve at
n^3 (bench media) in both precisions (development tool).

    python tools/time_cycle.py [--n 128]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2307_03242_b200 as E  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=128)
    a = ap.parse_args()
    g, med, omega = bench.build_problem(a.n, E)
    opt = E.MgOptions(n_levels=bench.levels_for(a.n), cycle="v", nu1=2, nu2=2, damping=bench.DAMPING,
                      vanka_mode="full", sweep="red_black")
    A = E.make_opdata(g, med, E.OperatorParams(bench.BETA, omega, 0.0))
    b = torch.from_numpy(E.make_point_source(g, 0, (a.n // 2,) * 3)).cuda()
    for prec in ("double", "mixed"):
        mg = E.Multigrid(g, med, E.OperatorParams(bench.BETA, omega, bench.ALPHA), opt, precision=prec)
        r = torch.randn_like(b)
        z = torch.zeros_like(b)
        for _ in range(3):
            mg.precondition(r, z)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(20):
            mg.precondition(r, z)
        torch.cuda.synchronize()
        tc = (time.perf_counter() - t0) / 20
        out = {"n": a.n, "precision": prec, "cycle_ms": round(tc * 1e3, 3)}
        for orth in ("classical", "modified", "classical", "modified"):
            x = torch.zeros_like(b)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = E.fgmres(A, mg, b, x, E.KrylovOptions(restart=10, max_iterations=600, orthogonalization=orth))
            torch.cuda.synchronize()
            ts = time.perf_counter() - t0
            out[orth + ("" if orth not in out else "_2")] = {"iterations": res.iterations, "seconds": round(ts, 3),
                         "ms_per_iteration": round(ts / max(1, res.iterations) * 1e3, 3)}
        print(json.dumps(out), flush=True)
        del mg


if __name__ == "__main__":
    main()
