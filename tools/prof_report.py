"""Per-kernel CUDA-event profile of one preconditioner application at n^3
(bench media), double or mixed precision (development tool).

    python tools/prof_report.py [--n 256] [--precision double|mixed]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2307_03242_b200 as E  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--precision", default="double")
    a = ap.parse_args()
    g, med, omega = bench.build_problem(a.n, E)
    opt = E.MgOptions(n_levels=bench.levels_for(a.n), cycle="v", nu1=2, nu2=2, damping=bench.DAMPING,
                      vanka_mode="full", sweep="red_black")
    mg = E.Multigrid(g, med, E.OperatorParams(bench.BETA, omega, bench.ALPHA), opt,
                     precision=a.precision)
    N = g.n_dofs()
    r = torch.randn(N, dtype=torch.complex128, device="cuda")
    z = torch.zeros_like(r)
    for _ in range(2):
        mg.precondition(r, z)
    torch.cuda.synchronize()
    E.profile_enable(True)
    mg.precondition(r, z)
    torch.cuda.synchronize()
    rep = E.profile_report()
    E.profile_enable(False)
    tot = sum(t for (_, _, _, t) in rep)
    for name, lev, cnt, ms in sorted(rep, key=lambda t: -t[3]):
        print(f"{name:14s} L{lev}  x{cnt:3d}  {ms:8.3f} ms  avg {ms / cnt:7.4f}  {100 * ms / tot:5.1f}%")
    print(f"total {tot:.3f} ms")


if __name__ == "__main__":
    main()
