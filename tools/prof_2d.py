"""Per-kernel profile of one preconditioner application on a 2D grid
(development tool): python tools/prof_2d.py [--n 1024] [--levels 7]"""
import argparse
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2307_03242_b200 as E  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--levels", type=int, default=7)
    a = ap.parse_args()
    n = a.n
    g = E.StaggeredGrid((n, n), 1.0 / n)
    med = E.MediaModel.homogeneous(g, 2.0, 1.0, 1.0, 0.01)
    med.gamma = E.build_attenuation_profile(g, 0.01, E.SpongeConfig(32))
    opt = E.MgOptions(n_levels=a.levels, cycle="v", nu1=2, nu2=2, damping=0.25, vanka_mode="full",
                      sweep="red_black")
    mg = E.Multigrid(g, med, E.OperatorParams(2 / 3, 2 * math.pi * n / 10, 0.5), opt)
    r = torch.randn(g.n_dofs(), dtype=torch.complex128, device="cuda")
    z = torch.zeros_like(r)
    for _ in range(3):
        mg.precondition(r, z)
    torch.cuda.synchronize()
    st = torch.cuda.ExternalStream(mg.stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(10):
        mg.precondition(r, z)
    e1.record(st)
    torch.cuda.synchronize()
    print(f"V-cycle {e0.elapsed_time(e1) / 10:.3f} ms (graphs)")
    E.profile_enable(True)
    mg.precondition(r, z)
    torch.cuda.synchronize()
    rep = E.profile_report()
    E.profile_enable(False)
    tot = sum(t for (_, _, _, t) in rep)
    for name, lev, cnt, ms in sorted(rep, key=lambda t: -t[3])[:12]:
        print(f"{name:14s} L{lev}  x{cnt:3d}  {ms:8.3f} ms  avg {ms / cnt:7.4f}  {100 * ms / tot:5.1f}%")
    print(f"total {tot:.3f} ms")


if __name__ == "__main__":
    main()
