"""Short driver for ncu captures of the hot kernels at the bench size.

    python tools/prof_kernels.py [--n 256] [--what apply|cycle|solve]
"""
import argparse
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2307_03242_b200 as E  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--what", default="apply")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    n = a.n
    g = E.StaggeredGrid((n, n, n), 1.0 / n)
    med = E.MediaModel.homogeneous(g, 2.0, 1.0, 1.0, 0.01)
    med.gamma = E.build_attenuation_profile(g, 0.01, E.SpongeConfig(min(24, n // 4)))
    omega = 2 * math.pi / (10 / n)
    N = g.n_dofs()
    r = torch.randn(N, dtype=torch.complex128, device="cuda")
    y = torch.empty_like(r)
    bvec = torch.randn(N, dtype=torch.complex128, device="cuda")  # distinct b: no L2 reuse of x
    if a.what == "apply":
        D = E.make_opdata(g, med, E.OperatorParams(2 / 3, omega, 0.5))
        for _ in range(a.reps):
            E.residual(D, bvec, r, y)
    else:
        opt = E.MgOptions(n_levels=5 if n >= 64 else 3, cycle="v", nu1=2, nu2=2, damping=0.25,
                          vanka_mode="full", sweep="red_black")
        mg = E.Multigrid(g, med, E.OperatorParams(2 / 3, omega, 0.5), opt)
        if a.what == "solve":  # a few FGMRES iterations (MGS passes, scale/copy, restart update)
            D0 = E.make_opdata(g, med, E.OperatorParams(2 / 3, omega, 0.0))
            b = E.make_point_source(g, 0, (n // 2, n // 2, n // 2))
            x = b * 0
            E.fgmres(D0, mg, b, x, E.KrylovOptions(restart=10, max_iterations=4 * a.reps))
        else:
            for _ in range(a.reps):
                mg.precondition(r, y)
    torch.cuda.synchronize()
    print("ok", float(y.abs().max()))


if __name__ == "__main__":
    main()
