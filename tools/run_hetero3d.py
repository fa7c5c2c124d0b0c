"""configs[3]-style heterogeneous 3D solve on one GPU (development check):
layered media from the reference's builder (experiments.hpp:78) with a seed,
10 points per wavelength at the minimum shear speed, source near the top,
FGMRES(10) + V(2,2) to 1e-6 in complex128 and with the complex64 hierarchy;
prints iterations, time and the true relative residual.

    python tools/run_hetero3d.py [--n 256] [--levels 5]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2307_03242_b200 as E  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--levels", type=int, default=5)
    ap.add_argument("--seed", type=int, default=2023)
    a = ap.parse_args()
    n = a.n
    g = E.StaggeredGrid((n, n, n), 1.0 / n)
    sp = E.SpongeConfig(32 if n >= 256 else max(4, n // 8))
    med = E.layered_media(g, 0.01, a.seed)
    med.gamma = E.build_attenuation_profile(g, 0.01, sp)
    omega = E.omega_from_gs(g, med, 10.0, sp)
    par = E.OperatorParams(2 / 3, omega, 0.5)
    opt = E.MgOptions(n_levels=a.levels, cycle="v", nu1=2, nu2=2, damping=0.25, vanka_mode="full",
                      sweep="red_black")
    b = E.make_point_source(g, 2, (n // 2, n // 2, n - n // 8))
    bd = torch.from_numpy(b).cuda()
    A = E.make_opdata(g, med, E.OperatorParams(2 / 3, omega, 0.0))
    out = {"config": f"3D layered (seed {a.seed}) {n + 1}^3 nodes, {a.levels} levels, omega {omega:.1f}"}
    for prec in ("double", "mixed"):
        mg = E.Multigrid(g, med, par, opt, precision=prec)
        # warm: lazy per-kernel setup and graph capture stay out of the timing
        E.fgmres(A, mg, bd, torch.zeros_like(bd), E.KrylovOptions(restart=10, max_iterations=3))
        x = torch.zeros_like(bd)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = E.fgmres(A, mg, bd, x, E.KrylovOptions(restart=10, max_iterations=1500))
        torch.cuda.synchronize()
        ts = time.perf_counter() - t0
        r = bd - E.apply_mixed_operator(A, x)
        true_rel = float(r.abs().pow(2).sum().sqrt() / bd.abs().pow(2).sum().sqrt())
        out[prec] = {"status": res.status, "iterations": res.iterations, "relres": res.relres,
                     "true_relres": true_rel, "seconds": round(ts, 3)}
        del mg
    print(json.dumps(out))


if __name__ == "__main__":
    main()
