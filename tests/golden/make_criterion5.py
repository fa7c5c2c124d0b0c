"""Golden fixture: the reference's acceptance criterion 5
(/root/reference/proj/tests/test_acceptance.cpp:212-239) run through the
reference's OWN components (oracle/_ref: operator, Vanka, transfers, FGMRES,
restated W-cycle, exact coarsest solve -- banded LU for the 49K-DOF coarse
grid since Eigen's SparseLU is absent) with run_solve's defaults
(experiments.hpp:258-330): 512x128 slab, two levels, W(1,1) full red-black
Vanka, FGMRES(5), pressure point source at middle_of_top_row, alpha 0.1,
default damping, lambda 20 mu 1 rho 1 (homogeneous) or linear media.

    python tests/golden/make_criterion5.py   # ~10-20 min on 5 cores

Writes tests/golden/criterion5.json (iterations, status, relres per case).
"""
import json
import math
import os
import sys
from concurrent.futures import ProcessPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

CASES = [("slab_b1", 1.0, 10.0, "homogeneous"), ("slab_b23_g10", 2 / 3, 10.0, "homogeneous"),
         ("slab_b23_g8", 2 / 3, 8.0, "homogeneous"), ("slab_lin_b23", 2 / 3, 10.0, "linear"),
         ("slab_lin_b1", 1.0, 10.0, "linear")]
DIMS = (512, 128)


def media(problem):
    """experiments.hpp:60 linear_media / MediaModel::homogeneous, gamma from the
    20-cell sponge (media.hpp:95) -- built with the oracle's restatements."""
    from oracle import oracle as O
    n0, n1 = DIMS
    n = n0 * n1
    if problem == "homogeneous":
        lam, mu, rho = np.full(n, 20.0), np.full(n, 1.0), np.full(n, 1.0)
    else:
        t = ((np.arange(n) // n0) + 0.5) / n1
        rho, lam, mu = 2 + t, 4 + 16 * t, 1 + 14 * t
    gam = O.attenuation(DIMS, 0.01, 20)
    return O.Media(lam, mu, rho, gam)


def min_interior_vs(m, L=20):
    n0, n1 = DIMS
    vs = np.sqrt(m.mu / m.rho).reshape(n1, n0)
    inner = vs[:n1 - L, L:n0 - L]  # top is free (absorb_top = false)
    return inner.min() if inner.size else vs.min()


def run(case):
    from oracle import oracle as O
    tag, beta, gs, problem = case
    m = media(problem)
    h = 1.0 / DIMS[1]
    omega = 2 * math.pi * min_interior_vs(m) / (gs * h)
    w = (0.55 if gs >= 9 else 0.5)  # experiments.hpp:221, two levels
    b = np.zeros(O.n_dofs(DIMS), np.complex128)
    # pressure point source (component Dim) at middle_of_top_row: cell (n0/2, 0), 1/h^2
    off = (DIMS[0] + 1) * DIMS[1] + DIMS[0] * (DIMS[1] + 1)
    b[off + DIMS[0] // 2] = 1.0 / (h * h)
    _, info = O.ref_solve(DIMS, h, m, beta, omega, 0.1, b, n_levels=2, cycle="w", nu1=1, nu2=1, damping=w,
                          restart=5, max_iterations=600)
    return tag, {"beta": beta, "g_s": gs, "problem": problem, "omega": omega, "damping": w,
                 "iterations": info["iterations"], "status": info["status"], "relres": info["relres"]}


if __name__ == "__main__":
    with ProcessPoolExecutor(len(CASES)) as ex:
        out = dict(ex.map(run, CASES))
    out["_source"] = ("oracle/_ref (reference headers) with a banded exact coarsest LU; "
                      "tests/golden/make_criterion5.py")
    with open(os.path.join(HERE, "criterion5.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))
