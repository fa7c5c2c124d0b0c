"""BASELINE configs[0..3] through the public API on the GPU (the workloads
pinned in paper_2307_03242_b200/configs.py), one FGMRES(10) + V(2,2) solve
each, with the reference CPU cycle timed beside configs[0] (a bounded sample).

    python tools/run_configs.py [--which 0,1,2,3] [--scale 1] [--no-ref]

Prints one JSON object per config.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2307_03242_b200 as E  # noqa: E402
from paper_2307_03242_b200 import configs as K  # noqa: E402


def solve(w, max_it):
    t0 = time.perf_counter()
    mg = E.Multigrid(w.grid, w.media, w.shifted, w.mg)
    D0 = E.make_opdata(w.grid, w.media, w.unshifted)
    setup = time.perf_counter() - t0
    b = w.rhs(0)
    x = np.zeros(w.grid.n_dofs(), np.complex128)
    E.fgmres(D0, mg, b, x.copy(), E.KrylovOptions(restart=10, max_iterations=5))  # warm (graphs)
    t0 = time.perf_counter()
    res = E.fgmres(D0, mg, b, x, E.KrylovOptions(restart=10, max_iterations=max_it))
    ts = time.perf_counter() - t0
    return {"status": res.status, "iterations": res.iterations, "relres": res.relres,
            "seconds": round(ts, 3), "setup_s": round(setup, 3)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--which", default="0,1")
    ap.add_argument("--scale", type=int, default=1)
    ap.add_argument("--max-it", type=int, default=4000)
    ap.add_argument("--no-ref", action="store_true")
    a = ap.parse_args()
    for i in [int(v) for v in a.which.split(",")]:
        w = K.CONFIGS[i](scale=a.scale)
        g = w.grid
        out = {"config": w.name, "dims": list(g.dims), "levels": w.mg.n_levels, "omega": w.shifted.omega,
               "alpha": w.shifted.alpha, "damping": w.mg.damping, "source": w.notes,
               "b200": solve(w, a.max_it)}
        if i == 0 and not a.no_ref:
            from oracle import oracle as O
            m = w.media
            b = w.rhs(0)
            ncyc = 3
            _, secs = O.ref_mg_cycles(g.dims, g.h, O.Media(m.lambda_, m.mu, m.rho, m.gamma), w.shifted.beta,
                                      w.shifted.omega, w.shifted.alpha, b, np.zeros_like(b), ncycles=ncyc,
                                      n_levels=w.mg.n_levels, cycle="v", nu1=2, nu2=2, damping=w.mg.damping,
                                      vanka="full", sweep="red_black")
            per = secs / ncyc
            it = out["b200"]["iterations"]
            out["reference_cpu"] = {"v_cycle_s": round(per, 4), "cores": 1,
                                    "solve_s_extrapolated": round(per * it, 2),
                                    "sample": f"{ncyc} V(2,2) cycles of oracle/_ref at the same size; "
                                              f"x {it} iterations (cycle cost only, 1 core)"}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
