"""Generate golden vectors from the REFERENCE itself (oracle/_ref, i.e. the
unmodified reference headers compiled by oracle/Makefile).

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
Writes tests/golden/golden.npz. The fixtures pin the C oracle (CPU tests)
and the CUDA path (GPU tests) to the reference's own outputs.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def media(rng, dims, gscale=0.05):
    n = O.n_cells(dims)
    return O.Media(3 * rng.uniform(0.5, 2, n), rng.uniform(0.5, 2, n), rng.uniform(0.5, 2, n),
                   gscale * rng.uniform(0.5, 2, n))


def field(rng, n):
    return rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)


def main():
    rng = np.random.default_rng(20230707)
    out = {}
    cases = []
    # operator apply across the parameter matrix (test_operator.cpp:58)
    for dims, beta, omega, alpha in [((9, 7), 1.0, 9.7, 0.2), ((9, 7), 2 / 3, 9.7, 0.0),
                                     ((9, 7), 0.5, 0.0, 0.2), ((12, 10), 2 / 3, 9.7, 0.2),
                                     ((5, 4, 6), 2 / 3, 6.1, 0.15), ((5, 4, 6), 1.0, 6.1, 0.0),
                                     ((6, 6, 4), 0.5, 4.0, 0.3)]:
        m = media(rng, dims)
        h = 1.0 / dims[0]
        x = field(rng, O.n_dofs(dims))
        y = O.ref_apply(dims, h, m, beta, omega, alpha, x)
        ys = O.ref_apply(dims, h, m, beta, omega, alpha, x, schur=True)
        cases.append(("apply", dims, h, m, (beta, omega, alpha), dict(x=x, y=y, ys=ys)))
    # Vanka: both modes, both orders, 2D and 3D (test_smoothers.cpp:157)
    for dims, mode, order in [((6, 5), 0, 0), ((6, 5), 0, 1), ((6, 5), 1, 0), ((6, 5), 1, 1),
                              ((4, 4, 4), 0, 0), ((4, 4, 4), 1, 1), ((4, 4, 6), 0, 1)]:
        m = media(rng, dims, 0.0)
        h = 1.0 / dims[0]
        b, x = field(rng, O.n_dofs(dims)), field(rng, O.n_dofs(dims))
        xs, cache = O.ref_vanka(dims, h, m, 2 / 3, 4.5, 0.15, mode, order, 0.8, 2, b, x)
        cases.append(("vanka", dims, h, m, (2 / 3, 4.5, 0.15),
                      dict(b=b, x=x, xs=xs, cache=cache.ravel(), mode=mode, order=order, w=0.8,
                           nsweeps=2)))
    # transfers (test_transfer.cpp)
    for dims in [(8, 6), (8, 8), (4, 6, 4), (8, 4, 6)]:
        xf = field(rng, O.n_dofs(dims))
        dc = [d // 2 for d in dims]
        xc = field(rng, O.n_dofs(dc))
        cases.append(("transfer", dims, 1.0, None, None,
                      dict(xf=xf, xc=xc, r=O.ref_transfer(dims, True, xf),
                           p=O.ref_transfer(dims, False, xc))))
    # media coarsening + sponge profile
    for dims in [(8, 6), (4, 6, 4)]:
        v = rng.uniform(0.5, 2, O.n_cells(dims))
        cases.append(("coarsen", dims, 1.0, None, None, dict(v=v, c=O.ref_coarsen(dims, v))))
    for dims, L, top in [((48, 44), 20, False), ((30, 30, 30), 8, True), ((30, 30, 30), 8, False)]:
        cases.append(("sponge", dims, 1.0, None, None,
                      dict(L=L, top=int(top), g=O.ref_attenuation(dims, 0.01, L, 1.0, top))))
    # multigrid cycles (V, W; full red-black and economic lexicographic)
    for dims, nl, cyc, vmode, sweep, nu in [((16, 16), 3, "v", "full", "red_black", 2),
                                           ((16, 8), 2, "w", "economic", "lexicographic", 1),
                                           ((16, 16), 3, "w", "full", "red_black", 1),
                                           ((8, 8, 8), 2, "v", "full", "red_black", 2),
                                           ((16, 8, 8), 3, "v", "full", "red_black", 1)]:
        m = media(rng, dims)
        h = 1.0 / dims[0]
        omega = 2 * np.pi * dims[0] / 10
        b = field(rng, O.n_dofs(dims))
        x0 = np.zeros_like(b)
        x1, _ = O.ref_mg_cycles(dims, h, m, 2 / 3, omega, 0.3, b, x0, ncycles=2, n_levels=nl,
                                cycle=cyc, nu1=nu, nu2=nu, damping=0.55, vanka=vmode, sweep=sweep)
        cases.append(("mg", dims, h, m, (2 / 3, omega, 0.3),
                      dict(b=b, x=x1, nl=nl, cyc=cyc, vmode=vmode, sweep=sweep, nu=nu)))
    # full FGMRES solves: point source, sponge, V(2,2) preconditioner
    for dims, nl, alpha, w, beta in [((32, 32), 3, 0.3, 0.35, 2 / 3), ((64, 32), 2, 0.1, 0.55, 1.0),
                                     ((16, 16, 16), 2, 0.3, 0.55, 2 / 3)]:
        n = O.n_cells(dims)
        L = 4
        gam = O.ref_attenuation(dims, 0.01, L)
        m = O.Media(np.full(n, 2.0), np.ones(n), np.ones(n), gam)
        h = 1.0 / dims[-1]
        omega = 2 * np.pi / (10 * h)
        b = np.zeros(O.n_dofs(dims), complex)
        nd = len(dims)
        idx = [d // 2 for d in dims[:-1]] + [0]
        cs = [int(np.prod(s)) for s in O.comp_shapes(dims)]
        lin = idx[-1]
        for a in range(nd - 2, -1, -1):
            lin = lin * dims[a] + idx[a]
        b[sum(cs[:nd]) + lin] = 1.0 / h ** nd
        x, info = O.ref_solve(dims, h, m, beta, omega, alpha, b, n_levels=nl, cycle="v", nu1=2,
                              nu2=2, damping=w, restart=10)
        cases.append(("solve", dims, h, m, (beta, omega, alpha),
                      dict(b=b, x=x, nl=nl, w=w, iterations=info["iterations"],
                           status=info["status"], relres=info["relres"],
                           history=np.array(info["history"]))))
    for i, (kind, dims, h, m, par, data) in enumerate(cases):
        p = f"c{i:02d}_"
        out[p + "kind"] = np.array(kind)
        out[p + "dims"] = np.array(dims)
        out[p + "h"] = np.array(h)
        if m is not None:
            for nm, a in zip(("lam", "mu", "rho", "gam"), m.arrays()):
                out[p + nm] = a
        if par is not None:
            out[p + "par"] = np.array(par)
        for k, v in data.items():
            out[p + k] = np.asarray(v)
    np.savez_compressed(OUT, **out)
    print(f"wrote {len(cases)} cases to {OUT} ({os.path.getsize(OUT) / 1e6:.2f} MB)")


if __name__ == "__main__":
    main()
