"""Mixed precision (experiments.hpp:241 MixedPrecondition; config
"precision": "mixed"): complex64 hierarchy behind complex128 FGMRES.

Parity: the reference's own float hierarchy (oracle/_ref, RefMGT<float>)
driven by the same double FGMRES gives the iteration count to match within
+-1; one mixed V-cycle agrees with the complex128 cycle to float accuracy
(relative 1e-5), which exercises the complex64 3D stencil, Vanka update,
transfers and coarsest inverse.
"""
import numpy as np
import pytest

import paper_2307_03242_b200 as E
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def problem(dims, seed=3):
    g = E.StaggeredGrid(dims, 1.0 / dims[-1])
    L = 8 if len(dims) == 2 else 4
    sp = E.SpongeConfig(L)
    med = E.layered_media(g, 0.01, seed)
    med.gamma = E.build_attenuation_profile(g, 0.01, sp)
    omega = E.omega_from_gs(g, med, 10.0, sp)
    return g, med, omega


@pytest.mark.parametrize("dims", [(64, 64), (32, 32, 32), (36, 20, 24), (64, 24, 20)])
def test_mixed_vcycle_close_to_double(dims):
    g, med, omega = problem(dims)
    opt = E.MgOptions(n_levels=3, cycle="v", nu1=2, nu2=2, damping=0.35, vanka_mode="full",
                      sweep="red_black")
    par = E.OperatorParams(2 / 3, omega, 0.5)
    rng = np.random.default_rng(7)
    r = rng.standard_normal(g.n_dofs()) + 1j * rng.standard_normal(g.n_dofs())
    zd = E.Multigrid(g, med, par, opt).precondition(r)
    mgm = E.Multigrid(g, med, par, opt, precision="mixed")
    zm = mgm.precondition(r)
    assert zm.dtype == np.complex128
    assert rel(zm, zd) < 1e-5
    assert not np.array_equal(zm, zd)  # really ran in float
    for _ in range(2):  # graph capture / replay of the mixed application
        assert np.array_equal(mgm.precondition(r), zm)


@pytest.mark.parametrize("dims", [(96, 64), (24, 20, 32)])
def test_mixed_fgmres_vs_reference_mixed(dims):
    g, med, omega = problem(dims)
    src = tuple(d // 2 for d in dims[:-1]) + (2,)
    b = E.make_point_source(g, len(dims), src)
    opt = E.MgOptions(n_levels=3, cycle="v", nu1=2, nu2=2, damping=0.35, vanka_mode="full",
                      sweep="red_black")
    mg = E.Multigrid(g, med, E.OperatorParams(2 / 3, omega, 0.5), opt, precision="mixed")
    D0 = E.make_opdata(g, med, E.OperatorParams(2 / 3, omega, 0.0))
    x = np.zeros(g.n_dofs(), complex)
    res = E.fgmres(D0, mg, b, x, E.KrylovOptions(restart=10, max_iterations=300))
    om = O.Media(med.lambda_, med.mu, med.rho, med.gamma)
    xr, info = O.ref_solve(dims, g.h, om, 2 / 3, omega, 0.5, b, n_levels=3, cycle="v", nu1=2, nu2=2,
                           damping=0.35, restart=10, max_iterations=300, precision="mixed")
    assert res.status == info["status"] == "converged"
    assert abs(res.iterations - info["iterations"]) <= 1
    r = E.residual(D0, b, x)
    assert np.linalg.norm(r) / np.linalg.norm(b) < 1e-6


def test_mixed_cycle_and_w_cycle():
    g, med, omega = problem((32, 16, 16))
    par = E.OperatorParams(2 / 3, omega, 0.5)
    rng = np.random.default_rng(11)
    b = rng.standard_normal(g.n_dofs()) + 1j * rng.standard_normal(g.n_dofs())
    x0 = rng.standard_normal(g.n_dofs()) * 1e-3 + 0j
    for cyc in ("v", "w"):
        opt = E.MgOptions(n_levels=3, cycle=cyc, nu1=1, nu2=1, damping=0.35, vanka_mode="full",
                          sweep="red_black")
        xd = E.Multigrid(g, med, par, opt).cycle(b, x0.copy())
        xm = E.Multigrid(g, med, par, opt, precision="mixed").cycle(b, x0.copy())
        assert rel(xm, xd) < 1e-5


def test_mixed_rejects_k_cycle_and_lexicographic():
    g, med, omega = problem((32, 32))
    par = E.OperatorParams(2 / 3, omega, 0.5)
    with pytest.raises(ValueError):
        E.Multigrid(g, med, par, E.MgOptions(n_levels=3, cycle="k", sweep="red_black"), precision="mixed")
    with pytest.raises(ValueError):
        E.Multigrid(g, med, par, E.MgOptions(n_levels=3, cycle="v", sweep="lexicographic"),
                    precision="mixed")
    with pytest.raises(ValueError):
        E.Multigrid(g, med, par, E.MgOptions(n_levels=3), precision="half")


def test_run_solve_mixed_layered():
    out = E.run_solve({"dims": [64, 32], "problem": "layered", "precision": "mixed", "levels": 3,
                       "cycle": "v", "nu1": 2, "nu2": 2, "sponge_cells": 8, "restart": 10,
                       "max_iterations": 300, "alpha": 0.5}, seed=5)
    assert out["precision"] == "mixed" and out["status"] == "converged"
