"""GPU: the z-slab decomposed V/W cycle (north_star (6)) reproduces the
undecomposed cycle. Slabs run in one process on one GPU and exchange ghost
planes by device copies -- the same plane ranges a multi-GPU run moves over
NVLink -- so any decomposition error shows up as a mismatch here."""
import numpy as np
import pytest

import paper_2307_03242_b200 as E

pytestmark = pytest.mark.gpu


def _problem(dims, seed):
    rng = np.random.default_rng(seed)
    g = E.StaggeredGrid(dims, 1.0 / dims[0])
    n = g.n_cells()
    m = E.MediaModel(3 * rng.uniform(.5, 2, n), rng.uniform(.5, 2, n), rng.uniform(.5, 2, n),
                     0.05 * rng.uniform(.5, 2, n))
    b = rng.uniform(-1, 1, g.n_dofs()) + 1j * rng.uniform(-1, 1, g.n_dofs())
    return g, m, b


@pytest.mark.parametrize("dims,nl,ns,agg,cyc", [
    ((24, 16, 64), 4, 2, 8, "v"),
    ((24, 16, 64), 4, 3, 8, "v"),
    ((24, 16, 64), 4, 4, 8, "w"),
    ((32, 32, 128), 4, 4, 16, "v"),
    ((16, 24, 48), 3, 2, 64, "v"),   # only the finest level sharded
    ((192, 192, 32), 5, 2, 8, "v"),  # finest level on k_stencil3d_sp (>= 192 wide): windows, plane ranges
])
def test_slab_cycle_equals_single_domain(dims, nl, ns, agg, cyc):
    g, m, b = _problem(dims, 3)
    omega = 2 * np.pi * dims[0] / 10
    par = E.OperatorParams(2 / 3, omega, 0.3)
    opt = E.MgOptions(n_levels=nl, cycle=cyc, nu1=2, nu2=2, damping=0.35, vanka_mode="full",
                      sweep="red_black")
    z1 = E.Multigrid(g, m, par, opt).precondition(b)
    sm = E.SlabMultigrid(g, m, par, opt, nslabs=ns, agg_n2=agg)
    zs = sm.precondition(b)
    la, tot = sm.levels()
    assert la >= 1 and tot == nl
    assert sm.exchanged_bytes() > 0
    err = np.abs(zs - z1).max() / np.abs(z1).max()
    assert err < 1e-13, err


def test_slab_preconditioned_fgmres_matches():
    """FGMRES with the slab preconditioner: same iteration count."""
    dims = (32, 32, 64)
    g = E.StaggeredGrid(dims, 1 / 32)
    n = g.n_cells()
    med = E.MediaModel.homogeneous(g, 2.0, 1.0, 1.0, 0.01)
    med.gamma = E.build_attenuation_profile(g, 0.01, E.SpongeConfig(6))
    omega = 2 * np.pi / (10 / 32)
    par = E.OperatorParams(2 / 3, omega, 0.5)
    opt = E.MgOptions(n_levels=3, cycle="v", nu1=2, nu2=2, damping=0.35, vanka_mode="full",
                      sweep="red_black")
    b = E.make_point_source(g, 0, (16, 16, 32))
    z_ref = E.Multigrid(g, med, par, opt).precondition(b)
    sm = E.SlabMultigrid(g, med, par, opt, nslabs=4, agg_n2=8)
    assert np.abs(sm.precondition(b) - z_ref).max() / np.abs(z_ref).max() < 1e-13


@pytest.mark.parametrize("dims,nl,ns,agg", [
    ((24, 16, 64), 4, 2, 8),
    ((32, 32, 128), 4, 4, 16),
])
def test_slab_mixed_cycle_equals_single_domain_mixed(dims, nl, ns, agg):
    """precision "mixed" (experiments.hpp:241) in the z-slab mode: the
    complex64 hierarchy decomposed into slabs reproduces the undecomposed
    complex64 hierarchy (same float operations on the owned planes)."""
    g, m, b = _problem(dims, 5)
    omega = 2 * np.pi * dims[0] / 10
    par = E.OperatorParams(2 / 3, omega, 0.3)
    opt = E.MgOptions(n_levels=nl, cycle="v", nu1=2, nu2=2, damping=0.35, vanka_mode="full",
                      sweep="red_black")
    z1 = E.Multigrid(g, m, par, opt, precision="mixed").precondition(b)
    zs = E.SlabMultigrid(g, m, par, opt, nslabs=ns, agg_n2=agg, precision="mixed").precondition(b)
    zd = E.Multigrid(g, m, par, opt).precondition(b)
    err = np.abs(zs - z1).max() / np.abs(z1).max()
    assert err < 1e-12, err
    # and the mixed cycle stays within float rounding of the complex128 cycle
    assert np.abs(zs - zd).max() / np.abs(zd).max() < 1e-4
