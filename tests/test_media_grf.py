"""BASELINE configs[1]/[3]/[4] media recipe: layered + smooth Gaussian random
field perturbations (csrc/ehmg_media.cuh; C restatement
oracle/ehmg_oracle.c:og_layered_grf_media).

CPU: the restated recipe's contract -- horizontal layers on the last axis
starting at depth 0, per-layer values inside the BASELINE ranges, factors
inside +-perturbation, unit-variance smooth fields with the stated
correlation, determinism per seed. GPU: the library's device builder equals
the C restatement bit for bit."""
import numpy as np
import pytest

from oracle import oracle as O

CS, Q, RHO = (1.0, 2.5), (1.7, 2.2), (1.0, 2.5)


def _fields(m):
    lam, mu, rho, gam = m.arrays()
    cs = np.sqrt(mu / rho)
    q = np.sqrt((lam + 2 * mu) / mu)
    return cs, q, rho, gam


@pytest.mark.parametrize("dims", [(48, 40), (12, 10, 24)])
def test_recipe_layers_and_ranges(dims):
    m = O.layered_grf_media(dims, 11, n_layers=8, corr_cells=4)
    cs, q, rho, gam = _fields(m)
    assert cs.min() >= CS[0] * 0.9 - 1e-12 and cs.max() <= CS[1] * 1.1 + 1e-12
    assert q.min() >= Q[0] * 0.9 - 1e-12 and q.max() <= Q[1] * 1.1 + 1e-12
    assert rho.min() >= RHO[0] * 0.9 - 1e-12 and rho.max() <= RHO[1] * 1.1 + 1e-12
    assert np.all(gam == 0.01)
    # without perturbation: horizontal layers, 8 distinct depth bands, top = 0
    m0 = O.layered_grf_media(dims, 11, n_layers=8, perturbation=0.0, corr_cells=4)
    cs0 = _fields(m0)[0].reshape(dims[::-1]).reshape(dims[-1], -1)
    assert np.all(cs0 == cs0[:, :1])
    col = cs0[:, 0]
    assert 1 + np.count_nonzero(np.diff(col)) == 8
    # the perturbation factor of every cell stays within +-10% of its layer value
    f = _fields(m)[0].reshape(dims[::-1]).reshape(dims[-1], -1) / cs0
    assert np.abs(f - 1).max() < 0.1


def test_recipe_deterministic_and_seeded():
    a = O.layered_grf_media((32, 24), 5, corr_cells=3).arrays()
    b = O.layered_grf_media((32, 24), 5, corr_cells=3).arrays()
    c = O.layered_grf_media((32, 24), 6, corr_cells=3).arrays()
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    assert not np.array_equal(a[1], c[1])


def test_grf_unit_variance_and_correlation_length():
    # single-valued ranges: cs = factor, so the field g is recoverable
    n, corr = 256, 8.0
    m = O.layered_grf_media((n, n), 3, n_layers=1, cs=(1.0, 1.0), cp_over_cs=(2.0, 2.0), rho=(1.0, 1.0),
                            perturbation=0.5, corr_cells=corr)
    y = (_fields(m)[0] - 1.0) / 0.5
    g = (y / np.sqrt(1 - y * y)).reshape(n, n)
    assert abs(g.std() - 1.0) < 0.15 and abs(g.mean()) < 0.25
    # covariance exp(-r^2 / corr^2): lag corr/2 -> e^-0.25, lag corr -> e^-1
    for lag, want in [(int(corr / 2), np.exp(-0.25)), (int(corr), np.exp(-1.0))]:
        rho_x = np.mean(g[:, :-lag] * g[:, lag:]) / g.var()
        rho_y = np.mean(g[:-lag, :] * g[lag:, :]) / g.var()
        assert abs(rho_x - want) < 0.1 and abs(rho_y - want) < 0.1


@pytest.mark.gpu
@pytest.mark.parametrize("dims,corr,seed", [((64, 48), 6.0, 3), ((20, 16, 24), 3.0, 5), ((33, 18), 20.0, 2023)])
def test_device_builder_matches_restatement(dims, corr, seed):
    import paper_2307_03242_b200 as E
    g = E.StaggeredGrid(dims, 1.0 / dims[0])
    m = E.layered_grf_media(g, seed, corr_cells=corr, gamma_phys=0.02)
    r = O.layered_grf_media(dims, seed, corr_cells=corr, gamma_phys=0.02)
    for got, want in zip((m.lambda_, m.mu, m.rho, m.gamma), r.arrays()):
        assert np.array_equal(got, want)


def test_device_builder_validates_before_touching_the_device():
    import paper_2307_03242_b200 as E
    g = E.StaggeredGrid((16, 12), 1 / 16)
    with pytest.raises(ValueError, match="cp/cs must stay above sqrt"):
        E.layered_grf_media(g, 1, cp_over_cs=(1.2, 2.0))
    with pytest.raises(ValueError, match="1..64 layers"):
        E.layered_grf_media(g, 1, n_layers=0)
    with pytest.raises(ValueError, match="corr in"):
        E.layered_grf_media(g, 1, corr_cells=0.0)
