"""Host-side media builders of the library (no GPU needed).

layered_media restates experiments.hpp:78 with the same std::mt19937_64 /
<random> draws; experiments.hpp itself cannot be compiled here (it needs
nlohmann/json and Eigen's dense module through lfa.hpp), so these tests pin
the builder by the reference's stated contract instead of its binary output:
5..10 layers starting at depth 0, per-layer vs in [0.5, 2], rho in [1.5, 3],
lambda/mu in [2, 20], mu = rho vs^2, determinism per seed.
"""
import numpy as np
import pytest

import paper_2307_03242_b200 as E


@pytest.mark.parametrize("dims", [(16, 40), (8, 6, 40), (4, 4, 12)])
@pytest.mark.parametrize("seed", [1, 7, 2024])
def test_layered_media_contract(dims, seed):
    g = E.StaggeredGrid(dims, 1.0 / dims[-1])
    m = E.layered_media(g, 0.01, seed)
    nd = dims[-1]
    shape = dims[::-1]
    rho = m.rho.reshape(shape)
    lam = m.lambda_.reshape(shape)
    mu = m.mu.reshape(shape)
    # horizontal layers: every depth plane is constant
    for arr in (rho, lam, mu):
        flat = arr.reshape(nd, -1)
        assert np.all(flat == flat[:, :1])
    col_r, col_l, col_m = rho.reshape(nd, -1)[:, 0], lam.reshape(nd, -1)[:, 0], mu.reshape(nd, -1)[:, 0]
    tops = [0] + [z for z in range(1, nd) if (col_r[z], col_l[z], col_m[z]) != (col_r[z - 1], col_l[z - 1], col_m[z - 1])]
    assert 5 <= len(tops) <= 10  # every dims here has >= 10 planes
    vs = np.sqrt(col_m / col_r)
    assert np.all((vs >= 0.5 - 1e-12) & (vs <= 2.0 + 1e-12))
    assert np.all((col_r >= 1.5) & (col_r <= 3.0))
    q = col_l / col_m
    assert np.all((q >= 2.0 - 1e-12) & (q <= 20.0 + 1e-12))
    assert np.all(m.gamma == 0.01)
    m2 = E.layered_media(g, 0.01, seed)
    assert np.array_equal(m.rho, m2.rho) and np.array_equal(m.lambda_, m2.lambda_)


def test_layered_media_seed_changes_layers():
    g = E.StaggeredGrid((8, 64), 1 / 64)
    a = E.layered_media(g, 0.0, 1)
    b = E.layered_media(g, 0.0, 2)
    assert not np.array_equal(a.rho, b.rho)


def test_layered_media_layer_count_range():
    # over many seeds the layer count spans the reference's 5..10 draw
    g = E.StaggeredGrid((2, 200), 1 / 200)
    counts = set()
    for seed in range(60):
        r = E.layered_media(g, 0.0, seed).rho.reshape(200, 2)[:, 0]
        counts.add(1 + int(np.count_nonzero(np.diff(r))))
    assert min(counts) >= 5 and max(counts) <= 10
    assert counts == set(range(5, 11))


def test_run_solve_rejects_unknown_problem():
    with pytest.raises(ValueError):
        E.run_solve({"dims": [16, 16], "problem": "nope"})
