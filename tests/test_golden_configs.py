"""CPU: the configuration-level golden fixtures made by the reference's own
components (tests/golden/make_golden_configs.py, make_criterion5.py) are
present and self-consistent, and the C oracle's restated cycle reproduces the
reference's 5-level V(2,2) cycle at the bench parameters."""
import json
import os

import numpy as np

import paper_2307_03242_b200 as E
from oracle import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = np.load(os.path.join(HERE, "golden", "golden_configs.npz"))
C5 = json.load(open(os.path.join(HERE, "golden", "criterion5.json")))


def test_criterion5_reference_components_orderings():
    # test_acceptance.cpp:212-239: beta=2/3 at 10 ppw < 8 ppw < beta=1, graded 2/3 < 1
    assert all(C5[k]["status"] == "converged" for k in C5 if not k.startswith("_"))
    assert C5["slab_b23_g10"]["iterations"] < C5["slab_b23_g8"]["iterations"] < C5["slab_b1"]["iterations"]
    assert C5["slab_lin_b23"]["iterations"] < C5["slab_lin_b1"]["iterations"]


def test_config_goldens_converge_as_recorded():
    assert str(GOLD["c0_status"]) == "converged" and float(GOLD["c0_relres"]) <= 1e-6
    assert str(GOLD["c1_status"]) == "converged" and float(GOLD["c1_relres"]) <= 1e-6
    # the reference default shift (0.1) does not converge at 5 levels
    assert str(GOLD["c0_a01_status"]) != "converged"


def test_oracle_reproduces_reference_five_level_cycle():
    n = 64
    dims = (n, n, n)
    g = E.StaggeredGrid(dims, 1.0 / n)
    gam = E.build_attenuation_profile(g, 0.01, E.SpongeConfig(6))
    c = O.n_cells(dims)
    m = O.Media(np.full(c, 2.0), np.full(c, 1.0), np.full(c, 1.0), gam)
    rng = np.random.default_rng(64064)
    r = rng.uniform(-1, 1, O.n_dofs(dims)) + 1j * rng.uniform(-1, 1, O.n_dofs(dims))
    assert np.array_equal(r[:16], GOLD["cycle5_r_head"])
    z = O.MG(dims, 1.0 / n, m, 2 / 3, 2 * np.pi / (10.0 / n), 0.5, n_levels=5, cycle="v", nu1=2, nu2=2,
             damping=0.25).precondition(r)
    idx = GOLD["cycle5_idx"]
    assert np.abs(z[idx] - GOLD["cycle5_z"]).max() <= 1e-12 * np.abs(GOLD["cycle5_z"]).max()
