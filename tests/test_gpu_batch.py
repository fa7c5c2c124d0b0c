"""GPU: the pipelined batch preconditioner (ehmg_multigrid_precondition_many)
returns exactly what one synchronous precondition() call per right-hand side
returns, in complex128 and in the mixed-precision hierarchy, with repeated
output buffers written in order."""
import numpy as np
import pytest

import paper_2307_03242_b200 as E

pytestmark = pytest.mark.gpu


def _mg(precision):
    dims = (32, 32, 32)
    g = E.StaggeredGrid(dims, 1 / 32)
    med = E.MediaModel.homogeneous(g, 2.0, 1.0, 1.0, 0.01)
    med.gamma = E.build_attenuation_profile(g, 0.01, E.SpongeConfig(6))
    par = E.OperatorParams(2 / 3, 2 * np.pi / (10 / 32), 0.5)
    opt = E.MgOptions(n_levels=3, cycle="v", nu1=2, nu2=2, damping=0.35, vanka_mode="full",
                      sweep="red_black")
    return g, E.Multigrid(g, med, par, opt, precision=precision)


@pytest.mark.parametrize("precision", ["double", "mixed"])
def test_precondition_many_equals_single_calls(precision):
    g, mg = _mg(precision)
    rng = np.random.default_rng(11)
    n = g.n_dofs()
    rs = [rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n) for _ in range(5)]
    ref = [mg.precondition(r) for r in rs]
    zs = mg.precondition_many(rs)
    for a, b in zip(zs, ref):
        assert np.array_equal(a, b)
    # two outputs reused in turn: the last two right-hand sides' results remain
    out = [np.zeros(n, np.complex128) for _ in range(2)]
    mg.precondition_many(rs, [out[i & 1] for i in range(len(rs))])
    assert np.array_equal(out[0], ref[4]) and np.array_equal(out[1], ref[3])


def test_precondition_many_rejects_mismatch():
    g, mg = _mg("double")
    n = g.n_dofs()
    with pytest.raises(ValueError):
        mg.precondition_many([np.zeros(n, np.complex128)], [])
