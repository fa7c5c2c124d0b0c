"""Small operator applies / residuals through both complex128 3D kernels, for
compute-sanitizer runs (memcheck / racecheck) on a B200:

    compute-sanitizer --tool memcheck python tools/sanitize_stencil.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2307_03242_b200 as E  # noqa: E402


def main():
    rng = np.random.default_rng(0)
    for dims in [(200, 196, 6), (40, 24, 12)]:  # k_stencil3d_sp, k_stencil3d_rr
        n = int(np.prod(dims))
        g = E.StaggeredGrid(dims, 1.0 / dims[0])
        med = E.MediaModel(3 * rng.uniform(.5, 2, n), rng.uniform(.5, 2, n), rng.uniform(.5, 2, n),
                           0.05 * rng.uniform(.5, 2, n))
        D = E.make_opdata(g, med, E.OperatorParams(2 / 3, 2 * np.pi * dims[0] / 10, 0.15))
        N = g.n_dofs()
        x = rng.uniform(-1, 1, N) + 1j * rng.uniform(-1, 1, N)
        b = rng.uniform(-1, 1, N) + 1j * rng.uniform(-1, 1, N)
        y = E.apply_mixed_operator(D, x)
        r = E.residual(D, b, x)
        print(dims, float(np.abs(y).max()), float(np.abs(r - (b - y)).max()))


if __name__ == "__main__":
    main()
