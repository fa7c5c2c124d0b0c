"""B200-native GMRES + shifted-Laplacian multigrid for the staggered elastic
Helmholtz equation (the data-parallel core of arXiv:2307.03242).

Host mirror of the reference interface: :mod:`paper_2307_03242_b200.ehmg`.
Kernels and C ABI: ``csrc/`` and ``include/ehmg_b200.h``.
"""
from .ehmg import *  # noqa: F401,F403
from .ehmg import lib  # noqa: F401
