"""BASELINE.json configs[0..4] as pinned, reproducible workloads.

Each builder returns a `Workload`: grid, media, the shifted (preconditioner)
and unshifted (Krylov) operator parameters, multigrid options, the right-hand
side(s) and Krylov options -- everything a solve or a bench line needs, built
only from seeds (synthetic data; no dataset is read). `scale` shrinks a
config by a power of two along every axis (cells, sponge width and
correlation length alike; one level fewer per halving) so the parity tests
can run the same recipe at sizes the CPU reference finishes in seconds.

Shared recipe (BASELINE.json "configs"):
  * staggered ux/uy(/uz) + p, complex128, beta = 2/3 (the paper's tuned
    coarse-stencil weights on every level), GMRES(10) right-preconditioned by
    one V(2,2) shifted-Laplacian cycle, full red-black Vanka, damping from
    experiments.hpp:221 default_solve_damping, coarsening to 16 cells
    (17 nodes) per axis, exact coarsest solve, rtol 1e-6;
  * shift alpha = 0.5: the reference default 0.1 stalls FGMRES once the
    hierarchy has 4+ levels (measured with the reference itself);
  * omega for 10 points per shear wavelength at the minimum interior cs
    (experiments.hpp:137 omega_from_gs);
  * heterogeneous media: `layered_grf_media` (8 layers, cs in [1, 2.5],
    cp/cs in [1.7, 2.2], rho in [1, 2.5], each times a +-10% smooth Gaussian
    random field with correlation length 20h), seed 2023.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

from . import ehmg as E

SEED = 2023
BETA = 2.0 / 3.0
ALPHA = 0.5
GAMMA_PHYS = 0.01
PPW = 10.0


@dataclasses.dataclass
class Workload:
    name: str
    grid: E.StaggeredGrid
    media: E.MediaModel
    shifted: E.OperatorParams
    unshifted: E.OperatorParams
    mg: E.MgOptions
    krylov: E.KrylovOptions
    sources: list            # [(component, index)]
    sponge: E.SpongeConfig
    notes: str = ""
    agg_n2: int = 32         # z-slab mode: levels with <= agg_n2 cell planes are agglomerated

    def rhs(self, k: int = 0) -> np.ndarray:
        comp, idx = self.sources[k]
        return E.make_point_source(self.grid, comp, idx)


def grf_media(g: E.StaggeredGrid, corr_cells: float) -> E.MediaModel:
    """the heterogeneous recipe (device builder, csrc/ehmg_media.cuh)"""
    return E.layered_grf_media(g, SEED, corr_cells=corr_cells, gamma_phys=GAMMA_PHYS)


def _levels_to_16(n_min: int) -> int:
    """levels coarsening the smallest axis down to 16 cells (>= 2)"""
    return max(2, int(round(math.log2(n_min / 16))) + 1)


def _finish(name, g, med, sponge, sources, levels, notes, agg_n2=32):
    med.gamma = E.build_attenuation_profile(g, GAMMA_PHYS, sponge)
    med.validate(g)
    omega = E.omega_from_gs(g, med, PPW, sponge)
    mg = E.MgOptions(n_levels=levels, cycle="v", nu1=2, nu2=2,
                     damping=E.default_solve_damping(PPW, levels), vanka_mode=E.FULL,
                     sweep=E.RED_BLACK, coarse="lu")
    return Workload(name, g, med, E.OperatorParams(BETA, omega, ALPHA), E.OperatorParams(BETA, omega, 0.0),
                    mg, E.KrylovOptions(restart=10, max_iterations=4000, rtol=1e-6), sources, sponge, notes,
                    agg_n2)


def _scaled(v: int, scale: int) -> int:
    return max(1, v // scale)


def config0(scale: int = 1, levels: int = 0) -> Workload:
    """2D homogeneous 257^2 nodes: rho = mu = 1, lambda = 2 (cs = 1, cp = 2),
    10 points per shear wavelength, 20-cell quadratic sponge, unit point source
    in the x-component at the centre, 5 levels (17^2 coarsest)."""
    n = 256 // scale
    g = E.StaggeredGrid((n, n), 1.0 / n)
    med = E.MediaModel.homogeneous(g, 2.0, 1.0, 1.0, GAMMA_PHYS)
    return _finish("configs[0]", g, med, E.SpongeConfig(_scaled(20, scale)), [(0, (n // 2, n // 2))],
                   levels or _levels_to_16(n), "x-component point source at the centre")


def config1(scale: int = 1, levels: int = 0) -> Workload:
    """2D heterogeneous 1025^2 nodes: layered + GRF media (seed 2023), 32-cell
    sponge, 10 ppw at the minimum cs, point source near the top: the
    vertical displacement 4 cells below the surface (a pressure-row source
    stalls this preconditioner in the reference as well)."""
    n = 1024 // scale
    g = E.StaggeredGrid((n, n), 1.0 / n)
    med = grf_media(g, 20.0 / scale)
    return _finish("configs[1]", g, med, E.SpongeConfig(_scaled(32, scale)), [(1, (n // 2, max(1, 4 // scale)))],
                   levels or _levels_to_16(n), "vertical-displacement point source near the top")


def config2(scale: int = 1, levels: int = 0) -> Workload:
    """3D homogeneous 257^3 nodes, media of configs[0], 24-cell sponge,
    x-component point source at the centre, 5 levels (17^3 coarsest)."""
    n = 256 // scale
    g = E.StaggeredGrid((n, n, n), 1.0 / n)
    med = E.MediaModel.homogeneous(g, 2.0, 1.0, 1.0, GAMMA_PHYS)
    return _finish("configs[2]", g, med, E.SpongeConfig(_scaled(24, scale)), [(0, (n // 2, n // 2, n // 2))],
                   levels or _levels_to_16(n), "x-component point source at the centre")


def config3(scale: int = 1, levels: int = 0) -> Workload:
    """3D heterogeneous 513^3 nodes: configs[1]'s recipe extended to 3D (3D
    Gaussian perturbations, seed 2023), 32-cell sponge, 10 ppw at the minimum
    cs, vertical point source near the top surface, 6 levels (17^3
    coarsest); the z-slab mode agglomerates levels below 65^3 nodes."""
    n = 512 // scale
    g = E.StaggeredGrid((n, n, n), 1.0 / n)
    med = grf_media(g, 20.0 / scale)
    return _finish("configs[3]", g, med, E.SpongeConfig(_scaled(32, scale)),
                   [(2, (n // 2, n // 2, max(1, 4 // scale)))], levels or _levels_to_16(n),
                   "vertical-displacement point source near the top", agg_n2=32 // scale)


def config4_weak(gpus: int = 1, scale: int = 1, levels: int = 0) -> Workload:
    """Weak scaling: 384 x 384 x (192 G) cells on G GPUs with configs[3]'s
    media recipe; 6 levels (12 x 12 x 6G coarsest)."""
    nx, nz = 384 // scale, 192 * gpus // scale
    g = E.StaggeredGrid((nx, nx, nz), 1.0 / nx)
    med = grf_media(g, 20.0 / scale)
    return _finish(f"configs[4] weak x{gpus}", g, med, E.SpongeConfig(_scaled(32, scale)),
                   [(2, (nx // 2, nx // 2, max(1, 4 // scale)))], levels or max(2, 6 - int(math.log2(scale))),
                   "vertical-displacement point source near the top", agg_n2=32 // scale)


def config4_sources(n_sources: int = 32, scale: int = 1, levels: int = 0) -> Workload:
    """32 surface point sources on the 257^3 grid with configs[3]'s media
    recipe: vertical displacement on the top surface (z = 0, as the
    reference's middle_of_top_row places sources, grid.hpp:174-179), on a
    4 x 8 pattern; each is an independent preconditioned FGMRES solve."""
    n = 256 // scale
    g = E.StaggeredGrid((n, n, n), 1.0 / n)
    med = grf_media(g, 20.0 / scale)
    pos = [(int((i + 0.5) * n / 8), int((j + 0.5) * n / 4), 0) for j in range(4) for i in range(8)]
    return _finish("configs[4] sources", g, med, E.SpongeConfig(_scaled(24, scale)),
                   [(2, p) for p in pos[:n_sources]], levels or _levels_to_16(n),
                   "vertical-displacement point sources on the top surface (z = 0)")


CONFIGS = {0: config0, 1: config1, 2: config2, 3: config3}
