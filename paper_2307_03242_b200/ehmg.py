"""Host-side mirror of the reference's solver interface over the B200 C ABI.

The names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/include/ehmg/*.hpp) so a caller of the reference's
matrix-free path can switch to this package:

    reference (C++)                          here (Python over include/ehmg_b200.h)
    StaggeredGrid<Dim>(dims, h)              StaggeredGrid(dims, h)
    MediaModel<Dim>::homogeneous(...)        MediaModel.homogeneous(...)
    build_attenuation_profile(g, gp, sp)     build_attenuation_profile(g, gp, sp)
    make_point_source<double>(g, comp, idx)  make_point_source(g, comp, idx)
    make_opdata<double>(g, media, par)       make_opdata(g, media, par)
    apply_mixed_operator(D, x, y)            apply_mixed_operator(D, x, y)
    VankaSmoother<double,Dim>(mode).sweep    VankaSmoother(mode).sweep(D, b, x, w, order)
    restrict_field / prolong_field           restrict_field / prolong_field
    coarsen_media / coarsen_grid             coarsen_media / coarsen_grid
    Multigrid<double,Dim>(g, m, par, opt)    Multigrid(g, m, par, opt)
    fgmres(A, M, b, x, opt)                  fgmres(D0, mg, b, x, opt)
    run_solve(cfg, out, threads, seed)       run_solve(cfg)

Fields are complex128 vectors in the reference flatten() order; numpy arrays
are host buffers (copied through HBM inside each call), CUDA tensors
(torch, complex128) stay resident in HBM. There is no CPU fallback: every
call fails loudly without the sm_100a library or a CUDA device.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import math
import os
from typing import Optional, Sequence

import numpy as np

from . import build as _build

HOST, DEVICE = 0, 1
_ERRORS = {-1: ValueError, -2: RuntimeError, -3: RuntimeError, -4: IndexError}

_lib = None


class _MgOpts(C.Structure):
    _fields_ = [("n_levels", C.c_int), ("cycle", C.c_int), ("nu1", C.c_int), ("nu2", C.c_int),
                ("damping", C.c_double), ("vanka_mode", C.c_int), ("sweep", C.c_int),
                ("k_inner_iterations", C.c_int), ("k_inner_rtol", C.c_double),
                ("precision", C.c_int), ("coarse", C.c_int), ("lu_dof_budget", C.c_int64),
                ("kz_sweeps_per_apply", C.c_int), ("kz_damping", C.c_double), ("kz_rtol", C.c_double),
                ("kz_max_iterations", C.c_int), ("kz_restart", C.c_int)]


class _MOpts(C.Structure):
    _fields_ = [("warmup", C.c_int), ("tol", C.c_double), ("max_cycles", C.c_int),
                ("growth_limit", C.c_int)]


class _MRes(C.Structure):
    _fields_ = [("factor", C.c_double), ("cycles", C.c_int), ("diverged", C.c_int),
                ("n_history", C.c_int)]


class _KOpts(C.Structure):
    _fields_ = [("restart", C.c_int), ("max_iterations", C.c_int), ("rtol", C.c_double),
                ("stall_factor", C.c_double), ("stall_cycles", C.c_int), ("orthogonalization", C.c_int)]


class _KRes(C.Structure):
    _fields_ = [("status", C.c_int), ("iterations", C.c_int), ("relres", C.c_double),
                ("n_history", C.c_int)]


def lib():
    """Load the sm_100a library (raises if it is missing)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_build.LIB):
            raise RuntimeError(f"B200 library not built: {_build.LIB} (run __graft_entry__.build())")
        L = C.CDLL(_build.LIB)
        vp, ip, dp = C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_double)
        i64 = C.c_int64
        L.ehmg_last_error.restype = C.c_char_p
        L.ehmg_version.restype = C.c_char_p
        L.ehmg_op_create.argtypes = [C.c_int, ip, C.c_double, vp, vp, vp, vp, C.c_double,
                                     C.c_double, C.c_double, C.POINTER(vp)]
        L.ehmg_op_destroy.argtypes = [vp]
        L.ehmg_op_n_dofs.argtypes = [vp]
        L.ehmg_op_n_dofs.restype = i64
        L.ehmg_op_stream.argtypes = [vp]
        L.ehmg_op_stream.restype = C.c_uint64
        L.ehmg_apply_mixed_operator.argtypes = [vp, vp, vp, C.c_int]
        L.ehmg_residual.argtypes = [vp, vp, vp, vp, C.c_int]
        L.ehmg_vanka_create.argtypes = [vp, C.c_int, C.POINTER(vp)]
        L.ehmg_vanka_destroy.argtypes = [vp]
        L.ehmg_vanka_per_cell_complex_count.argtypes = [vp]
        L.ehmg_vanka_cache.argtypes = [vp, vp]
        L.ehmg_vanka_sweep.argtypes = [vp, vp, vp, C.c_double, C.c_int, C.c_int, C.c_int]
        L.ehmg_restrict_field.argtypes = [C.c_int, ip, vp, vp, C.c_int]
        L.ehmg_prolong_field.argtypes = [C.c_int, ip, vp, vp, C.c_int]
        L.ehmg_coarsen_media.argtypes = [C.c_int, ip, vp, vp]
        L.ehmg_layered_media.argtypes = [C.c_int, ip, C.c_double, C.c_uint64, vp, vp, vp, vp]
        L.ehmg_layered_grf_media.argtypes = [C.c_int, ip, C.c_int, vp, C.c_double, C.c_double,
                                             C.c_double, C.c_uint64, vp, vp, vp, vp]
        L.ehmg_multigrid_measure_convergence.argtypes = [vp, C.c_uint64, C.POINTER(_MOpts),
                                                         C.POINTER(_MRes), vp, C.c_int]
        L.ehmg_attenuation_profile.argtypes = [C.c_int, ip, C.c_double, C.c_int, C.c_double,
                                               C.c_int, vp]
        L.ehmg_multigrid_create.argtypes = [C.c_int, ip, C.c_double, vp, vp, vp, vp, C.c_double,
                                            C.c_double, C.c_double, C.POINTER(_MgOpts),
                                            C.POINTER(vp)]
        L.ehmg_multigrid_destroy.argtypes = [vp]
        L.ehmg_multigrid_n_levels.argtypes = [vp]
        L.ehmg_multigrid_factor_sets.argtypes = [vp, C.c_int]
        L.ehmg_multigrid_cycle.argtypes = [vp, vp, vp, C.c_int]
        L.ehmg_multigrid_precondition.argtypes = [vp, vp, vp, C.c_int]
        L.ehmg_multigrid_precondition_many.argtypes = [vp, C.c_int, C.POINTER(vp), C.POINTER(vp)]
        L.ehmg_multigrid_stream.argtypes = [vp]
        L.ehmg_multigrid_stream.restype = C.c_uint64
        L.ehmg_multigrid_time_precondition.argtypes = [vp, vp, vp, C.c_int, dp]
        L.ehmg_fgmres_solve.argtypes = [vp, vp, vp, vp, C.c_int, C.POINTER(_KOpts),
                                        C.POINTER(_KRes), vp, C.c_int]
        L.ehmg_field_dot.argtypes = [i64, vp, vp, vp]
        L.ehmg_field_norm.argtypes = [i64, vp, dp]
        L.ehmg_field_axpy.argtypes = [i64, C.c_double, C.c_double, vp, vp]
        L.ehmg_set_device.argtypes = [C.c_int]
        L.ehmg_slab_plan.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, ip, ip]
        L.ehmg_slab_multigrid_create.argtypes = [C.c_int, ip, C.c_double, vp, vp, vp, vp,
                                                 C.c_double, C.c_double, C.c_double,
                                                 C.POINTER(_MgOpts), C.c_int, C.c_int,
                                                 C.POINTER(vp)]
        L.ehmg_slab_multigrid_destroy.argtypes = [vp]
        L.ehmg_slab_multigrid_levels.argtypes = [vp, ip, ip]
        L.ehmg_slab_multigrid_precondition.argtypes = [vp, vp, vp, C.c_int]
        L.ehmg_slab_multigrid_exchanged_bytes.argtypes = [vp]
        L.ehmg_slab_multigrid_exchanged_bytes.restype = i64
        L.ehmg_dist_create.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, ip,
                                       C.c_double, vp, vp, vp, vp, C.c_double, C.c_double,
                                       C.c_double, C.POINTER(_MgOpts), C.c_int, C.POINTER(vp)]
        L.ehmg_dist_destroy.argtypes = [vp]
        L.ehmg_dist_window.argtypes = [vp, ip, ip, ip, ip]
        L.ehmg_dist_precondition.argtypes = [vp, vp, vp]
        L.ehmg_dist_time_precondition.argtypes = [vp, vp, C.c_int, dp]
        L.ehmg_dist_exchanged_bytes.argtypes = [vp]
        L.ehmg_dist_exchanged_bytes.restype = i64
        L.ehmg_dist_solve.argtypes = [vp, vp, vp, C.POINTER(_KOpts), C.POINTER(_KRes), vp,
                                      C.c_int]
        L.ehmg_profile_enable.argtypes = [C.c_int]
        L.ehmg_profile_report.argtypes = [C.c_char_p, C.c_int]
        _lib = L
    return _lib


def profile_enable(on: bool = True) -> None:
    """Per-launch CUDA-event timing of the cycle kernels (bench roofline)."""
    _check(lib().ehmg_profile_enable(int(on)))


def profile_report() -> list:
    """[(kernel, level, count, total_ms)] for the launches since enable."""
    buf = C.create_string_buffer(1 << 16)
    _check(lib().ehmg_profile_report(buf, len(buf)))
    rows = []
    for line in buf.value.decode().splitlines():
        k, lv, c, ms = line.split()
        rows.append((k, int(lv), int(c), float(ms)))
    return rows


def _check(rc: int) -> None:
    if rc != 0:
        msg = lib().ehmg_last_error().decode()
        raise _ERRORS.get(rc, RuntimeError)(msg)


# ---------------------------------------------------------------- buffers
def _is_device(a) -> bool:
    return hasattr(a, "is_cuda") and bool(a.is_cuda)


def _ptr(a, n: int, writable: bool = False):
    """(pointer, where) for a field buffer; validates dtype and size."""
    if _is_device(a):
        import torch
        if a.dtype != torch.complex128 or not a.is_contiguous() or a.numel() != n:
            raise ValueError("device field must be a contiguous complex128 tensor of n_dofs")
        # the library runs on its own non-blocking streams: whatever torch
        # still has queued on this tensor must land first (ehmg_b200.h,
        # "Ordering of EHMG_DEVICE buffers")
        torch.cuda.current_stream(a.device).synchronize()
        return C.c_void_p(a.data_ptr()), DEVICE
    if not isinstance(a, np.ndarray) or a.dtype != np.complex128 or not a.flags.c_contiguous:
        raise ValueError("host field must be a C-contiguous complex128 numpy array")
    if a.size != n:
        raise ValueError(f"field size {a.size} does not match grid ({n} DOFs)")
    if writable and not a.flags.writeable:
        raise ValueError("output field is read-only")
    return C.c_void_p(a.ctypes.data), HOST


def _dims_arr(dims):
    a = (C.c_int * 3)(0, 0, 0)
    for i, d in enumerate(dims):
        a[i] = int(d)
    return a


def _cell_arr(v, n):
    a = np.ascontiguousarray(v, dtype=np.float64)
    if a.size != n:
        raise ValueError("media: field sizes do not match grid")
    return a


# ------------------------------------------------------------------- grid
class StaggeredGrid:
    """grid.hpp:64 -- cells per axis + uniform mesh width."""

    def __init__(self, dims: Sequence[int], h: float):
        self.dims = tuple(int(d) for d in dims)
        self.h = float(h)
        if len(self.dims) not in (2, 3):
            raise ValueError("grid: 2D or 3D only")
        if not self.h > 0:
            raise ValueError("grid: h must be positive")
        if any(d < 2 for d in self.dims):
            raise ValueError("grid: need >= 2 cells per axis")

    @property
    def ndim(self) -> int:
        return len(self.dims)

    def cell_box(self):
        return self.dims

    def face_box(self, axis: int):
        d = list(self.dims)
        d[axis] += 1
        return tuple(d)

    def edge_box(self, a: int, b: int):
        d = list(self.dims)
        d[a] += 1
        d[b] += 1
        return tuple(d)

    def n_cells(self) -> int:
        return int(np.prod(self.dims))

    def n_faces(self, axis: int) -> int:
        return int(np.prod(self.face_box(axis)))

    def n_dofs(self) -> int:
        return self.n_cells() + sum(self.n_faces(a) for a in range(self.ndim))

    def comp_offsets(self):
        off, o = [], 0
        for k in range(self.ndim):
            off.append(o)
            o += self.n_faces(k)
        off.append(o)
        return off

    def lin(self, box, idx) -> int:
        r = idx[-1]
        for a in range(len(box) - 2, -1, -1):
            r = r * box[a] + idx[a]
        return int(r)


def can_coarsen(g: StaggeredGrid) -> bool:
    """transfer.hpp:25"""
    return all(d % 2 == 0 and d // 2 >= 2 for d in g.dims)


def coarsen_grid(g: StaggeredGrid) -> StaggeredGrid:
    """transfer.hpp:31"""
    if not can_coarsen(g):
        raise ValueError("coarsen_grid: dims must be even and >= 4")
    return StaggeredGrid([d // 2 for d in g.dims], 2.0 * g.h)


# ------------------------------------------------------------------ media
@dataclasses.dataclass
class SpongeConfig:
    """media.hpp:85"""
    layer_width: int = 20
    gamma_max: float = 1.0
    absorb_top: bool = False


class MediaModel:
    """media.hpp:13 -- cell-centred lambda, mu, rho, gamma (axis-0-fastest)."""

    def __init__(self, lambda_, mu, rho, gamma):
        self.lambda_ = np.ascontiguousarray(lambda_, np.float64).ravel()
        self.mu = np.ascontiguousarray(mu, np.float64).ravel()
        self.rho = np.ascontiguousarray(rho, np.float64).ravel()
        self.gamma = np.ascontiguousarray(gamma, np.float64).ravel()

    @staticmethod
    def homogeneous(g: StaggeredGrid, lambda_: float, mu: float, rho: float,
                    gamma: float = 0.0) -> "MediaModel":
        n = g.n_cells()
        return MediaModel(np.full(n, lambda_), np.full(n, mu), np.full(n, rho), np.full(n, gamma))

    def validate(self, g: StaggeredGrid) -> None:
        n = g.n_cells()
        if any(a.size != n for a in (self.lambda_, self.mu, self.rho, self.gamma)):
            raise ValueError("media: field sizes do not match grid")
        if not np.all(self.rho > 0):
            raise ValueError("media: rho must be positive")
        if not np.all(self.mu > 0):
            raise ValueError("media: mu must be positive")
        if not np.all(self.lambda_ + self.mu > 0):
            raise ValueError("media: lambda+mu must be positive")
        if not np.all(self.gamma >= 0):
            raise ValueError("media: gamma must be nonnegative")

    def vs(self):
        return np.sqrt(self.mu / self.rho)

    def vp(self):
        return np.sqrt((self.lambda_ + 2 * self.mu) / self.rho)

    def arrays(self, g: StaggeredGrid):
        n = g.n_cells()
        return tuple(_cell_arr(a, n) for a in (self.lambda_, self.mu, self.rho, self.gamma))


def build_attenuation_profile(g: StaggeredGrid, gamma_phys: float,
                              sponge: SpongeConfig = SpongeConfig()) -> np.ndarray:
    """media.hpp:95"""
    out = np.zeros(g.n_cells(), np.float64)
    _check(lib().ehmg_attenuation_profile(g.ndim, _dims_arr(g.dims), gamma_phys,
                                          int(sponge.layer_width), sponge.gamma_max,
                                          int(sponge.absorb_top), out.ctypes.data))
    return out


def coarsen_media(gf: StaggeredGrid, m: MediaModel) -> MediaModel:
    """transfer.hpp:40 -- each coarse cell is the mean of its children."""
    gc = coarsen_grid(gf)
    outs = []
    for a in m.arrays(gf):
        o = np.zeros(gc.n_cells(), np.float64)
        _check(lib().ehmg_coarsen_media(gf.ndim, _dims_arr(gf.dims), a.ctypes.data, o.ctypes.data))
        outs.append(o)
    return MediaModel(*outs)


def make_point_source(g: StaggeredGrid, component: int, index) -> np.ndarray:
    """grid.hpp:161 -- unit impulse scaled by the inverse cell volume."""
    box = g.face_box(component) if component < g.ndim else g.cell_box()
    if any(i < 0 or i >= d for i, d in zip(index, box)):
        raise IndexError("point source index outside grid")
    f = np.zeros(g.n_dofs(), np.complex128)
    f[g.comp_offsets()[component] + g.lin(box, index)] = 1.0 / g.h ** g.ndim
    return f


def middle_of_top_row(g: StaggeredGrid):
    """grid.hpp:174"""
    return tuple(list(d // 2 for d in g.dims[:-1]) + [0])


# --------------------------------------------------------------- operator
@dataclasses.dataclass
class OperatorParams:
    """operator.hpp:27"""
    beta: float = 1.0
    omega: float = 0.0
    alpha: float = 0.0
    periodic: bool = False


class OpData:
    """operator.hpp:40 OpData, resident in HBM."""

    def __init__(self, grid: StaggeredGrid, media: MediaModel, par: OperatorParams):
        if par.periodic:
            raise ValueError("periodic operators are LFA-probe only (out of scope on the B200 path)")
        self.grid, self.par = grid, par
        arrs = media.arrays(grid)
        h = C.c_void_p()
        _check(lib().ehmg_op_create(grid.ndim, _dims_arr(grid.dims), grid.h,
                                    *[a.ctypes.data for a in arrs], par.beta, par.omega, par.alpha,
                                    C.byref(h)))
        self._h = h
        self.n = grid.n_dofs()

    def __del__(self):
        if _lib is not None and getattr(self, "_h", None):
            _lib.ehmg_op_destroy(self._h)
            self._h = None

    @property
    def stream(self) -> int:
        return int(lib().ehmg_op_stream(self._h))


def make_opdata(grid: StaggeredGrid, media: MediaModel, par: OperatorParams) -> OpData:
    """operator.hpp:76"""
    return OpData(grid, media, par)


def make_field(D) -> np.ndarray:
    """operator.hpp:481"""
    return np.zeros(D.grid.n_dofs(), np.complex128)


def apply_mixed_operator(D: OpData, x, y=None):
    """operator.hpp:437 -- y = H x (H shifted when par.alpha > 0)."""
    if y is None:
        y = np.zeros(D.n, np.complex128) if not _is_device(x) else x.new_empty(D.n)
    px, wx = _ptr(x, D.n)
    py, wy = _ptr(y, D.n, writable=True)
    if wx != wy:
        raise ValueError("x and y must both be host arrays or both device tensors")
    _check(lib().ehmg_apply_mixed_operator(D._h, px, py, wx))
    return y


apply_shifted_operator = apply_mixed_operator  # operator.hpp:449


def residual(D: OpData, b, x, r=None):
    """multigrid.hpp:210 -- r = b - H x."""
    if r is None:
        r = np.zeros(D.n, np.complex128) if not _is_device(x) else x.new_empty(D.n)
    pb, wb = _ptr(b, D.n)
    px, wx = _ptr(x, D.n)
    pr, wr = _ptr(r, D.n, writable=True)
    if not wb == wx == wr:
        raise ValueError("fields must all be host arrays or all device tensors")
    _check(lib().ehmg_residual(D._h, pb, px, pr, wx))
    return r


# ------------------------------------------------------------------ Vanka
FULL, ECONOMIC = "full", "economic"
LEXICOGRAPHIC, RED_BLACK = "lexicographic", "red_black"


class VankaSmoother:
    """vanka.hpp:27 -- cell-wise box relaxation (full / economic)."""

    def __init__(self, mode: str = FULL):
        if mode not in (FULL, ECONOMIC):
            raise ValueError(f"config: unknown vanka mode '{mode}'")
        self.mode = mode
        self._h = None
        self._D = None
        self._builds = 0

    def __del__(self):
        if _lib is not None and getattr(self, "_h", None):
            _lib.ehmg_vanka_destroy(self._h)
            self._h = None

    def per_cell_complex_count(self, ndim: int) -> int:
        """vanka.hpp:35"""
        return ndim * ((4 if self.mode == FULL else 2) + 4) + 1

    def builds(self) -> int:
        return self._builds

    def ensure_cache(self, D: OpData) -> None:
        """vanka.hpp:40 -- rebuilt when the operator changes."""
        if self._D is D and self._h is not None:
            return
        if self._h is not None:
            lib().ehmg_vanka_destroy(self._h)
        h = C.c_void_p()
        _check(lib().ehmg_vanka_create(D._h, 0 if self.mode == FULL else 1, C.byref(h)))
        self._h, self._D = h, D
        self._builds += 1

    def cache(self, D: OpData) -> np.ndarray:
        self.ensure_cache(D)
        stride = lib().ehmg_vanka_per_cell_complex_count(self._h)
        out = np.zeros(D.grid.n_cells() * stride, np.complex128)
        _check(lib().ehmg_vanka_cache(self._h, out.ctypes.data))
        return out.reshape(-1, stride)

    def sweep(self, D: OpData, b, x, w: float, order: str = RED_BLACK, nsweeps: int = 1):
        """vanka.hpp:49 -- x updated in place (and returned)."""
        if order not in (LEXICOGRAPHIC, RED_BLACK):
            raise ValueError(f"config: unknown sweep order '{order}'")
        self.ensure_cache(D)
        pb, wb = _ptr(b, D.n)
        px, wx = _ptr(x, D.n, writable=True)
        if wb != wx:
            raise ValueError("b and x must both be host arrays or both device tensors")
        _check(lib().ehmg_vanka_sweep(self._h, pb, px, w, 1 if order == RED_BLACK else 0, nsweeps,
                                      wx))
        return x


# -------------------------------------------------------------- transfers
def _transfer(gf: StaggeredGrid, xin, restricting: bool):
    gc = coarsen_grid(gf)
    nin = gf.n_dofs() if restricting else gc.n_dofs()
    nout = gc.n_dofs() if restricting else gf.n_dofs()
    out = np.zeros(nout, np.complex128) if not _is_device(xin) else xin.new_empty(nout)
    pi, wi = _ptr(xin, nin)
    po, _ = _ptr(out, nout, writable=True)
    f = lib().ehmg_restrict_field if restricting else lib().ehmg_prolong_field
    _check(f(gf.ndim, _dims_arr(gf.dims), pi, po, wi))
    return out


def restrict_field(gf: StaggeredGrid, gc: StaggeredGrid, xf, periodic: bool = False):
    """transfer.hpp:188"""
    if periodic:
        raise ValueError("periodic transfers are LFA-probe only (out of scope on the B200 path)")
    return _transfer(gf, xf, True)


def prolong_field(gf: StaggeredGrid, gc: StaggeredGrid, xc, periodic: bool = False):
    """transfer.hpp:197"""
    if periodic:
        raise ValueError("periodic transfers are LFA-probe only (out of scope on the B200 path)")
    return _transfer(gf, xc, False)


# -------------------------------------------------------------- multigrid
_CYCLES = {"two_grid": 0, "v": 1, "w": 2, "k": 3}


@dataclasses.dataclass
class MgOptions:
    """multigrid.hpp:34 (coarsest level solved exactly)."""
    n_levels: int = 2
    cycle: str = "v"
    nu1: int = 1
    nu2: int = 1
    damping: float = 0.75
    vanka_mode: str = ECONOMIC
    sweep: str = LEXICOGRAPHIC
    # multigrid.hpp:22/:40-50. "automatic" and "lu" take the exact coarsest
    # solve; "kaczmarz" is rejected by the library
    coarse: str = "automatic"
    lu_dof_budget: int = 4_000_000
    kz_sweeps_per_apply: int = 5
    kz_damping: float = 0.8
    kz_rtol: float = 0.01
    kz_max_iterations: int = 150
    kz_restart: int = 40
    k_inner_iterations: int = 2
    k_inner_rtol: float = 0.25


_COARSE = {"automatic": 0, "lu": 1, "kaczmarz": 2}


def _mg_opts(opt: "MgOptions", precision: str) -> _MgOpts:
    if opt.coarse not in _COARSE:
        raise ValueError(f"config: unknown coarse solver '{opt.coarse}'")
    return _MgOpts(opt.n_levels, _CYCLES[opt.cycle], opt.nu1, opt.nu2, opt.damping,
                   0 if opt.vanka_mode == FULL else 1, 1 if opt.sweep == RED_BLACK else 0,
                   opt.k_inner_iterations, opt.k_inner_rtol, 1 if precision == "mixed" else 0,
                   _COARSE[opt.coarse], int(opt.lu_dof_budget), opt.kz_sweeps_per_apply,
                   opt.kz_damping, opt.kz_rtol, opt.kz_max_iterations, opt.kz_restart)


@dataclasses.dataclass
class MeasureOptions:
    """multigrid.hpp:56"""
    warmup: int = 5
    tol: float = 1e-9
    max_cycles: int = 500
    growth_limit: int = 20


@dataclasses.dataclass
class MeasureResult:
    """multigrid.hpp:63"""
    factor: float
    cycles: int
    diverged: bool
    history: list


class Multigrid:
    """multigrid.hpp:70 -- shifted-Laplacian hierarchy resident in HBM."""

    def __init__(self, grid: StaggeredGrid, media: MediaModel, par: OperatorParams,
                 opt: MgOptions, precision: str = "double"):
        """precision "mixed": complex64 hierarchy behind complex128
        precondition()/cycle() (experiments.hpp:241 MixedPrecondition)."""
        if precision not in ("double", "mixed"):
            raise ValueError(f"config: unknown precision '{precision}'")
        self.precision = precision
        if opt.cycle not in _CYCLES:
            raise ValueError(f"config: unknown cycle '{opt.cycle}'")
        if par.periodic:
            raise ValueError("periodic hierarchies are LFA-probe only (out of scope)")
        self.grid, self.par, self.opt = grid, par, opt
        o = _mg_opts(opt, precision)
        arrs = media.arrays(grid)
        h = C.c_void_p()
        _check(lib().ehmg_multigrid_create(grid.ndim, _dims_arr(grid.dims), grid.h,
                                           *[a.ctypes.data for a in arrs], par.beta, par.omega,
                                           par.alpha, C.byref(o), C.byref(h)))
        self._h = h
        self.n = grid.n_dofs()

    def __del__(self):
        if _lib is not None and getattr(self, "_h", None):
            _lib.ehmg_multigrid_destroy(self._h)
            self._h = None

    def n_levels(self) -> int:
        return lib().ehmg_multigrid_n_levels(self._h)

    def factor_sets(self, level: int = 0) -> int:
        """Distinct Vanka factor entry sets of a level when its colour updates use the factor
        dictionary (0: per-cell cache). No reference counterpart (measurement)."""
        return lib().ehmg_multigrid_factor_sets(self._h, int(level))

    def coarse_kind(self) -> str:
        return "lu"

    def coarse_exact(self) -> bool:
        return True

    @property
    def stream(self) -> int:
        return int(lib().ehmg_multigrid_stream(self._h))

    def cycle(self, b, x):
        """multigrid.hpp:133 -- one cycle on A x = b, x updated in place."""
        pb, wb = _ptr(b, self.n)
        px, wx = _ptr(x, self.n, writable=True)
        if wb != wx:
            raise ValueError("b and x must both be host arrays or both device tensors")
        _check(lib().ehmg_multigrid_cycle(self._h, pb, px, wx))
        return x

    def measure_convergence_factor(self, seed: int, mo: MeasureOptions = None) -> MeasureResult:
        """multigrid.hpp:143 -- stationary cycles on the homogeneous problem from
        the reference's seeded random start; geometric-mean reduction factor."""
        mo = mo or MeasureOptions()
        o = _MOpts(mo.warmup, mo.tol, mo.max_cycles, mo.growth_limit)
        r = _MRes()
        hist = np.zeros(mo.max_cycles + 8, np.float64)
        _check(lib().ehmg_multigrid_measure_convergence(self._h, int(seed) & (2**64 - 1), C.byref(o),
                                                        C.byref(r), hist.ctypes.data, len(hist)))
        return MeasureResult(r.factor, r.cycles, bool(r.diverged),
                             list(hist[:min(r.n_history, len(hist))]))

    def precondition(self, r, z=None):
        """multigrid.hpp:136 -- z = one cycle from zero applied to r."""
        if z is None:
            z = np.zeros(self.n, np.complex128) if not _is_device(r) else r.new_empty(self.n)
        pr, wr = _ptr(r, self.n)
        pz, wz = _ptr(z, self.n, writable=True)
        if wr != wz:
            raise ValueError("r and z must both be host arrays or both device tensors")
        _check(lib().ehmg_multigrid_precondition(self._h, pr, pz, wr))
        return z

    def precondition_many(self, rs, zs=None):
        """multigrid.hpp:136 precondition over several host right-hand sides
        (r[i] -> z[i]); host<->device copies of neighbouring right-hand sides
        overlap the current cycle (pinned host arrays for the overlap).
        Output arrays may repeat (written in order)."""
        rs = list(rs)
        if zs is None:
            zs = [np.zeros(self.n, np.complex128) for _ in rs]
        zs = list(zs)
        if len(zs) != len(rs):
            raise ValueError("precondition_many: as many outputs as right-hand sides")
        pr = (C.c_void_p * max(1, len(rs)))()
        pz = (C.c_void_p * max(1, len(rs)))()
        for i, (r, z) in enumerate(zip(rs, zs)):
            a, wr = _ptr(r, self.n)
            b, wz = _ptr(z, self.n, writable=True)
            if wr != HOST or wz != HOST:
                raise ValueError("precondition_many takes host arrays (device buffers: precondition)")
            pr[i], pz[i] = a, b
        _check(lib().ehmg_multigrid_precondition_many(self._h, len(rs), pr, pz))
        return zs

    def time_precondition(self, r_dev, z_dev, count: int) -> float:
        """CUDA-event time (ms) of `count` preconditioner applications."""
        ms = C.c_double(0)
        pr, _ = _ptr(r_dev, self.n)
        pz, _ = _ptr(z_dev, self.n, writable=True)
        _check(lib().ehmg_multigrid_time_precondition(self._h, pr, pz, count, C.byref(ms)))
        return ms.value


# ------------------------------------------------------- z-slab decomposition
SLAB_GHOST_LO, SLAB_GHOST_HI = 3, 2


def slab_plan(n2: int, n_levels: int, nslabs: int, agg_n2: int = 64):
    """Slab partition of the z axis (pure host): (distributed levels, level-0
    boundaries). Boundaries are multiples of 2**La; every distributed level
    keeps >= 4 owned planes per slab."""
    la = C.c_int(0)
    z0 = (C.c_int * (nslabs + 1))()
    _check(lib().ehmg_slab_plan(n2, n_levels, nslabs, agg_n2, C.byref(la), z0))
    return la.value, [z0[i] for i in range(nslabs + 1)]


def slab_windows(n2: int, n_levels: int, nslabs: int, agg_n2: int = 64, level: int = 0):
    """[(Z0, Z1, W0, W1)] per slab at `level`: owned cell planes and stored
    window [Z0 - 3, Z1 + 2) clipped to the grid."""
    la, z0 = slab_plan(n2, n_levels, nslabs, agg_n2)
    if level >= la:
        raise ValueError("level is agglomerated (replicated), not distributed")
    nl = n2 >> level
    out = []
    for q in range(nslabs):
        a, b = z0[q] >> level, z0[q + 1] >> level
        out.append((a, b, max(0, a - SLAB_GHOST_LO), min(nl, b + SLAB_GHOST_HI)))
    return out


class SlabMultigrid:
    """The shifted-Laplacian hierarchy decomposed into z-slabs (north_star
    (6)): fine levels sharded with ghost-plane exchange, levels with z extent
    <= agg_n2 agglomerated. Same options and results as Multigrid."""

    def __init__(self, grid: StaggeredGrid, media: MediaModel, par: OperatorParams,
                 opt: MgOptions, nslabs: int, agg_n2: int = 64, precision: str = "double"):
        if precision not in ("double", "mixed"):
            raise ValueError(f"config: unknown precision '{precision}'")
        o = _mg_opts(opt, precision)
        arrs = media.arrays(grid)
        h = C.c_void_p()
        _check(lib().ehmg_slab_multigrid_create(grid.ndim, _dims_arr(grid.dims), grid.h,
                                                *[a.ctypes.data for a in arrs], par.beta,
                                                par.omega, par.alpha, C.byref(o), nslabs, agg_n2,
                                                C.byref(h)))
        self._h = h
        self.n = grid.n_dofs()
        self.nslabs = nslabs

    def __del__(self):
        if _lib is not None and getattr(self, "_h", None):
            _lib.ehmg_slab_multigrid_destroy(self._h)
            self._h = None

    def levels(self):
        d, t = C.c_int(0), C.c_int(0)
        _check(lib().ehmg_slab_multigrid_levels(self._h, C.byref(d), C.byref(t)))
        return d.value, t.value

    def exchanged_bytes(self) -> int:
        return int(lib().ehmg_slab_multigrid_exchanged_bytes(self._h))

    def precondition(self, r, z=None):
        if z is None:
            z = np.zeros(self.n, np.complex128) if not _is_device(r) else r.new_empty(self.n)
        pr, wr = _ptr(r, self.n)
        pz, wz = _ptr(z, self.n, writable=True)
        if wr != wz:
            raise ValueError("r and z must both be host arrays or both device tensors")
        _check(lib().ehmg_slab_multigrid_precondition(self._h, pr, pz, wr))
        return z


class DistributedSlabSolver:
    """One z-slab of the hierarchy per process (one process per GPU). Ranks
    of one job meet in a shared-memory segment named `job`, exchange ghost
    planes by peer copies (CUDA IPC) and sum reductions in rank order.
    Fields are full host arrays; results carry this rank's owned planes."""

    def __init__(self, job: str, rank: int, nranks: int, device: int, grid: StaggeredGrid,
                 media: MediaModel, par: OperatorParams, opt: MgOptions, agg_n2: int = 64,
                 precision: str = "double"):
        if precision not in ("double", "mixed"):
            raise ValueError(f"config: unknown precision '{precision}'")
        o = _mg_opts(opt, precision)
        arrs = media.arrays(grid)
        h = C.c_void_p()
        _check(lib().ehmg_dist_create(job.encode(), rank, nranks, device, grid.ndim,
                                      _dims_arr(grid.dims), grid.h, *[a.ctypes.data for a in arrs],
                                      par.beta, par.omega, par.alpha, C.byref(o), agg_n2,
                                      C.byref(h)))
        self._h = h
        self.grid, self.n, self.rank, self.nranks = grid, grid.n_dofs(), rank, nranks

    def close(self):
        if _lib is not None and getattr(self, "_h", None):
            _check(_lib.ehmg_dist_destroy(self._h))
            self._h = None

    __del__ = close

    def window(self):
        v = [C.c_int(0) for _ in range(4)]
        _check(lib().ehmg_dist_window(self._h, *[C.byref(a) for a in v]))
        return tuple(a.value for a in v)

    def owned_mask(self):
        """Boolean mask of the flat DOFs this rank owns."""
        z0, z1, _, _ = self.window()
        g = self.grid
        off = g.comp_offsets() + [g.n_dofs()]
        m = np.zeros(self.n, bool)
        for k in range(4):
            ps = (g.dims[0] + (k == 0)) * (g.dims[1] + (k == 1))
            top = z1 + (1 if (k == 2 and self.rank == self.nranks - 1) else 0)
            m[off[k] + z0 * ps:off[k] + top * ps] = True
        return m

    def precondition(self, r):
        r = np.ascontiguousarray(r, np.complex128)
        z = np.zeros(self.n, np.complex128)
        _check(lib().ehmg_dist_precondition(self._h, r.ctypes.data, z.ctypes.data))
        return z

    def time_precondition(self, r, count: int) -> float:
        """CUDA-event ms of `count` applications on the resident window."""
        r = np.ascontiguousarray(r, np.complex128)
        ms = C.c_double(0)
        _check(lib().ehmg_dist_time_precondition(self._h, r.ctypes.data, count, C.byref(ms)))
        return ms.value

    def exchanged_bytes(self) -> int:
        return int(lib().ehmg_dist_exchanged_bytes(self._h))

    def solve(self, b, opt: "KrylovOptions" = None):
        opt = opt or KrylovOptions()
        b = np.ascontiguousarray(b, np.complex128)
        x = np.zeros(self.n, np.complex128)
        ko = _KOpts(opt.restart, opt.max_iterations, opt.rtol, opt.stall_factor, opt.stall_cycles,
                    _ORTH[opt.orthogonalization])
        kr = _KRes()
        cap = opt.max_iterations + opt.max_iterations // max(1, opt.restart) + 8
        hist = np.zeros(cap, np.float64)
        _check(lib().ehmg_dist_solve(self._h, b.ctypes.data, x.ctypes.data, C.byref(ko),
                                     C.byref(kr), hist.ctypes.data, cap))
        return x, KrylovResult(_STATUS[kr.status], kr.iterations, kr.relres,
                               list(hist[:min(kr.n_history, cap)]))


# ----------------------------------------------------------------- Krylov
@dataclasses.dataclass
class KrylovOptions:
    """krylov.hpp:45"""
    restart: int = 5
    max_iterations: int = 600
    rtol: float = 1e-6
    stall_factor: float = 0.99
    stall_cycles: int = 2
    # B200 addition: "classical" (CGS passes, re-orthogonalised as the
    # reference decides; fewer HBM passes) or "modified" (krylov.hpp:115 order)
    orthogonalization: str = "classical"

    def __post_init__(self):
        if self.restart < 1:
            raise ValueError("fgmres: restart must be >= 1")
        if self.max_iterations < 0:
            raise ValueError("fgmres: max_iterations must be >= 0")
        if self.orthogonalization not in _ORTH:
            raise ValueError(f"krylov: unknown orthogonalization '{self.orthogonalization}'")


_ORTH = {"classical": 0, "modified": 1}
_STATUS = {0: "converged", 1: "max_iterations", 2: "breakdown", 3: "stalled"}


@dataclasses.dataclass
class KrylovResult:
    """krylov.hpp:55"""
    status: str = "max_iterations"
    iterations: int = 0
    relres: float = 1.0
    history: list = dataclasses.field(default_factory=list)


def fgmres(A: OpData, M: Optional[Multigrid], b, x, opt: KrylovOptions = KrylovOptions()):
    """krylov.hpp:65 with A = H (unshifted) and M = one cycle of the shifted
    hierarchy (experiments.hpp:313). x is updated in place."""
    n = A.n
    pb, wb = _ptr(b, n)
    px, wx = _ptr(x, n, writable=True)
    if wb != wx:
        raise ValueError("b and x must both be host arrays or both device tensors")
    ko = _KOpts(opt.restart, opt.max_iterations, opt.rtol, opt.stall_factor, opt.stall_cycles,
                    _ORTH[opt.orthogonalization])
    kr = _KRes()
    cap = opt.max_iterations + opt.max_iterations // max(1, opt.restart) + 8
    hist = np.zeros(cap, np.float64)
    _check(lib().ehmg_fgmres_solve(A._h, M._h if M is not None else None, pb, px, wx,
                                   C.byref(ko), C.byref(kr), hist.ctypes.data, cap))
    return KrylovResult(_STATUS[kr.status], kr.iterations, kr.relres,
                        list(hist[:min(kr.n_history, cap)]))


# -------------------------------------------------------- experiment drive
def linear_media(g: StaggeredGrid, gamma_phys: float) -> MediaModel:
    """experiments.hpp:61 -- rho, lambda, mu linear in depth (last axis)."""
    nd = g.dims[-1]
    t = (np.arange(nd) + 0.5) / nd
    shape = g.dims[::-1]
    tt = np.broadcast_to(t.reshape([nd] + [1] * (g.ndim - 1)), shape).ravel()
    n = g.n_cells()
    return MediaModel(4 + 16 * tt, 1 + 14 * tt, 2 + tt, np.full(n, gamma_phys))


def layered_media(g: StaggeredGrid, gamma_phys: float, seed: int) -> MediaModel:
    """experiments.hpp:78 -- seeded horizontal layers along the last axis
    (index 0 at the top): 5..10 layers, per-layer shear velocity in [0.5, 2],
    density in [1.5, 3] and lambda/mu in [2, 20]. Drawn by the library with
    the reference's std::mt19937_64 stream and <random> distributions."""
    n = g.n_cells()
    lam, mu, rho, gam = (np.empty(n, np.float64) for _ in range(4))
    dims = (C.c_int * 3)(*(list(g.dims) + [1] * (3 - g.ndim)))
    _check(lib().ehmg_layered_media(g.ndim, dims, float(gamma_phys), int(seed) & (2**64 - 1),
                                    lam.ctypes.data, mu.ctypes.data, rho.ctypes.data, gam.ctypes.data))
    return MediaModel(lam, mu, rho, gam)


def layered_grf_media(g: StaggeredGrid, seed: int, n_layers: int = 8, cs=(1.0, 2.5),
                      cp_over_cs=(1.7, 2.2), rho=(1.0, 2.5), perturbation: float = 0.1,
                      corr_cells: float = 20.0, gamma_phys: float = 0.01) -> MediaModel:
    """BASELINE configs[1]/[3]/[4] media: `n_layers` horizontal layers along the
    last axis (experiments.hpp:78 layout, index 0 at the top) with per-layer
    cs, cp/cs and rho drawn from the given ranges, each multiplied by its own
    smooth Gaussian random field (correlation length `corr_cells` cells)
    bounded to +-perturbation. Built on the device (csrc/ehmg_media.cuh),
    deterministic in `seed`; gamma = gamma_phys (apply a sponge afterwards)."""
    n = g.n_cells()
    lam, mu, rh, gam = (np.empty(n, np.float64) for _ in range(4))
    dims = (C.c_int * 3)(*(list(g.dims) + [1] * (3 - g.ndim)))
    rng = np.array([cs[0], cs[1], cp_over_cs[0], cp_over_cs[1], rho[0], rho[1]], np.float64)
    _check(lib().ehmg_layered_grf_media(g.ndim, dims, int(n_layers), rng.ctypes.data, float(perturbation),
                                        float(corr_cells), float(gamma_phys), int(seed) & (2**64 - 1),
                                        lam.ctypes.data, mu.ctypes.data, rh.ctypes.data, gam.ctypes.data))
    return MediaModel(lam, mu, rh, gam)


def min_interior_vs(g: StaggeredGrid, m: MediaModel, sponge: SpongeConfig) -> float:
    """experiments.hpp:116"""
    vs = m.vs().reshape(g.dims[::-1])
    L = sponge.layer_width
    sl = []
    for a in range(g.ndim - 1, -1, -1):
        top_free = (not sponge.absorb_top) and a == g.ndim - 1
        lo = 0 if top_free else L
        hi = g.dims[a] - L
        sl.append(slice(lo, max(lo, hi)))
    inner = vs[tuple(sl)]
    return float(inner.min()) if inner.size else float(vs.min())


def omega_from_gs(g: StaggeredGrid, m: MediaModel, g_s: float, sponge: SpongeConfig) -> float:
    """experiments.hpp:137 -- omega = 2 pi Vs_min / (g_s h)."""
    if not g_s > 2:
        raise ValueError("g_s must exceed 2 (Nyquist limit)")
    return 2 * math.pi * min_interior_vs(g, m, sponge) / (g_s * g.h)


def default_solve_damping(g_s: float, levels: int) -> float:
    """experiments.hpp:221"""
    if levels <= 2:
        return 0.55 if g_s >= 9 else 0.5
    if levels == 3:
        return 0.35
    return 0.25


def run_solve(cfg: dict, seed: int = 1) -> dict:
    """experiments.hpp:258 run_solve_dim (media: homogeneous / linear /
    layered(seed) or an explicit MediaModel under cfg['media']); `seed` is the
    CLI's --seed (tools/ehmg.cpp:22, default 1). Returns the summary dict."""
    import time
    dims = tuple(cfg.get("dims", (512, 128)))
    g = StaggeredGrid(dims, cfg.get("spacing", 1.0 / dims[-1]))
    sponge = SpongeConfig(cfg.get("sponge_cells", 20 if g.ndim == 2 else 8),
                          cfg.get("sponge_gamma_max", 1.0), cfg.get("absorb_top", False))
    gamma_phys = cfg.get("gamma", 0.01)
    if "media" in cfg:
        media = cfg["media"]
    else:
        problem = cfg.get("problem", "homogeneous")
        if problem == "homogeneous":
            media = MediaModel.homogeneous(g, cfg.get("lambda", 20.0), cfg.get("mu", 1.0),
                                           cfg.get("rho", 1.0), gamma_phys)
        elif problem == "linear":
            media = linear_media(g, gamma_phys)
        elif problem == "layered":
            media = layered_media(g, gamma_phys, seed)
        elif problem == "layered_grf":  # BASELINE configs[1]/[3] recipe (B200 addition)
            media = layered_grf_media(g, seed, corr_cells=cfg.get("corr_cells", 20.0), gamma_phys=gamma_phys)
        else:
            raise ValueError(f"config: unknown problem kind '{problem}'")
    media.gamma = build_attenuation_profile(g, gamma_phys, sponge)
    media.validate(g)
    g_s = cfg.get("g_s", 10.0)
    omega = cfg.get("omega", 0.0)
    if omega <= 0:
        omega = omega_from_gs(g, media, g_s, sponge)
    beta = cfg.get("beta", 2.0 / 3.0)
    alpha = cfg.get("alpha", 0.1)
    levels = cfg.get("levels", 2)
    w = cfg.get("w", default_solve_damping(g_s, levels))
    opt = MgOptions(n_levels=levels, cycle=cfg.get("cycle", "w"), nu1=cfg.get("nu1", 1),
                    nu2=cfg.get("nu2", 1), damping=w, vanka_mode=cfg.get("vanka", FULL),
                    sweep=cfg.get("order", RED_BLACK), coarse=cfg.get("coarse", "automatic"),
                    lu_dof_budget=cfg.get("lu_dof_budget", 4_000_000))
    precision = cfg.get("precision", "double")  # experiments.hpp:314
    if precision not in ("double", "mixed"):
        raise ValueError(f"config: unknown precision '{precision}'")
    D0 = make_opdata(g, media, OperatorParams(beta, omega, 0.0))
    mg = Multigrid(g, media, OperatorParams(beta, omega, alpha), opt, precision=precision)
    comp = cfg.get("source_component", g.ndim)
    src = cfg.get("source_index", middle_of_top_row(g))
    b = make_point_source(g, comp, src)
    x = np.zeros(g.n_dofs(), np.complex128)
    ko = KrylovOptions(cfg.get("restart", 5), cfg.get("max_iterations", 600), cfg.get("rtol", 1e-6))
    t0 = time.perf_counter()
    res = fgmres(D0, mg, b, x, ko)
    secs = time.perf_counter() - t0
    return dict(grid="x".join(map(str, dims)), beta=beta, g_s=g_s, levels=levels, alpha=alpha,
                w=w, omega=omega, precision=precision, iterations=res.iterations, final_relres=res.relres,
                wall_time_s=secs, status=res.status, history=res.history, solution=x)
