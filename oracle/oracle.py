"""ctypes bindings for the CPU ORACLE (test infrastructure only).

Two libraries, both CPU-only and both used ONLY as checkers by tests/,
``__graft_entry__.smoke()`` and bench.py's cpu-baseline / reference arm:

* ``build/libehmg_oracle.so`` -- the C restatement in ehmg_oracle.c.
* ``_ref/libehmg_ref.so``     -- the reference's own headers compiled in
  place (oracle/Makefile); present wherever it was built (it travels with
  the repo snapshot to the GPU box).

Fields are complex128 numpy arrays in the reference flatten() order.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "libehmg_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libehmg_ref.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_cp = np.ctypeslib.ndpointer(dtype=np.complex128, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


# --------------------------------------------------------------- geometry
def n_cells(dims) -> int:
    return int(np.prod(dims))


def comp_shapes(dims):
    """Per-component shapes (axis-0 fastest) in flatten() order."""
    nd = len(dims)
    out = []
    for k in range(nd):
        d = list(dims)
        d[k] += 1
        out.append(tuple(d))
    out.append(tuple(dims))
    return out


def n_dofs(dims) -> int:
    return sum(int(np.prod(s)) for s in comp_shapes(dims))


def split(x, dims):
    """Split a flat field into per-component arrays indexed [i0, i1(, i2)]."""
    parts, o = [], 0
    for s in comp_shapes(dims):
        n = int(np.prod(s))
        parts.append(x[o:o + n].reshape(s[::-1]).transpose())
        o += n
    return parts


# ----------------------------------------------------------------- oracle
class _KOpts(C.Structure):
    _fields_ = [("restart", C.c_int), ("max_iterations", C.c_int), ("rtol", C.c_double),
                ("stall_factor", C.c_double), ("stall_cycles", C.c_int)]


class _KRes(C.Structure):
    _fields_ = [("status", C.c_int), ("iterations", C.c_int), ("relres", C.c_double),
                ("n_history", C.c_int), ("history", C.POINTER(C.c_double))]


class _MgOpts(C.Structure):
    _fields_ = [("n_levels", C.c_int), ("cycle", C.c_int), ("nu1", C.c_int), ("nu2", C.c_int),
                ("damping", C.c_double), ("vanka_mode", C.c_int), ("sweep", C.c_int),
                ("k_inner_iterations", C.c_int), ("k_inner_rtol", C.c_double)]


STATUS = {0: "converged", 1: "max_iterations", 2: "breakdown", 3: "stalled"}
CYCLES = {"two_grid": 0, "v": 1, "w": 2, "k": 3}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        L.og_op_create.restype = C.c_void_p
        L.og_op_create.argtypes = [C.c_int, _ip, C.c_double, _dp, _dp, _dp, _dp, C.c_double,
                                   C.c_double, C.c_double]
        L.og_op_destroy.argtypes = [C.c_void_p]
        L.og_apply.argtypes = [C.c_void_p, _cp, _cp]
        L.og_schur_apply.argtypes = [C.c_void_p, _cp, _cp]
        L.og_assemble_dense.argtypes = [C.c_void_p, _cp]
        L.og_vanka_create.restype = C.c_void_p
        L.og_vanka_create.argtypes = [C.c_void_p, C.c_int]
        L.og_vanka_destroy.argtypes = [C.c_void_p]
        L.og_vanka_per_cell.argtypes = [C.c_void_p]
        L.og_vanka_cache.restype = C.c_void_p
        L.og_vanka_cache.argtypes = [C.c_void_p]
        L.og_vanka_sweep.argtypes = [C.c_void_p, C.c_void_p, _cp, _cp, C.c_double, C.c_int]
        L.og_restrict.argtypes = [C.c_int, _ip, _cp, _cp]
        L.og_prolong.argtypes = [C.c_int, _ip, _cp, _cp]
        L.og_coarsen_cell_field.argtypes = [C.c_int, _ip, _dp, _dp]
        L.og_attenuation_profile.argtypes = [C.c_int, _ip, C.c_double, C.c_int, C.c_double,
                                             C.c_int, _dp]
        L.og_mg_create.restype = C.c_void_p
        L.og_mg_create.argtypes = [C.c_int, _ip, C.c_double, _dp, _dp, _dp, _dp, C.c_double,
                                   C.c_double, C.c_double, C.POINTER(_MgOpts)]
        L.og_mg_destroy.argtypes = [C.c_void_p]
        L.og_mg_cycle.argtypes = [C.c_void_p, _cp, _cp]
        L.og_mg_precondition.argtypes = [C.c_void_p, _cp, _cp]
        L.og_mg_level_op.restype = C.c_void_p
        L.og_mg_level_op.argtypes = [C.c_void_p, C.c_int]
        L.og_solve.argtypes = [C.c_void_p, C.c_void_p, _cp, _cp, C.POINTER(_KOpts),
                               C.POINTER(_KRes)]
        L.og_free.argtypes = [C.c_void_p]
        L.og_layered_grf_media.argtypes = [C.c_int, _ip, C.c_int, _dp, C.c_double, C.c_double,
                                           C.c_double, C.c_uint64, _dp, _dp, _dp, _dp]
        _lib = L
    return _lib


def _dims(d):
    a = np.zeros(3, np.int32)
    a[:len(d)] = d
    return a


class Media:
    """Cell-centred media (lambda, mu, rho, gamma), flat axis-0-fastest."""

    def __init__(self, lam, mu, rho, gamma):
        self.lam = np.ascontiguousarray(lam, np.float64)
        self.mu = np.ascontiguousarray(mu, np.float64)
        self.rho = np.ascontiguousarray(rho, np.float64)
        self.gamma = np.ascontiguousarray(gamma, np.float64)

    def arrays(self):
        return self.lam, self.mu, self.rho, self.gamma


class Op:
    """OpData + apply (operator.hpp:76/:437)."""

    def __init__(self, dims, h, media: Media, beta, omega, alpha):
        self.dims = tuple(dims)
        self.n = n_dofs(dims)
        self.h = lib().og_op_create(len(dims), _dims(dims), h, *media.arrays(), beta, omega, alpha)

    def __del__(self):
        if _lib is not None and getattr(self, "h", None):
            _lib.og_op_destroy(self.h)

    def apply(self, x):
        y = np.zeros(self.n, np.complex128)
        lib().og_apply(self.h, np.ascontiguousarray(x, np.complex128), y)
        return y

    def schur(self, x):
        y = np.zeros(self.n, np.complex128)
        lib().og_schur_apply(self.h, np.ascontiguousarray(x, np.complex128), y)
        return y

    def dense(self):
        A = np.zeros(self.n * self.n, np.complex128)
        lib().og_assemble_dense(self.h, A)
        return A.reshape(self.n, self.n).T  # stored column-major


class Vanka:
    def __init__(self, op: Op, mode: int):
        self.op = op
        self.h = lib().og_vanka_create(op.h, mode)

    def __del__(self):
        if _lib is not None and getattr(self, "h", None):
            _lib.og_vanka_destroy(self.h)

    def cache(self):
        L = lib()
        stride = L.og_vanka_per_cell(self.h)
        n = n_cells(self.op.dims) * stride
        p = L.og_vanka_cache(self.h)
        buf = (C.c_double * (2 * n)).from_address(p)
        return np.frombuffer(buf, np.float64).copy().view(np.complex128).reshape(-1, stride)

    def sweep(self, b, x, w, order):
        x = np.array(x, np.complex128, copy=True)
        lib().og_vanka_sweep(self.h, self.op.h, np.ascontiguousarray(b, np.complex128), x, w,
                             order)
        return x


def restrict(dims_f, xf):
    dc = [d // 2 for d in dims_f]
    xc = np.zeros(n_dofs(dc), np.complex128)
    lib().og_restrict(len(dims_f), _dims(dims_f), np.ascontiguousarray(xf, np.complex128), xc)
    return xc


def prolong(dims_f, xc):
    xf = np.zeros(n_dofs(dims_f), np.complex128)
    lib().og_prolong(len(dims_f), _dims(dims_f), np.ascontiguousarray(xc, np.complex128), xf)
    return xf


def coarsen(dims_f, v):
    dc = [d // 2 for d in dims_f]
    out = np.zeros(n_cells(dc), np.float64)
    lib().og_coarsen_cell_field(len(dims_f), _dims(dims_f), np.ascontiguousarray(v, np.float64),
                                out)
    return out


def attenuation(dims, gamma_phys, width, gamma_max=1.0, absorb_top=False):
    out = np.zeros(n_cells(dims), np.float64)
    rc = lib().og_attenuation_profile(len(dims), _dims(dims), gamma_phys, width, gamma_max,
                                      int(absorb_top), out)
    if rc != 0:
        raise ValueError("sponge: invalid layer width")
    return out


class MG:
    """Multigrid hierarchy with exact coarsest solve (multigrid.hpp:70)."""

    def __init__(self, dims, h, media: Media, beta, omega, alpha, n_levels=2, cycle="v", nu1=1,
                 nu2=1, damping=0.75, vanka="full", sweep="red_black", k_inner_iterations=2,
                 k_inner_rtol=0.25):
        o = _MgOpts(n_levels, CYCLES[cycle], nu1, nu2, damping, 0 if vanka == "full" else 1,
                    1 if sweep == "red_black" else 0, k_inner_iterations, k_inner_rtol)
        self.dims = tuple(dims)
        self.n = n_dofs(dims)
        self.h = lib().og_mg_create(len(dims), _dims(dims), h, *media.arrays(), beta, omega,
                                    alpha, C.byref(o))
        if not self.h:
            raise ValueError("multigrid: invalid options or grid cannot support levels")

    def __del__(self):
        if _lib is not None and getattr(self, "h", None):
            _lib.og_mg_destroy(self.h)

    def cycle(self, b, x):
        x = np.array(x, np.complex128, copy=True)
        lib().og_mg_cycle(self.h, np.ascontiguousarray(b, np.complex128), x)
        return x

    def precondition(self, r):
        z = np.zeros(self.n, np.complex128)
        lib().og_mg_precondition(self.h, np.ascontiguousarray(r, np.complex128), z)
        return z

    def solve(self, A0: Op, b, restart=5, max_iterations=600, rtol=1e-6):
        x = np.zeros(self.n, np.complex128)
        ko = _KOpts(restart, max_iterations, rtol, 0.99, 2)
        kr = _KRes()
        lib().og_solve(self.h, A0.h, np.ascontiguousarray(b, np.complex128), x, C.byref(ko),
                       C.byref(kr))
        hist = [kr.history[i] for i in range(kr.n_history)]
        lib().og_free(C.cast(kr.history, C.c_void_p))
        return x, dict(status=STATUS[kr.status], iterations=kr.iterations, relres=kr.relres,
                       history=hist)


# ------------------------------------------------------- reference (_ref)
_ref = None


def layered_grf_media(dims, seed, n_layers=8, cs=(1.0, 2.5), cp_over_cs=(1.7, 2.2), rho=(1.0, 2.5),
                      perturbation=0.1, corr_cells=20.0, gamma_phys=0.01):
    """BASELINE configs[1]/[3]/[4] media recipe, restated in C (og_layered_grf_media)."""
    n = n_cells(dims)
    out = [np.empty(n, np.float64) for _ in range(4)]
    rng = np.array([cs[0], cs[1], cp_over_cs[0], cp_over_cs[1], rho[0], rho[1]], np.float64)
    rc = lib().og_layered_grf_media(len(dims), _dims(dims), int(n_layers), rng, float(perturbation),
                                    float(corr_cells), float(gamma_phys), int(seed) & (2**64 - 1), *out)
    if rc != 0:
        raise ValueError("layered_grf_media: bad arguments")
    return Media(*out)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        L = C.CDLL(REF_SO)
        common = [C.c_int, _ip, C.c_double, _dp, _dp, _dp, _dp, C.c_double, C.c_double,
                  C.c_double]
        L.ref_apply.argtypes = common + [_cp, _cp]
        L.ref_schur_apply.argtypes = common + [_cp, _cp]
        L.ref_vanka.argtypes = common + [C.c_int, C.c_int, C.c_double, C.c_int, _cp, _cp,
                                         C.c_void_p]
        L.ref_transfer.argtypes = [C.c_int, _ip, C.c_int, _cp, _cp]
        L.ref_coarsen.argtypes = [C.c_int, _ip, _dp, _dp]
        L.ref_attenuation.argtypes = [C.c_int, _ip, C.c_double, C.c_int, C.c_double, C.c_int, _dp]
        L.ref_mg_cycles.argtypes = common + [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                             C.c_int, C.c_int, C.c_int, _cp, _cp,
                                             C.POINTER(C.c_double)]
        L.ref_solve.argtypes = common + [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                         C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, _cp, _cp,
                                         C.POINTER(C.c_int), C.POINTER(C.c_int),
                                         C.POINTER(C.c_double), _dp, C.c_int, C.POINTER(C.c_int)]
        L.ref_solve_mixed.argtypes = L.ref_solve.argtypes
        L.ref_measure.argtypes = common + [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int,
                                           C.c_uint64, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int,
                                           C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                           _dp, C.c_int, C.POINTER(C.c_int)]
        _ref = L
    return _ref


def _chk(rc):
    if rc != 0:
        raise RuntimeError("reference call failed")


def ref_apply(dims, h, media, beta, omega, alpha, x, schur=False):
    y = np.zeros(n_dofs(dims), np.complex128)
    f = ref().ref_schur_apply if schur else ref().ref_apply
    _chk(f(len(dims), _dims(dims), h, *media.arrays(), beta, omega, alpha,
           np.ascontiguousarray(x, np.complex128), y))
    return y


def ref_vanka(dims, h, media, beta, omega, alpha, mode, order, w, nsweeps, b, x):
    x = np.array(x, np.complex128, copy=True)
    stride = len(dims) * ((4 if mode == 0 else 2) + 4) + 1
    cache = np.zeros(n_cells(dims) * stride, np.complex128)
    _chk(ref().ref_vanka(len(dims), _dims(dims), h, *media.arrays(), beta, omega, alpha, mode,
                         order, w, nsweeps, np.ascontiguousarray(b, np.complex128), x,
                         cache.ctypes.data))
    return x, cache.reshape(-1, stride)


def ref_transfer(dims_f, restricting, x):
    dc = [d // 2 for d in dims_f]
    out = np.zeros(n_dofs(dc if restricting else dims_f), np.complex128)
    _chk(ref().ref_transfer(len(dims_f), _dims(dims_f), int(restricting),
                            np.ascontiguousarray(x, np.complex128), out))
    return out


def ref_coarsen(dims_f, v):
    dc = [d // 2 for d in dims_f]
    out = np.zeros(n_cells(dc), np.float64)
    _chk(ref().ref_coarsen(len(dims_f), _dims(dims_f), np.ascontiguousarray(v, np.float64), out))
    return out


def ref_attenuation(dims, gamma_phys, width, gamma_max=1.0, absorb_top=False):
    out = np.zeros(n_cells(dims), np.float64)
    _chk(ref().ref_attenuation(len(dims), _dims(dims), gamma_phys, width, gamma_max,
                               int(absorb_top), out))
    return out


def ref_mg_cycles(dims, h, media, beta, omega, alpha, b, x, ncycles=1, n_levels=2, cycle="v",
                  nu1=1, nu2=1, damping=0.75, vanka="full", sweep="red_black"):
    x = np.array(x, np.complex128, copy=True)
    sec = C.c_double(0)
    _chk(ref().ref_mg_cycles(len(dims), _dims(dims), h, *media.arrays(), beta, omega, alpha,
                             n_levels, CYCLES[cycle], nu1, nu2, damping,
                             0 if vanka == "full" else 1, 1 if sweep == "red_black" else 0,
                             ncycles, np.ascontiguousarray(b, np.complex128), x, C.byref(sec)))
    return x, sec.value


def ref_solve(dims, h, media, beta, omega, alpha, b, n_levels=2, cycle="v", nu1=1, nu2=1,
              damping=0.75, vanka="full", sweep="red_black", restart=5, max_iterations=600,
              rtol=1e-6, precision="double"):
    """The reference's solve (experiments.hpp:313); precision "mixed" runs the
    reference float hierarchy behind a double FGMRES (MixedPrecondition)."""
    x = np.zeros(n_dofs(dims), np.complex128)
    it, st, nh = C.c_int(0), C.c_int(0), C.c_int(0)
    rr = C.c_double(0)
    hist = np.zeros(max_iterations + 64, np.float64)
    fn = ref().ref_solve_mixed if precision == "mixed" else ref().ref_solve
    _chk(fn(len(dims), _dims(dims), h, *media.arrays(), beta, omega, alpha,
                         n_levels, CYCLES[cycle], nu1, nu2, damping, 0 if vanka == "full" else 1,
                         1 if sweep == "red_black" else 0, restart, max_iterations, rtol,
                         np.ascontiguousarray(b, np.complex128), x, C.byref(it), C.byref(st),
                         C.byref(rr), hist, len(hist), C.byref(nh)))
    return x, dict(status=STATUS[st.value], iterations=it.value, relres=rr.value,
                   history=list(hist[:min(nh.value, len(hist))]))


def ref_measure(dims, h, media, beta, omega, alpha, seed, n_levels=2, cycle="v", nu1=1, nu2=1,
                damping=0.75, vanka="economic", sweep="lexicographic", warmup=5, tol=1e-9,
                max_cycles=500, growth_limit=20, precision="double"):
    """multigrid.hpp:143 measure_convergence_factor of the reference (restated
    driver loop around the reference's cycle components)."""
    f, cy, dv, nh = C.c_double(0), C.c_int(0), C.c_int(0), C.c_int(0)
    hist = np.zeros(max_cycles + 8, np.float64)
    _chk(ref().ref_measure(len(dims), _dims(dims), h, *media.arrays(), beta, omega, alpha, n_levels,
                           CYCLES[cycle], nu1, nu2, damping, 0 if vanka == "full" else 1,
                           1 if sweep == "red_black" else 0, seed, warmup, tol, max_cycles, growth_limit,
                           1 if precision == "mixed" else 0, C.byref(f), C.byref(cy), C.byref(dv), hist,
                           len(hist), C.byref(nh)))
    return dict(factor=f.value, cycles=cy.value, diverged=bool(dv.value),
                history=list(hist[:min(nh.value, len(hist))]))
