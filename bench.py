"""Headline benchmark: V-cycles/s (complex128) of the shifted-Laplacian
V(2,2) preconditioner at 257^3 nodes (256^3 cells) 3D elastic Helmholtz,
plus stencil GDOF/s and FGMRES time-to-1e-6 (BASELINE.json configs[2]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

One step = one preconditioner application z = M r (5 levels, 256^3 -> 16^3,
full red-black Vanka V(2,2), exact coarsest solve). `value` times K steps on
HBM-resident buffers with CUDA events on the solver stream; `e2e` times K
steps through the public API with pinned host buffers (every step's H2D of r
and D2H of z inside the timed region; `precondition_many` overlaps the copies
of neighbouring steps with the current cycle, `e2e.per_call` is one
synchronous call per step). Fields are 1.08 GB each, far larger than the
126 MB L2, so no explicit flush is needed between steps.
N > 1: one process per GPU, each running its own replica of the workload
(weak scaling; the z-slab decomposed hierarchy is DESIGN.md row (e)).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# workload: BASELINE.json configs[2]
# dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant
# kernel from one `ncu --set full` capture of the same residual at 256^3
# (distinct b and x; k_stencil3d_sp<8, 2>, profiles/round2/ncu_stencil3d_sp82_residual.txt:
# 11% above the algorithmic bytes: the 18 x 18 windows of the 14 x 14 tiles re-read their halo
# rows where the neighbouring tile's copy has left L2).
NCU_TRAFFIC = {"residual@L0": 3113847000 + 1063663000,
               "source": "profiles/round2/ncu_stencil3d_sp82_residual.txt (ncu --set full, 256^3 residual)"}
N_CELLS = 256
LEVELS = 5  # at 256^3: coarsest level 16^3 cells (17^3 nodes), BASELINE configs[2]


def levels_for(n):
    """levels coarsening n^3 cells down to 16^3 (the BASELINE's 17^3 nodes)"""
    return max(2, int(round(math.log2(n))) - 3)
BETA = 2.0 / 3.0
ALPHA = 0.5          # shift (the 0.1 default stalls at 5 levels)
DAMPING = 0.25       # experiments.hpp:221 default for >= 4 levels
AGG_N2 = 32          # z-slab mode: levels with <= 32 cell planes (< 65^3 nodes) are agglomerated
SPONGE = 24
GAMMA_PHYS = 0.01
LAM, MU, RHO = 2.0, 1.0, 1.0   # cs = 1, cp = 2
PPW = 10.0


def metric_name(n=256):
    return f"V-cycles/s (complex128) at {n + 1}^3 3D elastic Helmholtz"


def workload_config(n):
    return {"workload": f"configs[2]: 3D homogeneous {n + 1}^3 nodes ({n}^3 cells), h=1/{n}",
            "media": "lambda=2 mu=1 rho=1 (cs=1, cp=2)", "omega": f"2*pi/({PPW:g}h)",
            "sponge_cells": SPONGE, "gamma_phys": GAMMA_PHYS, "beta": BETA, "alpha": ALPHA,
            "cycle": "V(2,2) full red-black Vanka", "levels": levels_for(n),
            "coarsest": f"{n >> (levels_for(n) - 1)}^3 exact (LU-derived inverse in HBM)",
            "damping": DAMPING, "source": "unit point source, x-component, centre",
            "krylov": "FGMRES(10), rtol 1e-6",
            "l2": (f"inputs ({field_gb(n):.2f} GB/field) larger than the 126 MB L2" if field_gb(n) > 0.126
                   else f"inputs ({field_gb(n):.3f} GB/field) fit in L2: no flush between steps")}


def field_gb(n):
    """one complex128 field on n^3 cells (u0, u1, u2 faces + p)"""
    return 16 * (3 * n * n * (n + 1) + n ** 3) / 1e9


# ------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        cmd = ["nvidia-smi", "-i", str(self.index),
               "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
               "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
               "clocks_event_reasons.sw_power_cap,power.draw", "--format=csv,noheader,nounits",
               "-lms", "200"]
        try:
            self.proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                                         text=True)
        except OSError:
            self.proc = None
            return

        def rd():
            for line in self.proc.stdout:
                self.rows.append([s.strip() for s in line.split(",")])
        self.thread = threading.Thread(target=rd, daemon=True)
        self.thread.start()

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
                for nm, v in zip(names, r[2:6]):
                    if v.lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                pass
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------- dist
def dist_init(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist
        ndev = torch.cuda.device_count() if args.impl == "b200" else 0
        # NCCL needs distinct GPUs; several ranks sharing one GPU (smoke runs
        # of the multi-rank path) fall back to gloo for the bench plumbing.
        backend = "nccl" if ndev >= ws else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    return ws, rank, local


def spawn_ranks(n):
    """Re-launch this command as `python -m torch.distributed.run
    --nproc-per-node n` on 127.0.0.1 (a free port); rank 0 prints the line."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    print(f"bench: spawning {n} ranks: {' '.join(cmd)}", file=sys.stderr)
    return subprocess.call(cmd)


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(ws, v):
    if ws == 1:
        return v
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------- roofline bytes
def level_dims(dims, l):
    if isinstance(dims, int):
        dims = (dims,) * 3
    return tuple(d >> l for d in dims)


def ndofs(d):
    c = d[0] * d[1] * d[2]
    return c + sum(c // d[a] * (d[a] + 1) for a in range(3))


FACTOR_SETS = {}  # level -> distinct factor entry sets when the factor dictionary is active (0: per-cell cache)


def alg_bytes(kernel, n, level):
    """Algorithmic HBM bytes of one launch at a level;
    n = cube edge or the level-0 cell dims."""
    d = level_dims(n, level)
    C = d[0] * d[1] * d[2]
    N = ndofs(d)
    Nu = N - C
    if kernel == "residual":
        return 16 * 3 * N + 32 * C
    if kernel == "apply":
        return 16 * 2 * N + 32 * C
    if kernel == "vanka_update":
        if FACTOR_SETS.get(level, 0) > 0:
            # factor dictionary: a 4-byte id per colour cell (the table of distinct entry sets stays
            # on chip: FACTOR_SETS[level] x 208 bytes), r and x at the owned DOFs
            return 4 * (C // 2) + 16 * (Nu + C // 2) + 2 * 16 * (Nu + C // 2)
        if os.environ.get("EHMG_VANKA_KCACHE", "0")[:1] == "1":
            # colour-half of the stiffness cache (12 reals of K + 1/s per cell), rho and gamma of every
            # cell once (the mass part of the local blocks is rebuilt from them), r and x at the owned DOFs
            return 8 * 14 * (C // 2) + 16 * C + 16 * (Nu + C // 2) + 2 * 16 * (Nu + C // 2)
        # colour-half of the factor cache (13 complex per cell), r and x at the owned DOFs
        return 16 * 13 * (C // 2) + 16 * (Nu + C // 2) + 2 * 16 * (Nu + C // 2)
    if kernel == "restrict":
        return 16 * N + 16 * ndofs(level_dims(n, level + 1))
    if kernel == "prolong_add":
        return 16 * ndofs(level_dims(n, level + 1)) + 2 * 16 * N
    if kernel == "coarse_solve":  # S^-1 GEMV over the displacement DOFs + the rhs / pressure passes
        return 16 * Nu * Nu + 16 * (3 * N + Nu)
    return 0


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ------------------------------------------------------- CPU baseline
REF_SAMPLE_N = 64
REF_SAMPLE_LEVELS = 4
# one-time check of the DOF-ratio extrapolation against larger measured
# reference cycles (tools/ref_extrapolation.py on the GPU box's host cores)
REF_VALIDATION = ("single-core reference cycles measured at 32^3/3, 64^3/4 and 128^3/5 levels extrapolate "
                  "to 256^3 within +6.0% / +2.5% / 0 of each other, the 64^3 sample overestimating the "
                  "reference rate by 2.5% against the 128^3 measurement (profiles/round2/ref_extrapolation.json)")


def level_work(n, levels):
    """Sum of DOFs over the smoothed levels: V-cycle work scales with it."""
    return sum(ndofs(level_dims(n, l)) for l in range(levels - 1))


def cpu_sample_media(n):
    from oracle import oracle as O
    c = n ** 3
    gam = O.attenuation((n, n, n), GAMMA_PHYS, max(1, SPONGE * n // N_CELLS))
    return O.Media(np.full(c, LAM), np.full(c, MU), np.full(c, RHO), gam)


def run_cpu_sample(steps, threads, n=REF_SAMPLE_N, levels=None):
    """Reference V(2,2) cycles (oracle/_ref = the reference headers) on an
    n^3 cube with the same media/omega-per-h recipe, `threads` independent
    replicas in parallel (the reference is single-threaded). Returns
    (V-cycles/s extrapolated to N_CELLS^3, kind, raw seconds per sample
    cycle, wall seconds)."""
    from oracle import oracle as O
    kind = "reference" if O.ref_available() else "port"
    levels = levels or max(2, min(LEVELS, int(round(math.log2(n))) - 2))
    dims = (n, n, n)
    m = cpu_sample_media(n)
    omega = 2 * math.pi / (PPW / n)
    rng = np.random.default_rng(0)
    b = rng.standard_normal(O.n_dofs(dims)) + 1j * rng.standard_normal(O.n_dofs(dims))
    secs = []
    lock = threading.Lock()

    def work():
        if kind == "reference":
            _, s = O.ref_mg_cycles(dims, 1.0 / n, m, BETA, omega, ALPHA, b, np.zeros_like(b),
                                   ncycles=steps, n_levels=levels, cycle="v", nu1=2,
                                   nu2=2, damping=DAMPING)
        else:
            mg = O.MG(dims, 1.0 / n, m, BETA, omega, ALPHA, n_levels=levels, cycle="v",
                      nu1=2, nu2=2, damping=DAMPING)
            t0 = time.perf_counter()
            for _ in range(steps):
                mg.precondition(b)
            s = time.perf_counter() - t0
        with lock:
            secs.append(s / steps)

    ths = [threading.Thread(target=work) for _ in range(threads)]
    t0 = time.perf_counter()
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    wall = time.perf_counter() - t0
    per_cycle = max(secs)
    rate_sample = threads / per_cycle
    scale = level_work(n, levels) / level_work(N_CELLS, LEVELS)
    return rate_sample * scale, kind, per_cycle, wall, levels


# ------------------------------------------------------------ b200 arm
def build_problem(n, E):
    g = E.StaggeredGrid((n, n, n), 1.0 / n)
    med = E.MediaModel.homogeneous(g, LAM, MU, RHO, GAMMA_PHYS)
    med.gamma = E.build_attenuation_profile(g, GAMMA_PHYS, E.SpongeConfig(SPONGE))
    omega = 2 * math.pi * 1.0 / (PPW * g.h)
    return g, med, omega


class Problem:
    """One bench workload: grid, media, omega, hierarchy depth, source, and
    the line's metric/config (BASELINE configs[2] by default)."""

    def __init__(self, g, med, omega, levels, damping, source, metric, config, agg_n2=AGG_N2, scaling=None):
        self.g, self.med, self.omega, self.levels, self.damping = g, med, omega, levels, damping
        self.source, self.metric, self.config, self.agg_n2 = source, metric, config, agg_n2
        self.dims = tuple(g.dims)
        self.scaling = scaling


def make_problem(args, E, ws):
    if args.workload == "c2":
        n = args.n or N_CELLS
        g, med, omega = build_problem(n, E)
        return Problem(g, med, omega, levels_for(n), DAMPING, (0, (n // 2, n // 2, n // 2)), metric_name(n),
                       workload_config(n))
    from paper_2307_03242_b200 import configs as K
    if args.workload == "c3":
        n = args.n or 512
        w = K.config3(scale=512 // n)
        metric = f"V-cycles/s (complex128) at {n + 1}^3 3D heterogeneous elastic Helmholtz"
        wl = f"configs[3]: 3D heterogeneous {n + 1}^3 nodes ({n}^3 cells), layered + 3D GRF (seed {K.SEED})"
        scaling = "strong"
    else:  # c4w: weak scaling, 384 x 384 x 192 G cells on G GPUs
        scale = 384 // (args.n or 384)
        w = K.config4_weak(gpus=ws, scale=scale)
        d = w.grid.dims
        metric = f"V-cycles/s (complex128) weak scaling, {d[0] + 1}x{d[1] + 1}x(192*G/{scale}) nodes per G GPUs"
        wl = f"configs[4] weak: {d[0]}x{d[1]}x{d[2]} cells on {ws} GPU(s), layered + 3D GRF (seed {K.SEED})"
        scaling = "weak"
    d = w.grid.dims
    cfg = {"workload": wl, "media": "8 layers, cs in [1,2.5], cp/cs in [1.7,2.2], rho in [1,2.5], each x (1 +- 10% "
                                    "smooth GRF, correlation 20h); csrc/ehmg_media.cuh",
           "omega": f"{w.shifted.omega:.6g} (10 points per wavelength at the minimum interior cs)",
           "sponge_cells": w.sponge.layer_width, "gamma_phys": K.GAMMA_PHYS, "beta": K.BETA, "alpha": K.ALPHA,
           "cycle": "V(2,2) full red-black Vanka", "levels": w.mg.n_levels,
           "coarsest": "x".join(str(a >> (w.mg.n_levels - 1)) for a in d) + " exact (LU-derived inverse in HBM)",
           "damping": w.mg.damping, "source": w.notes, "krylov": "FGMRES(10), rtol 1e-6",
           "l2": "inputs larger than the 126 MB L2"}
    return Problem(w.grid, w.media, w.shifted.omega, w.mg.n_levels, w.mg.damping, w.sources[0], metric, cfg,
                   w.agg_n2, scaling)


def run_b200(args, ws, rank, local):
    import torch
    import paper_2307_03242_b200 as E
    torch.cuda.set_device(local)
    E.lib().ehmg_set_device(local)
    P = make_problem(args, E, 1)
    g, med, omega, n = P.g, P.med, P.omega, P.dims
    opt = E.MgOptions(n_levels=P.levels, cycle="v", nu1=2, nu2=2, damping=P.damping,
                      vanka_mode="full", sweep="red_black")
    t0 = time.perf_counter()
    mg = E.Multigrid(g, med, E.OperatorParams(BETA, omega, ALPHA), opt)
    D0 = E.make_opdata(g, med, E.OperatorParams(BETA, omega, 0.0))
    setup_s = time.perf_counter() - t0
    N = g.n_dofs()
    b = torch.from_numpy(E.make_point_source(g, *P.source)).cuda()
    gen = torch.Generator(device="cuda").manual_seed(1234 + rank)
    r = torch.randn(N, dtype=torch.complex128, device="cuda", generator=gen)
    z = torch.zeros(N, dtype=torch.complex128, device="cuda")
    stream = torch.cuda.ExternalStream(mg.stream)

    # warm-up
    for _ in range(args.warmup):
        mg.precondition(r, z)
    torch.cuda.synchronize()
    barrier(ws)
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    clk.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        mg.precondition(r, z)
    ev1.record(stream)
    torch.cuda.synchronize()
    clocks = clk.stop()
    barrier(ws)
    ms = ev0.elapsed_time(ev1)
    ms_max = max_over_ranks(ws, ms)
    value = ws * args.steps / (ms_max / 1e3)

    for lv in range(mg.n_levels()):
        FACTOR_SETS[lv] = mg.factor_sets(lv)
    # profile pass (same steps, per-launch events) -> dominant kernel
    E.profile_enable(True)
    for _ in range(args.steps):
        mg.precondition(r, z)
    torch.cuda.synchronize()
    prof = E.profile_report()
    E.profile_enable(False)
    launches_per_step = sum(c for (_, _, c, _) in prof) / args.steps
    top = max(prof, key=lambda t: t[3])
    peak, peak_src = load_peaks()
    kname, klev, kcount, kms = top
    avg_ms = kms / kcount
    nbytes = alg_bytes(kname, n, klev)
    achieved = nbytes / (avg_ms / 1e3) / 1e9
    # level-0 kernels for the record
    kernels = {f"{k}@L{lv}": {"avg_ms": round(t / c, 4), "count_per_step": c / args.steps,
                              "share": round(t / sum(p[3] for p in prof), 4),
                              "alg_GBps": round(alg_bytes(k, n, lv) / (t / c / 1e3) / 1e9, 1)}
               for (k, lv, c, t) in prof}

    # one red-black colour of the fine-level smoother = residual + Vanka update
    # (north_star's "smoother at >= 70% of HBM" read as the whole colour pass)
    smoother_pass = None
    kr, ku = kernels.get("residual@L0"), kernels.get("vanka_update@L0")
    if kr and ku:
        pb = alg_bytes("residual", n, 0) + alg_bytes("vanka_update", n, 0)
        pms = kr["avg_ms"] + ku["avg_ms"]
        smoother_pass = {"alg_bytes": pb, "ms": round(pms, 4), "GBps": round(pb / (pms / 1e3) / 1e9, 1),
                         "frac": round(pb / (pms / 1e3) / 1e9 / peak, 4),
                         "note": "residual@L0 + vanka_update@L0 per colour, algorithmic bytes of both"}

    # stencil throughput: the unshifted operator apply at full size
    y = torch.empty_like(r)
    for _ in range(3):
        E.apply_mixed_operator(D0, r, y)
    s0 = torch.cuda.ExternalStream(D0.stream)
    torch.cuda.synchronize()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    a0.record(s0)
    for _ in range(reps):
        E.apply_mixed_operator(D0, r, y)
    a1.record(s0)
    torch.cuda.synchronize()
    apply_ms = a0.elapsed_time(a1) / reps
    gdofs = N / (apply_ms / 1e3) / 1e9

    # e2e: public API with pinned host buffers (H2D r, D2H z per step).
    # precondition_many streams the steps' right-hand sides through the
    # preconditioner with the copies of neighbouring steps overlapping the
    # current cycle (the batched multi-source call); e2e_per_call times one
    # synchronous precondition() call per step.
    rh = torch.empty(N, dtype=torch.complex128, pin_memory=True)
    zh = [torch.empty(N, dtype=torch.complex128, pin_memory=True) for _ in range(2)]
    rh.copy_(r.cpu())
    rn, zn = rh.numpy(), [q.numpy() for q in zh]
    mg.precondition(rn, zn[0])
    mg.precondition_many([rn, rn], zn)
    barrier(ws)
    e_steps = max(2, args.steps)
    t0 = time.perf_counter()
    mg.precondition_many([rn] * e_steps, [zn[i & 1] for i in range(e_steps)])
    e2e_ms = max_over_ranks(ws, (time.perf_counter() - t0) * 1e3)
    e2e = ws * e_steps / (e2e_ms / 1e3)
    barrier(ws)
    c_steps = max(1, min(args.steps, 5))
    t0 = time.perf_counter()
    for _ in range(c_steps):
        mg.precondition(rn, zn[0])
    e2e1_ms = max_over_ranks(ws, (time.perf_counter() - t0) * 1e3)
    e2e_call = ws * c_steps / (e2e1_ms / 1e3)

    # GMRES time-to-1e-6 on the point-source problem (device buffers)
    solve = None
    free_b = torch.cuda.mem_get_info()[0]
    if args.solve and free_b < 16 * N * (2 * 10 + 6) * 1.05:
        solve = {"skipped": f"FGMRES(10) needs {16 * N * 26 / 1e9:.0f} GB beside the hierarchy; "
                            f"{free_b / 1e9:.0f} GB free on one GPU (the z-slab mode shards it)"}
    elif args.solve:
        # warm-up: a 20-iteration solve allocates the hierarchy's FGMRES
        # workspace and captures the cycle's CUDA graphs for its basis
        # buffers (one-time set-up, timed separately as warm_s)
        t0 = time.perf_counter()
        E.fgmres(D0, mg, b, torch.zeros(N, dtype=torch.complex128, device="cuda"),
                 E.KrylovOptions(restart=10, max_iterations=20, orthogonalization=args.orth))
        torch.cuda.synchronize()
        warm_s = time.perf_counter() - t0
        x = torch.zeros(N, dtype=torch.complex128, device="cuda")
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = E.fgmres(D0, mg, b, x, E.KrylovOptions(restart=10, max_iterations=args.max_it, orthogonalization=args.orth))
        torch.cuda.synchronize()
        ts = time.perf_counter() - t0
        solve = {"status": res.status, "iterations": res.iterations, "relres": res.relres,
                 "seconds": round(ts, 3), "s_per_iteration": round(ts / max(1, res.iterations), 5),
                 "orthogonalization": args.orth, "warm_s": round(warm_s, 3),
                 "note": "from x = 0 after a 20-iteration warm-up solve (workspace + graphs)"}

    # the reference's "precision": "mixed" mode (experiments.hpp:241): complex64
    # hierarchy behind the complex128 FGMRES -- reported beside the headline
    mixed = None
    if args.mixed:
        del mg  # the complex128 hierarchy is done: free HBM for the complex64 one
        mgm = E.Multigrid(g, med, E.OperatorParams(BETA, omega, ALPHA), opt, precision="mixed")
        for _ in range(args.warmup):
            mgm.precondition(r, z)
        sm = torch.cuda.ExternalStream(mgm.stream)
        torch.cuda.synchronize()
        m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        m0.record(sm)
        for _ in range(args.steps):
            mgm.precondition(r, z)
        m1.record(sm)
        torch.cuda.synchronize()
        mixed = {"v_cycles_per_s": round(args.steps / (m0.elapsed_time(m1) / 1e3), 4),
                 "note": "complex64 hierarchy, complex128 in/out (config 'precision': 'mixed')"}
        if args.solve:
            E.fgmres(D0, mgm, b, torch.zeros(N, dtype=torch.complex128, device="cuda"),
                     E.KrylovOptions(restart=10, max_iterations=20, orthogonalization=args.orth))  # warm-up
            x = torch.zeros(N, dtype=torch.complex128, device="cuda")
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = E.fgmres(D0, mgm, b, x, E.KrylovOptions(restart=10, max_iterations=args.max_it, orthogonalization=args.orth))
            torch.cuda.synchronize()
            ts = time.perf_counter() - t0
            mixed["gmres_time_to_1e-6"] = {"status": res.status, "iterations": res.iterations,
                                           "relres": res.relres, "seconds": round(ts, 3)}
        del mgm

    line = {
        "metric": P.metric, "value": round(value, 4), "unit": "V-cycles/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_max / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "complex128 (f64)",
        "data": f"synthetic ({P.config['workload'].split(':')[0]} media recipe; seeded residual)",
        "config": P.config,
        "e2e": {"value": round(e2e, 4), "unit": "V-cycles/s", "h2d_bytes_per_step": N * 16,
                "d2h_bytes_per_step": N * 16, "steps": e_steps,
                "api": "Multigrid.precondition_many (ehmg_multigrid_precondition_many): host r in, host z out "
                       "per step; copies of neighbouring steps overlap the current cycle",
                "per_call": round(e2e_call, 4)},
        "stencil_gdofs": round(gdofs, 3), "stencil_apply_ms": round(apply_ms, 4),
        "gmres_time_to_1e-6": solve, "mixed_precision": mixed, "setup_s": round(setup_s, 2),
        "gpu_launches": int(round(launches_per_step * args.steps)),
        "roofline": {"bound": "hbm", "kernel": f"{kname}@L{klev}", "achieved": round(achieved, 1),
                     "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "traffic": (NCU_TRAFFIC.get(f"{kname}@L{klev}")
                                 if args.workload == "c2" and n == (N_CELLS,) * 3 else None),
                     "traffic_source": NCU_TRAFFIC["source"], "alg_bytes_per_launch": nbytes,
                     "limiter": ("instruction issue at 2 warps/scheduler (8 warps x 255 registers, 2 rows per "
                                 "thread): 564 M warp instructions per launch (43% FP64, 20% LDS/SHFL) at IPC 1.91; "
                                 "each pipe alone would allow 0.44 ms (FP64, 2 issue cycles per warp DFMA), 0.65 ms "
                                 "(184 M shared-memory wavefronts) and 0.58 ms (HBM) -- the launch needs all three "
                                 "overlapped; stalls: 29% fixed-latency FP64 waits, 17% LDS/SHFL results, 6% block "
                                 "barrier (profiles/round2/ncu_stencil3d_sp82_residual.txt; DESIGN.md)"),
                     "avg_launch_ms": round(avg_ms, 4), "peak_source": peak_src},
        "kernels": kernels, "smoother_colour_pass_L0": smoother_pass, "clocks": clocks,
        "vanka_factor_sets": {f"L{lv}": c for lv, c in sorted(FACTOR_SETS.items())},
    }
    if rank == 0 and ws == 1 and not args.no_cpu and args.workload == "c2":
        rate, kind, per, wall, lv = run_cpu_sample(1, 1, args.ref_cells)
        line["cpu_baseline"] = {
            "value": rate, "unit": "V-cycles/s", "cores": 1, "kind": kind, "extrapolated": True,
            "sample": (f"one V(2,2) cycle of the reference on a {args.ref_cells}^3 cube "
                       f"({lv} levels, same media/omega*h/shift/damping), "
                       f"{per:.2f} s, extrapolated to {N_CELLS}^3 by smoothed-level DOF ratio "
                       f"(validated against measured 64^3 and 128^3 reference cycles: {REF_VALIDATION})")}
    return line


def run_b200_slabs(args, ws, rank, local):
    """N > 1: one z-slab per GPU (strong scaling of one V-cycle over the
    fixed 257^3 problem). Ghost planes move by CUDA-IPC peer copies over
    NVLink; levels below 65^3 nodes (<= 32^3 cells) are agglomerated
    (replicated on every rank), as BASELINE configs[3] states."""
    import torch
    import torch.distributed as dist
    import paper_2307_03242_b200 as E
    ndev = max(1, torch.cuda.device_count())
    dev = local % ndev
    torch.cuda.set_device(dev)
    E.lib().ehmg_set_device(dev)
    obj = [f"bench{os.getpid()}_{int(time.time() * 1e3) % 10**9}" if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    job = obj[0]
    P = make_problem(args, E, ws)
    g, med, omega = P.g, P.med, P.omega
    opt = E.MgOptions(n_levels=P.levels, cycle="v", nu1=2, nu2=2, damping=P.damping,
                      vanka_mode="full", sweep="red_black")
    t0 = time.perf_counter()
    d = E.DistributedSlabSolver(job, rank, ws, dev, g, med, E.OperatorParams(BETA, omega, ALPHA),
                                opt, agg_n2=P.agg_n2)
    setup_s = time.perf_counter() - t0
    # which device each rank's slab attached (CUDA-IPC inboxes of every peer)
    rank_devs = [None] * ws
    dist.all_gather_object(rank_devs, {"rank": rank, "device": dev, "window": list(d.window())})
    rng = np.random.default_rng(1234)
    N = g.n_dofs()
    r = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    d.time_precondition(r, args.warmup)
    barrier(ws)
    clk = ClockSampler(dev)
    clk.start()
    b0 = d.exchanged_bytes()
    ms = d.time_precondition(r, args.steps)
    halo = (d.exchanged_bytes() - b0) / args.steps
    clocks = clk.stop()
    ms_max = max_over_ranks(ws, ms)
    value = args.steps / (ms_max / 1e3)
    barrier(ws)
    # per-launch profile of one application on this rank -> launches per step
    # and the dominant kernel's roofline on this rank's window
    E.profile_enable(True)
    d.time_precondition(r, 1)
    prof = E.profile_report()
    E.profile_enable(False)
    launches_per_step = sum(c for (_, _, c, _) in prof)
    z0w, z1w, w0w, w1w = d.window()
    kname, klev, kcount, kms = max(prof, key=lambda t: t[3])
    wd = (P.dims[0] >> klev, P.dims[1] >> klev, max(1, (w1w - w0w) >> klev))
    C = wd[0] * wd[1] * wd[2]
    Nw = ndofs(wd)
    nbytes = {"residual": 16 * 3 * Nw + 32 * C, "apply": 16 * 2 * Nw + 32 * C,
              "vanka_update": 16 * 13 * (C // 2) + 3 * 16 * (Nw - C + C // 2)}.get(kname, 0)
    peak, peak_src = load_peaks()
    # an overlapped apply is split into interior + boundary-row launches:
    # count whole-window evaluations (V(2,2): 3 pre-smoothing applies after
    # the zero-start colour, 1 for the restriction, 4 post-smoothing)
    evals = {"residual": 8, "vanka_update": 8}.get(kname, kcount)
    per_eval = kms / evals
    achieved = nbytes / (per_eval / 1e3) / 1e9 if nbytes else 0.0
    roofline = {"bound": "hbm", "kernel": f"{kname}@L{klev} (rank-0 window {wd[0]}x{wd[1]}x{wd[2]})",
                "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": None,
                "alg_bytes_per_launch": nbytes, "avg_launch_ms": round(per_eval, 4),
                "launches_per_eval": round(kcount / evals, 2), "peak_source": peak_src}
    barrier(ws)
    e_steps = max(1, min(args.steps, 3))
    t0 = time.perf_counter()
    for _ in range(e_steps):
        d.precondition(r)
    e2e_ms = max_over_ranks(ws, (time.perf_counter() - t0) * 1e3)
    z0, z1, w0, w1 = d.window()
    solve = None
    if args.solve:
        b = E.make_point_source(g, *P.source)
        t0 = time.perf_counter()
        _, res = d.solve(b, E.KrylovOptions(restart=10, max_iterations=args.max_it, orthogonalization=args.orth))
        ts = max_over_ranks(ws, time.perf_counter() - t0)
        solve = {"status": res.status, "iterations": res.iterations, "relres": res.relres,
                 "seconds": round(ts, 3), "s_per_iteration": round(ts / max(1, res.iterations), 5)}
    d.close()
    cfg = dict(P.config)
    cfg["parallelism"] = f"z-slab x{ws} (levels with <= {P.agg_n2} cell planes agglomerated)"
    return {
        "metric": P.metric, "value": round(value, 4), "unit": "V-cycles/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 4),
        "higher_is_better": True, "scaling": P.scaling or "strong", "vs_baseline": None,
        "dtype": "complex128 (f64)", "data": f"synthetic ({cfg['workload'].split(':')[0]} media recipe)",
        "config": cfg,
        "e2e": {"value": round(e_steps / (e2e_ms / 1e3), 4), "unit": "V-cycles/s",
                "h2d_bytes_per_step": 16 * N // ws, "d2h_bytes_per_step": 16 * N // ws},
        "halo_bytes_per_step_rank0": int(halo), "slab_rank0": [z0, z1, w0, w1],
        "ipc_ranks_attached": rank_devs,
        # halo traffic against NVLink 5 (900 GB/s per direction per GPU): the
        # bandwidth the exchanges would need if spread over the whole cycle
        "halo_vs_nvlink": {"GBps_over_cycle": round(halo / (ms_max / args.steps / 1e3) / 1e9, 2),
                           "nvlink_GBps_per_direction": 900.0,
                           "frac": round(halo / (ms_max / args.steps / 1e3) / 1e9 / 900.0, 4)},
        "roofline": roofline,
        "gmres_time_to_1e-6": solve, "setup_s": round(setup_s, 2), "clocks": clocks,
        "gpu_launches": int(launches_per_step * args.steps),
    }


def run_b200_sources(args, ws, rank, local):
    """BASELINE configs[4] (second part): independent preconditioned FGMRES
    solves for surface point sources on the 257^3 grid with configs[3]'s
    media recipe (paper_2307_03242_b200/configs.py config4_sources),
    distributed across the GPUs (one hierarchy per GPU, sources round-robin,
    no data-path collective). value = solves/s."""
    import torch
    import paper_2307_03242_b200 as E
    from paper_2307_03242_b200 import configs as K
    ndev = max(1, torch.cuda.device_count())
    dev = local % ndev
    torch.cuda.set_device(dev)
    E.lib().ehmg_set_device(dev)
    w = K.config4_sources(args.sources, scale=256 // (args.n or 256))
    g = w.grid
    mg = E.Multigrid(g, w.media, w.shifted, w.mg)
    D0 = E.make_opdata(g, w.media, w.unshifted)
    N = g.n_dofs()
    mine = [k for k in range(len(w.sources)) if k % ws == rank]
    x = torch.zeros(N, dtype=torch.complex128, device="cuda")
    warm = torch.from_numpy(w.rhs(0)).cuda()
    # warm-up: workspace on the handle + the cycle's graphs for all basis buffers
    E.fgmres(D0, mg, warm, x, E.KrylovOptions(restart=10, max_iterations=20, orthogonalization=args.orth))
    barrier(ws)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    its, st, rr = [], [], []
    for k in mine:
        b = torch.from_numpy(w.rhs(k)).cuda()
        x.zero_()
        res = E.fgmres(D0, mg, b, x, E.KrylovOptions(restart=10, max_iterations=args.max_it, orthogonalization=args.orth))
        its.append(res.iterations)
        st.append(res.status)
        rr.append(res.relres)
    torch.cuda.synchronize()
    secs = max_over_ranks(ws, time.perf_counter() - t0)
    nsrc = len(w.sources)
    cfg = {"workload": f"configs[4] sources: {nsrc} surface point sources on {g.dims[0] + 1}^3, independent solves",
           "media": "configs[3] recipe (8 layers + 10% 3D GRF, seed 2023)", "omega": w.shifted.omega,
           "levels": w.mg.n_levels, "source": w.notes, "krylov": "FGMRES(10), rtol 1e-6",
           "parallelism": f"{ws} GPUs, sources round-robin (no data-path collective)"}
    return {"metric": "solves/s (FGMRES(10) to 1e-6, complex128)", "value": round(nsrc / secs, 5),
            "unit": "solves/s", "n_gpus": ws, "steps": nsrc, "warmup": 1,
            "ms_per_step": round(secs * 1e3 / max(1, nsrc), 2), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "complex128 (f64)",
            "data": "synthetic (configs[3] media recipe; surface point sources)", "config": cfg,
            "iterations_rank0": its, "status_rank0": sorted(set(st)), "max_relres_rank0": max(rr) if rr else None,
            "e2e": None, "gpu_launches": None}


def run_reference(args, ws, rank):
    if rank != 0:
        return None
    threads = max(1, os.cpu_count() or 1)
    if args.warmup > 0:  # page-in / thread start-up: one small cycle per replica
        run_cpu_sample(1, threads, 32)
    rate, kind, per, wall, lv = run_cpu_sample(args.steps, threads, args.ref_cells)
    return {
        "metric": metric_name(), "value": rate, "unit": "V-cycles/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup,
        # time of one extrapolated 256^3 cycle on the whole box (1 / value);
        # the measured sample cycle is cpu_baseline.sample_ms_per_cycle
        "ms_per_step": 1e3 / rate, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "complex128 (f64)", "data": "synthetic", "config": workload_config(N_CELLS),
        "impl": "reference", "extrapolated": True,
        "cpu_baseline": {"value": rate, "unit": "V-cycles/s", "cores": threads, "kind": kind,
                         "extrapolated": True, "sample_ms_per_cycle": round(per * 1e3, 2),
                         "sample": (f"{threads} concurrent replicas x {args.steps} V(2,2) cycles "
                                    f"of the reference (single-threaded) on a {args.ref_cells}^3 cube "
                                    f"({lv} levels), extrapolated to "
                                    f"{N_CELLS}^3 by smoothed-level DOF ratio; validation: {REF_VALIDATION}")},
        "e2e": {"value": rate, "unit": "V-cycles/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--cells", dest="n", type=int, default=None,
                    help="cube edge in cells (c2 default 256, c3 512; c4w: the 384 edge, z = n/2 per GPU)")
    ap.add_argument("--workload", choices=["c2", "c3", "c4w"], default="c2",
                    help="c2 = BASELINE configs[2] (headline), c3 = configs[3] heterogeneous 513^3, "
                         "c4w = configs[4] weak scaling 384x384x192G")
    ap.add_argument("--solve", type=int, default=1)
    ap.add_argument("--mixed", type=int, default=1, help="also time the complex64-hierarchy mode")
    ap.add_argument("--max-it", type=int, default=None,
                    help="FGMRES iteration cap (default 600 for c2, 3000 for the heterogeneous workloads)")
    ap.add_argument("--orth", choices=["classical", "modified"], default="classical",
                    help="FGMRES Arnoldi variant (modified = the reference's MGS order)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--ref-cells", type=int, default=REF_SAMPLE_N,
                    help="reference arm / cpu_baseline: cube edge of the measured reference sample")
    ap.add_argument("--sources", type=int, default=32, help="--mode sources: number of point sources")
    ap.add_argument("--mode", choices=["slabs", "replicas", "sources"], default="slabs",
                    help="N > 1: z-slab decomposition (strong) or independent replicas (weak)")
    args = ap.parse_args()
    if args.max_it is None:
        args.max_it = 600 if (args.workload == "c2" and args.mode != "sources") else 3000
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # launched directly with --gpus N: start the N ranks ourselves (one
        # process per GPU), exactly as the driver's torchrun line would
        sys.exit(spawn_ranks(args.gpus))
    ws_env = int(os.environ.get("WORLD_SIZE", "1"))
    if ws_env != args.gpus:
        print(json.dumps({"error": f"WORLD_SIZE={ws_env} but --gpus {args.gpus}: launch one rank per GPU"}))
        sys.exit(2)
    ws, rank, local = dist_init(args)
    if args.impl == "reference":
        line = run_reference(args, ws, rank)
    elif args.mode == "sources":
        line = run_b200_sources(args, ws, rank, local)
    elif ws > 1 and args.mode == "slabs":
        line = run_b200_slabs(args, ws, rank, local)
    else:
        line = run_b200(args, ws, rank, local)
    if rank == 0 and line is not None:
        print(json.dumps(line))
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
