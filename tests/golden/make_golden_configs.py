"""Golden fixtures for BASELINE's own configurations, produced by the
REFERENCE's components (oracle/_ref: the reference headers; the cycle is
restated around them with an exact coarsest LU, ref_driver.cpp).

    python tests/golden/make_golden_configs.py      # ~5 min, 3 processes

Writes tests/golden/golden_configs.npz:
  cycle5_*  one 5-level V(2,2) preconditioner application on 64^3 cells with
            the bench's parameters (configs[2] recipe at 1/4 scale: beta 2/3,
            alpha 0.5, damping 0.25, lambda 2 mu 1 rho 1, 6-cell sponge, full
            red-black Vanka, coarsest 4^3); input r from a seeded generator
            (first values stored to detect drift), output sampled at 8192
            seeded indices plus its 2-norm and sum (the vectors are 17 MB);
  c0_*      configs[0] (2D 256^2 cells, 5 levels, FGMRES(10) to 1e-6) with
            alpha 0.5 (status, iterations, relres, sampled solution) and with
            the reference default alpha 0.1 (status, iterations: it stalls);
  c1_*      configs[1]'s layered + GRF recipe at 1/8 scale (128^2, 4 levels,
            correlation 2.5 cells, 4-cell sponge), FGMRES(10) to 1e-6;
  c3s_*     configs[3]'s 3D recipe at 1/16 scale (32^3, 3 levels, 8^3
            coarsest, correlation 1.25 cells, 2-cell sponge), FGMRES(10).
The media of c1 come from the C restatement of the recipe
(oracle og_layered_grf_media), which the GPU tests pin bit for bit to the
device builder.
"""
import os
import sys
from concurrent.futures import ProcessPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
OUT = os.path.join(HERE, "golden_configs.npz")
NSAMP = 8192


def oracle_grf(g, corr):
    import paper_2307_03242_b200 as E
    from oracle import oracle as O
    from paper_2307_03242_b200 import configs as K
    m = O.layered_grf_media(g.dims, K.SEED, corr_cells=corr, gamma_phys=K.GAMMA_PHYS)
    return E.MediaModel(*m.arrays())


def workload(which):
    from paper_2307_03242_b200 import configs as K
    K.grf_media = oracle_grf  # host restatement (bit-identical to the device builder)
    if which == "c0":
        return K.config0()
    if which == "c1":
        return K.config1(scale=8)
    if which == "c3s":
        return K.config3(scale=16, levels=3)
    return K.config2(scale=4, levels=5)


def cycle5_input(n):
    rng = np.random.default_rng(64064)
    return rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)


def sample_idx(n, seed):
    return np.sort(np.random.default_rng(seed).choice(n, NSAMP, replace=False))


def media_of(w):
    from oracle import oracle as O
    m = w.media
    return O.Media(m.lambda_, m.mu, m.rho, m.gamma)


def run(job):
    from oracle import oracle as O
    which, alpha = job
    w = workload("c2" if which == "cycle5" else which)
    g = w.grid
    m = media_of(w)
    out = {}
    if which == "cycle5":
        r = cycle5_input(g.n_dofs())
        z, _ = O.ref_mg_cycles(g.dims, g.h, m, w.shifted.beta, w.shifted.omega, w.shifted.alpha, r,
                               np.zeros_like(r), ncycles=1, n_levels=w.mg.n_levels, cycle="v", nu1=2, nu2=2,
                               damping=w.mg.damping, vanka="full", sweep="red_black")
        idx = sample_idx(g.n_dofs(), 1)
        out = {"cycle5_r_head": r[:16], "cycle5_idx": idx, "cycle5_z": z[idx],
               "cycle5_norm": np.linalg.norm(z), "cycle5_sum": z.sum(), "cycle5_levels": w.mg.n_levels,
               "cycle5_damping": w.mg.damping}
        return out
    b = w.rhs(0)
    a = w.shifted.alpha if alpha is None else alpha
    x, info = O.ref_solve(g.dims, g.h, m, w.shifted.beta, w.shifted.omega, a, b, n_levels=w.mg.n_levels,
                          cycle="v", nu1=2, nu2=2, damping=w.mg.damping, vanka="full", sweep="red_black",
                          restart=10, max_iterations=2000 if alpha is None else 700)
    tag = which if alpha is None else f"{which}_a01"
    out[f"{tag}_iterations"] = info["iterations"]
    out[f"{tag}_status"] = info["status"]
    out[f"{tag}_relres"] = info["relres"]
    out[f"{tag}_omega"] = w.shifted.omega
    if alpha is None:
        idx = sample_idx(g.n_dofs(), 2)
        out[f"{tag}_idx"] = idx
        out[f"{tag}_x"] = x[idx]
        out[f"{tag}_xnorm"] = np.linalg.norm(x)
    return out


if __name__ == "__main__":
    jobs = [("cycle5", None), ("c0", None), ("c0", 0.1), ("c1", None), ("c3s", None)]
    if len(sys.argv) > 1:  # regenerate only the named jobs, keep the others
        jobs = [j for j in jobs if j[0] in sys.argv[1:]]
    res = dict(np.load(OUT)) if os.path.exists(OUT) and len(sys.argv) > 1 else {}
    with ProcessPoolExecutor(len(jobs)) as ex:
        for d in ex.map(run, jobs):
            res.update(d)
    np.savez_compressed(OUT, **{k: np.asarray(v) for k, v in res.items()})
    for k, v in sorted(res.items()):
        if np.ndim(v) == 0:
            print(k, v)
