"""A/B of the FGMRES Arnoldi variants at the bench size (BASELINE configs[2],
257^3, complex128 and mixed): classical passes (default) vs the reference's
MGS order. Prints one JSON line per variant. Run on a B200 box."""
import json, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench as B
import paper_2307_03242_b200 as E

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
g, med, omega = B.build_problem(n, E)
opt = E.MgOptions(n_levels=B.levels_for(n), cycle="v", nu1=2, nu2=2, damping=B.DAMPING,
                  vanka_mode="full", sweep="red_black")
D0 = E.make_opdata(g, med, E.OperatorParams(B.BETA, omega, 0.0))
b = torch.from_numpy(E.make_point_source(g, 0, (n // 2, n // 2, n // 2))).cuda()
for prec in ["double", "mixed"]:
    mg = E.Multigrid(g, med, E.OperatorParams(B.BETA, omega, B.ALPHA), opt, precision=prec)
    xw = torch.zeros_like(b)
    E.fgmres(D0, mg, b, xw, E.KrylovOptions(restart=10, max_iterations=12))  # graphs, lazy setup
    for orth in ["classical", "modified", "classical"]:
        x = torch.zeros_like(b)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = E.fgmres(D0, mg, b, x, E.KrylovOptions(restart=10, max_iterations=600, orthogonalization=orth))
        torch.cuda.synchronize()
        ts = time.perf_counter() - t0
        print(json.dumps({"n": n, "precision": prec, "orth": orth, "status": res.status,
                          "iterations": res.iterations, "relres": res.relres, "seconds": round(ts, 3),
                          "s_per_iteration": round(ts / max(1, res.iterations), 5)}), flush=True)
    del mg
