"""Convergence of FGMRES(10) + V(2,2) for the heterogeneous workloads with
different source placements (configs[3]/[4] media recipe), on the GPU."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2307_03242_b200 as E  # noqa: E402
from paper_2307_03242_b200 import configs as K  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w = K.config4_sources(1, scale=scale)
g = w.grid
n = g.dims[0]
mg = E.Multigrid(g, w.media, w.shifted, w.mg)
D0 = E.make_opdata(g, w.media, w.unshifted)
cases = [("u2 face z=0 (surface)", 2, (n // 2, n // 2, 0)), ("u2 face z=1", 2, (n // 2, n // 2, 1)),
         ("u2 face z=2", 2, (n // 2, n // 2, 2)), ("p cell z=0 (reference default)", 3, (n // 2, n // 2, 0)),
         ("u0 face z=0", 0, (n // 2, n // 2, 0)), ("u2 centre", 2, (n // 2, n // 2, n // 2))]
for name, comp, idx in cases:
    b = torch.from_numpy(E.make_point_source(g, comp, idx)).cuda()
    x = torch.zeros_like(b)
    t0 = time.perf_counter()
    res = E.fgmres(D0, mg, b, x, E.KrylovOptions(restart=10, max_iterations=3000))
    torch.cuda.synchronize()
    h = res.history
    print(json.dumps({"n": n, "source": name, "status": res.status, "iterations": res.iterations,
                      "relres": res.relres, "s": round(time.perf_counter() - t0, 2),
                      "relres_at": {k: h[k] for k in (100, 300, 600, 1000, 2000) if k < len(h)}}), flush=True)
