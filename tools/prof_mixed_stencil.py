import sys; sys.path.insert(0, '/root/repo')
import torch, bench, paper_2307_03242_b200 as E
g, med, omega = bench.build_problem(256, E)
opt = E.MgOptions(n_levels=5, cycle="v", nu1=1, nu2=1, damping=0.25, vanka_mode="full", sweep="red_black")
mg = E.Multigrid(g, med, E.OperatorParams(bench.BETA, omega, bench.ALPHA), opt, precision="mixed")
r = torch.randn(g.n_dofs(), dtype=torch.complex128, device="cuda"); z = torch.zeros_like(r)
mg.precondition(r, z); torch.cuda.synchronize(); print("ok")
