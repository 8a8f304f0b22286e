import sys, numpy as np, torch
sys.path.insert(0, '.')
from oracle import oracle as orc
from paper_1809_01948_b200 import Solver, problems
A = orc.stencil_csr(2, 100, 100, 1, problems.poisson2d_coef())
xs = problems.x_star(A.n, 0); b = orc.spmv(A, xs)
S = Solver.stencil(2, 100, 100, 1, problems.poisson2d_coef())
bd = S.apply(torch.from_numpy(xs).cuda())
S.set_option("bench", 1)
r0 = S.solve(bd, tol=0.0, maxit=60, gap=True)
print("plain", r0.rnorm[:4], r0.gap[:4])
S.set_option("rr_auto", 1)
r = S.solve(bd, tol=0.0, maxit=60, gap=True)
fr, rrl = S.rr_info(r.iters)
ref = orc.pbicgstab(A, b, tol=0.0, maxit=60, bench=True, auto_rr=True)
print("auto", r.rnorm[:4], r.gap[:4])
print("ref ", ref.rnorm[:4], ref.gap[:4])
print("fr", fr[:6]); print("rf", ref.bounds[:6, 0]); print(rrl, ref.rr_iters)
