import sys, numpy as np, torch
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
from oracle import oracle as orc
from paper_1809_01948_b200 import Solver, problems
from test_gpu_parity import stencil_case, coef_of
for (dim, nx, ny, nz, kind) in ((2, 2050, 9, 1, "cd2"), (3, 1100, 5, 6, "cd3")):
    solver, A, xs, b, b_d = stencil_case(Solver, orc, dim, nx, ny, nz, coef_of(kind))
    ref = orc.pbicgstab(A, b, tol=1e-11, maxit=120, rr_period=7)
    for rep in range(3):
        res = solver.solve(b_d, tol=1e-11, maxit=120, rr_period=7, gap=True)
        k = min(res.iters, ref.iters) + 1
        dr = np.nonzero(res.rnorm[:k] != ref.rnorm[:k])[0]
        dg = np.nonzero(res.gap[:k] != ref.gap[:k])[0]
        print(dim, nx, rep, res.iters, ref.iters, "rnorm diff@", dr[:3], "gap diff@", dg[:3],
              res.gap[:4], ref.gap[:4])
