import sys, numpy as np, torch
sys.path.insert(0, '.')
from oracle import oracle as orc
from paper_1809_01948_b200 import Solver, problems
for nx, ny in ((2050, 9),):
    coef = problems.cfg2_coef()
    A = orc.stencil_csr(2, nx, ny, 1, coef)
    xs = problems.x_star(A.n, 0); b = orc.spmv(A, xs)
    S = Solver.stencil(2, nx, ny, 1, coef)
    bd = S.apply(torch.from_numpy(xs).cuda())
    for graphs in (1, 0):
        S.set_option("graphs", graphs)
        r = S.solve(bd, tol=1e-11, maxit=120, rr_period=7, gap=True)
        ref = orc.pbicgstab(A, b, tol=1e-11, maxit=120, rr_period=7, gap=True)
        k = min(r.iters, ref.iters) + 1
        dr = np.nonzero(r.rnorm[:k] != ref.rnorm[:k])[0]
        print("graphs", graphs, r.iters, ref.iters, r.outcome, ref.outcome, "first rnorm diff", dr[:5])
        if dr.size:
            i = dr[0]
            print(r.rnorm[i-1:i+3], ref.rnorm[i-1:i+3])
            print("gap", r.gap[i-1:i+3], ref.gap[i-1:i+3])
    S.close()
