import sys, numpy as np, torch
sys.path.insert(0, '.')
from oracle import oracle as orc
from paper_1809_01948_b200 import Solver, problems
A = orc.stencil_csr(2, 64, 64, 1, problems.cfg2_coef())
xs = problems.x_star(A.n, 0); b = orc.spmv(A, xs)
S = Solver.stencil(2, 64, 64, 1, problems.cfg2_coef())
bd = S.apply(torch.from_numpy(xs).cuda())
S.set_option("bench", 1)
S.set_option("rr_auto", 1)
r = S.solve(bd, tol=0.0, maxit=300, gap=True)
fr, rrl = S.rr_info(r.iters)
ref = orc.pbicgstab(A, b, tol=0.0, maxit=300, bench=True, auto_rr=True)
print(rrl); print(ref.rr_iters)
d = np.nonzero(r.rnorm != ref.rnorm)[0]
print("first rnorm diff", d[:5])
rel = np.abs(fr - ref.bounds[:, 0]) / ref.bounds[:, 0]
print("fr rel max", rel.max(), np.argmax(rel))
tau = 2 ** -26.5
m = fr / (tau * r.rnorm); mo = ref.bounds[:, 0] / (tau * ref.rnorm)
for j in sorted(set(rrl) ^ set(ref.rr_iters)):
    print(j, m[j-2:j+2], mo[j-2:j+2])
