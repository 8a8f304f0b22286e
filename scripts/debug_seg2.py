import subprocess, sys
code = r'''
import sys, torch
sys.path.insert(0, ".")
from paper_1809_01948_b200 import Solver, problems
dim, nx, ny, nz, maxit = (int(a) for a in sys.argv[1:6])
coef = problems.cfg34_coef() if dim == 3 else problems.cfg2_coef()
S = Solver.stencil(dim, nx, ny, nz, coef)
b = S.apply(torch.from_numpy(problems.x_star(S.n_local, 0)).cuda())
S.set_option("bench", 1)
r = S.solve(b, tol=0.0, maxit=maxit, gap=False)
print("ok", r.iters)
'''
for args in (("2", "4096", "4096", "1", "100"), ("2", "2048", "4096", "1", "100"),
             ("3", "2048", "64", "64", "40"), ("3", "2048", "256", "256", "40"), ("3", "1100", "5", "6", "40")):
    p = subprocess.run([sys.executable, "-c", code, *args], capture_output=True, text=True,
                       env={"CUDA_LAUNCH_BLOCKING": "1", **__import__("os").environ})
    print(args, p.stdout.strip()[-60:], p.stderr.strip().splitlines()[-1][-160:] if p.returncode else "")
