"""it/s and iteration roofline of p-BiCGStab for an arbitrary stencil grid
(quick measurement helper): python scripts/measure_shape.py dim nx ny nz [tile [pdl [graphs]]]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_01948_b200 import Solver, problems  # noqa: E402

dim, nx, ny, nz = (int(a) for a in sys.argv[1:5])
tile = int(sys.argv[5]) if len(sys.argv) > 5 else 1
pdl = int(sys.argv[6]) if len(sys.argv) > 6 else -1
graphs = int(sys.argv[7]) if len(sys.argv) > 7 else -1
coef = problems.cfg34_coef() if dim == 3 else problems.cfg2_coef()
S = Solver.stencil(dim, nx, ny, nz, coef)
S.set_option("tile", tile)
if pdl >= 0:
    S.set_option("pdl", pdl)
if graphs >= 0:
    S.set_option("graphs", graphs)
b = S.apply(torch.from_numpy(problems.x_star(S.n_local, 0)).cuda())
S.set_option("bench", 1)
for _ in range(2):
    S.solve(b, tol=0.0, maxit=100, gap=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
its = 0
for _ in range(3):
    its += S.solve(b, tol=0.0, maxit=100, gap=False).iters
e1.record()
torch.cuda.synchronize()
ips = its / (e0.elapsed_time(e1) / 1e3)
frac = S.kernel_bytes("iteration") * ips / 1e9 / 6550.4
print(f"dim={dim} {nx}x{ny}x{nz} tile={tile} pdl={pdl} graphs={graphs}: {ips:.1f} it/s, "
      f"iteration roofline {frac:.3f}")
