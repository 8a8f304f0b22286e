#!/usr/bin/env python
"""One short ILU(0)/ICC(0) solve for profiling the wavefront kernels under ncu:
    python scripts/profile_ilu.py cfg1|cfg3 [iterations]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_01948_b200 import Solver, problems  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
its = int(sys.argv[2]) if len(sys.argv) > 2 else 3
st = problems.configs()[name].stencil
prec = "icc0" if name == "cfg1" else "ilu0"
S = Solver.stencil(st.dim, st.nx, st.ny, st.nz, st.coef, block=prec)
b = S.apply(torch.from_numpy(problems.x_star(st.n, 0)).cuda())
S.set_option("bench", 1)
S.set_option("graphs", 0)
r = S.solve(b, tol=0.0, maxit=its, gap=False)
torch.cuda.synchronize()
print(name, prec, r.iters, r.rnorm[-1])
