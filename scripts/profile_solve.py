"""Small driver for ncu captures: one solve of a config through the public API."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1809_01948_b200 import Solver, problems  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--maxit", type=int, default=4)
ap.add_argument("--rr", type=int, default=2)
ap.add_argument("--gap", type=int, default=0)
ap.add_argument("--method", type=int, default=0)
ap.add_argument("--rr-auto", type=int, default=0)
ap.add_argument("--block", type=int, default=1)
ap.add_argument("--schedule", type=int, default=0)
a = ap.parse_args()
cfg = problems.configs()[a.config]
if cfg.kind == "csr":
    M = problems.csr_band(cfg.csr_n, nnz_row=27, band=4096, seed=1)
    S = Solver.csr(M.n, M.row_ptr, M.col, M.val, block=a.block)
    n = M.n
else:
    st = cfg.stencil
    coef = [2.0 * st.dim] + [-1.0] * 6 if a.method == 2 else st.coef  # p-CG needs SPD
    S = Solver.stencil(st.dim, st.nx, st.ny, st.nz, coef, block=a.block)
    n = st.n
xs = torch.from_numpy(problems.x_star(n, 0)).cuda()
b = S.apply(xs)
S.set_option("bench", 1)
S.set_option("graphs", 0)
S.set_option("method", a.method)
if a.schedule:
    S.set_option("schedule", a.schedule)
S.set_option("rr_auto", a.rr_auto)
rr = a.rr if (a.method == 0 and not a.rr_auto) else 0
r = S.solve(b, tol=0.0, maxit=a.maxit, rr_period=rr, gap=bool(a.gap))
print("iters", r.iters, r.outcome, r.rnorm[-1])
