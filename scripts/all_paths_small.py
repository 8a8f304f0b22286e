"""Small end-to-end run of every kernel family (a quick all-paths check):
stencil (tile + line kernels, 2D/3D, odd nx), all three methods, periodic and
automated replacement, gap tracking, CSR (window + gather SpMV) with Jacobi and
block Jacobi, loopback ranks, at tiny sizes."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_01948_b200 import Solver, problems  # noqa: E402
from paper_1809_01948_b200.binding import LoopbackGroup  # noqa: E402


def run(S, n, **kw):
    xs = torch.from_numpy(problems.x_star(n, 0)).cuda()
    b = S.apply(xs)
    return S.solve(b, **kw)


for dim, nx, ny, nz in ((3, 13, 7, 9), (2, 37, 21, 1), (3, 16, 8, 6)):
    coef = problems.cfg34_coef() if dim == 3 else problems.cfg2_coef()
    S = Solver.stencil(dim, nx, ny, nz, coef)
    n = S.n_local
    for tile in (1, 0):
        S.set_option("tile", tile)
        run(S, n, tol=1e-10, maxit=12, rr_period=3, gap=True)
    S.set_option("tile", 1)
    S.set_option("rr_auto", 1)
    run(S, n, tol=0.0, maxit=12, gap=True)
    S.set_option("rr_auto", 0)
    for m in (1, 2):
        S.set_option("method", m)
        run(S, n, tol=1e-10, maxit=12, gap=True)
    S.set_option("method", 0)
    S.close()
for bw, blk in ((200, 1), (200, 4), (6000, 8)):
    P = problems.csr_band(8192, nnz_row=27, band=bw, seed=1)
    S = Solver.csr(P.n, P.row_ptr, P.col, P.val, block=blk)
    run(S, P.n, tol=1e-12, maxit=10, rr_period=3, gap=True)
    for m in (1, 2):
        S.set_option("method", m)
        run(S, P.n, tol=1e-12, maxit=8, gap=True)
    S.set_option("method", 0)
    S.set_option("rr_auto", 1)
    run(S, P.n, tol=0.0, maxit=8, gap=True)
    S.close()
G = LoopbackGroup.stencil(3, 3, 12, 10, 9, problems.cfg34_coef())
xs = torch.from_numpy(problems.x_star(12 * 10 * 9, 0)).cuda()
bs = G.apply(G.split(xs))
G.solve(bs, tol=1e-10, maxit=10, rr_period=3, gap=True)
G.close()
torch.cuda.synchronize()
print("all_paths_small done")
