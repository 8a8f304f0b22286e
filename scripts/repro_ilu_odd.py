#!/usr/bin/env python
"""Loopback ILU(0) on one-plane slabs with an odd plane size (35 x 47 x 3, P = 3): run with a
library path (default: the product build).  usage: python scripts/repro_ilu_odd.py [LIB] [block]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
from paper_1809_01948_b200 import problems  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1] != "-":
    from ab_libs import load
    load(sys.argv[1])
block = sys.argv[2] if len(sys.argv) > 2 else "ilu0"
from paper_1809_01948_b200.binding import LoopbackGroup  # noqa: E402

for shape, P in (((35, 47, 3), 3), ((35, 47, 6), 3), ((35, 47, 3), 1)):
    nx, ny, nz = shape
    try:
        kw = {} if block == "jacobi" else {"block": block}
        G = LoopbackGroup.stencil(P, 3, nx, ny, nz, problems.cfg34_coef(), **kw)
        xs = problems.x_star(nx * ny * nz, 7)
        bs = G.apply(G.split(torch.from_numpy(xs).cuda()))
        res = G.solve(bs, tol=1e-13, maxit=12, rr_period=5, gap=False)
        print(shape, P, block, "ok", res.iters, res.rnorm[-1], flush=True)
        G.close()
    except Exception as e:
        print(shape, P, block, "FAILED", str(e)[:150], flush=True)
        break
