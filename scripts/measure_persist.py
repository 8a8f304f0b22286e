#!/usr/bin/env python
"""it/s of the fused stencil schedule with and without the persistent iteration
kernel (option persist), CUDA graphs on, bench mode, CUDA events around whole
solves on the solver stream; shapes: cfg2, cfg3, the cfg3 / cfg4 per-rank slabs
of 2/4/8 GPUs as stand-alone grids, cfg4.  Prints one JSON line per case."""
import json
import sys
import os

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_01948_b200 import Solver, problems  # noqa: E402

PEAK = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]
CASES = [("cfg2", 2, 1024, 1024, 1, problems.cfg2_coef(), 0),
         ("cfg3", 3, 256, 256, 256, problems.cfg34_coef(), 50),
         ("cfg3/2", 3, 256, 256, 128, problems.cfg34_coef(), 50),
         ("cfg3/4", 3, 256, 256, 64, problems.cfg34_coef(), 50),
         ("cfg3/8", 3, 256, 256, 32, problems.cfg34_coef(), 50),
         ("cfg4/8", 3, 512, 512, 64, problems.cfg34_coef(), 50),
         ("cfg4", 3, 512, 512, 512, problems.cfg34_coef(), 50)]
only = set(sys.argv[1:])
for name, dim, nx, ny, nz, coef, rr in CASES:
    if only and name not in only:
        continue
    st = torch.cuda.Stream()
    S = Solver.stencil(dim, nx, ny, nz, coef, stream=st)
    n = S.n_local
    xs = torch.from_numpy(problems.x_star(n, 0)).cuda()
    b = S.apply(xs)
    x0 = torch.zeros_like(b)
    x = torch.empty_like(b)
    S.set_option("bench", 1)
    maxit = 200
    out = {"case": name, "n": n}
    for p in (0, 1):
        S.set_option("persist", p)
        for _ in range(3):
            S.solve(b, x0, tol=0.0, maxit=maxit, rr_period=rr, gap=False, x_out=x)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        e0.record(st)
        for _ in range(reps):
            S.solve(b, x0, tol=0.0, maxit=maxit, rr_period=rr, gap=False, x_out=x)
        e1.record(st)
        torch.cuda.synchronize()
        its = reps * maxit / (e0.elapsed_time(e1) / 1e3)
        out[f"persist{p}_its"] = its
        out[f"persist{p}_frac192"] = 192 * n * its / 1e9 / PEAK
    print(json.dumps(out), flush=True)
    S.close()
