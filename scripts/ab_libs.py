#!/usr/bin/env python
"""A/B timing of two builds of libpbicgstab.so in one process (experiments only):
interleaves the two libraries case by case, several rounds, so clock / power drift
hits both alike.  CUDA graphs, bench mode, 200 iterations per solve, CUDA events
around 5 solves on the solver stream (the iteration rates of DESIGN.md section 8).

usage: python scripts/ab_libs.py LIB_A LIB_B [case ...]
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1809_01948_b200 import _build, binding, problems, Solver  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
CASES = {"cfg2": (2, 1024, 1024, 1, problems.cfg2_coef(), 0),
         "cfg3": (3, 256, 256, 256, problems.cfg34_coef(), 50),
         "cfg3/4": (3, 256, 256, 64, problems.cfg34_coef(), 50),
         "cfg3/8": (3, 256, 256, 32, problems.cfg34_coef(), 50),
         "cfg4/8": (3, 512, 512, 64, problems.cfg34_coef(), 50),
         "cfg4": (3, 512, 512, 512, problems.cfg34_coef(), 50)}


def load(path):
    binding._lib = None
    _build.LIB = path
    _build.build = lambda *a, **k: path
    return binding.lib(build=False)


def run(handle, case, reps=5, maxit=200):
    binding._lib = handle
    dim, nx, ny, nz, coef, rr = CASES[case]
    st = torch.cuda.Stream()
    S = Solver.stencil(dim, nx, ny, nz, coef, stream=st)
    n = S.n_local
    xs = torch.from_numpy(problems.x_star(n, 0)).cuda()
    b = S.apply(xs)
    x0 = torch.zeros_like(b)
    x = torch.empty_like(b)
    S.set_option("bench", 1)
    for _ in range(2):
        S.solve(b, x0, tol=0.0, maxit=maxit, rr_period=rr, gap=False, x_out=x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        S.solve(b, x0, tol=0.0, maxit=maxit, rr_period=rr, gap=False, x_out=x)
    e1.record(st)
    torch.cuda.synchronize()
    its = reps * maxit / (e0.elapsed_time(e1) / 1e3)
    S.close()
    return its, 192 * n * its / 1e9 / PEAK


def main():
    la, lb = sys.argv[1], sys.argv[2]
    cases = sys.argv[3:] or list(CASES)
    ha, hb = load(la), load(lb)
    for case in cases:
        res = {"A": [], "B": []}
        for _ in range(3):
            for tag, h in (("A", ha), ("B", hb)):
                res[tag].append(run(h, case))
        out = {"case": case}
        for tag in ("A", "B"):
            its = sorted(r[0] for r in res[tag])
            out[tag + "_its"] = round(its[len(its) // 2], 1)
            out[tag + "_frac192"] = round(sorted(r[1] for r in res[tag])[len(its) // 2], 4)
        out["B/A"] = round(out["B_its"] / out["A_its"], 4)
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
