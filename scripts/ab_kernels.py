#!/usr/bin/env python
"""A/B per-kernel timing of two builds of libpbicgstab.so in one process (experiments
only): the bench's kernel-timed mode (graphs off, CUDA events around every kernel on
the solver stream), cases interleaved A, B, A, B, ... so clock / power drift hits both
alike; prints the median per-kernel average duration and its fraction of the measured
HBM peak (the library's algorithmic bytes per launch).

usage: python scripts/ab_kernels.py LIB_A LIB_B [case ...]   (cases of ab_libs.py)
       env AB_PREC=bj2|bj4|bj8|ilu0 (instead of Jacobi), AB_AUTO=1 (automated replacement)
       AB_SCHED=2 (the split schedule)
"""
import json
import os
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))
from ab_libs import CASES, PEAK, load  # noqa: E402
from paper_1809_01948_b200 import binding, problems, Solver  # noqa: E402

KERNELS = ("sweepA", "sweepC", "spmvB", "spmvD", "rr1", "rr2", "gap", "init")


def run(handle, case, maxit=200, reps=2):
    binding._lib = handle
    dim, nx, ny, nz, coef, rr = CASES[case]
    st = torch.cuda.Stream()
    kw = {}
    prec = os.environ.get("AB_PREC", "")
    if prec.startswith("bj"):
        kw["block"] = int(prec[2:])
    elif prec in ("ilu0", "icc0"):
        kw["block"] = prec
    S = Solver.stencil(dim, nx, ny, nz, coef, stream=st, **kw)
    n = S.n_local
    xs = torch.from_numpy(problems.x_star(n, 0)).cuda()
    b = S.apply(xs)
    x0 = torch.zeros_like(b)
    x = torch.empty_like(b)
    S.set_option("bench", 1)
    if os.environ.get("AB_SCHED"):
        S.set_option("schedule", int(os.environ["AB_SCHED"]))
    if os.environ.get("AB_AUTO") == "1":
        S.set_option("rr_auto", 1)
        rr = 0
    for _ in range(2):
        S.solve(b, x0, tol=0.0, maxit=maxit, rr_period=rr, gap=True, x_out=x)
    torch.cuda.synchronize()
    S.set_option("timing", 1)
    S.kernel_time("all", reset=True)
    for _ in range(reps):
        S.solve(b, x0, tol=0.0, maxit=maxit, rr_period=rr, gap=True, x_out=x)
    torch.cuda.synchronize()
    out = {}
    for k in KERNELS:
        nk, tk = S.kernel_time(k)
        if nk:
            out[k] = (tk / nk, S.kernel_bytes(k))
    S.set_option("timing", 0)
    S.close()
    return out


def main():
    la, lb = sys.argv[1], sys.argv[2]
    cases = sys.argv[3:] or ["cfg4"]
    ha, hb = load(la), load(lb)
    for case in cases:
        res = {"A": [], "B": []}
        for _ in range(3):
            for tag, h in (("A", ha), ("B", hb)):
                res[tag].append(run(h, case))
        for k in KERNELS:
            if k not in res["A"][0]:
                continue
            row = {"case": case, "kernel": k}
            for tag in ("A", "B"):
                ms = sorted(r[k][0] for r in res[tag])[1]
                byt = res[tag][0][k][1]
                row[tag + "_ms"] = round(ms, 4)
                row[tag + "_frac"] = round(byt / (ms * 1e-3) / 1e9 / PEAK, 4) if byt else None
            row["B/A"] = round(row["B_ms"] / row["A_ms"], 4)
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
