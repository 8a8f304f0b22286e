#!/usr/bin/env python
"""ILU(0) stencil sweep tuning (experiments only): the M^-1 application time of one
config for several library builds x tile-width overrides (PBICG_ILU_TA), in the bench's
kernel-timed mode.  usage: python scripts/ilu_exp.py CONFIG LIB[,LIB...] TA[,TA...]"""
import json
import os
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))
from ab_libs import load  # noqa: E402
from paper_1809_01948_b200 import binding, problems, Solver  # noqa: E402


def run(handle, cfg, its=10, reps=3):
    binding._lib = handle
    st = problems.configs()[cfg].stencil
    S = Solver.stencil(st.dim, st.nx, st.ny, st.nz, st.coef, block="ilu0")
    b = S.apply(torch.from_numpy(problems.x_star(st.n, 0)).cuda())
    S.set_option("bench", 1)
    S.solve(b, tol=0.0, maxit=3, gap=False)
    S.set_option("timing", 1)
    out = []
    for _ in range(reps):
        S.kernel_time("all", reset=True)
        S.solve(b, tol=0.0, maxit=its, gap=False)
        torch.cuda.synchronize()
        n, ms = S.kernel_time("prec")
        out.append(ms / n)
    S.close()
    return sorted(out)[len(out) // 2]


cfg, libs, tas = sys.argv[1], sys.argv[2].split(","), sys.argv[3].split(",")
handles = {l: load(l) for l in libs}
for ta in tas:
    os.environ["PBICG_ILU_TA"] = ta
    for l in libs:
        try:
            v = run(handles[l], cfg)
        except Exception as e:  # e.g. a build whose shared memory does not fit
            print(json.dumps({"cfg": cfg, "lib": os.path.basename(l), "TA": int(ta),
                              "error": str(e)[:120]}), flush=True)
            continue
        print(json.dumps({"cfg": cfg, "lib": os.path.basename(l), "TA": int(ta), "prec_ms": round(v, 4)}), flush=True)
