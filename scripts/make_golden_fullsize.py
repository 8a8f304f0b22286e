#!/usr/bin/env python
"""Write tests/golden/fullsize_<cfg>.json: the ORACLE's converged solve of BASELINE
cfg2 (2D upwind conv-diff 1024^2, Jacobi, tol 1e-10) and cfg3 (3D 256^3, Jacobi,
tol 1e-10, replacement every 50) at full size, so the GPU test
(tests/test_gpu_fullsize.py) can compare bitwise without re-running a minutes-long
single-core oracle on the GPU box.  Calls only oracle/ (and problems.py for the
seeded inputs); nothing here comes from the CUDA path.

Stored: iterations, outcome, the whole ||r_i|| and gap histories (hex-exact), the
replacement iterations, ||x - x*|| / ||x*||, and sha256 of x's bytes (bitwise x).

    python scripts/make_golden_fullsize.py cfg2 cfg3        # ~17 min on one core
    python scripts/make_golden_fullsize.py cfg5_classic_bench   # cfg5 classic BiCGStab, bench mode
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as orc  # noqa: E402
from paper_1809_01948_b200 import problems  # noqa: E402


def cfg5_classic_bench():
    """cfg5 (CSR band 2^23 x 27) classic BiCGStab (Alg. 1) in bench mode (tol 0): the
    noise-regime exact breakdown bench.py's comparison line relies on."""
    M = problems.csr_band(1 << 23, nnz_row=27, band=4096, seed=1)
    A = orc.csr(M.row_ptr, M.col, M.val)
    xs = problems.x_star(A.n, 0)
    b = orc.spmv(A, xs)
    t0 = time.time()
    r = orc.bicgstab(A, b, tol=0.0, maxit=300, bench=True, gap=False)
    dt = time.time() - t0
    out = {"config": "cfg5_classic_bench", "desc": "cfg5, classic BiCGStab, bench mode, tol 0",
           "n": int(A.n), "maxit": 300, "x_star_seed": 0,
           "generator": "scripts/make_golden_fullsize.py (oracle/oracle.c orc_bicgstab)",
           "iters": int(r.iters), "outcome": r.outcome,
           "rnorm_hex": [float(v).hex() for v in r.rnorm],
           "x_sha256": hashlib.sha256(np.ascontiguousarray(r.x).tobytes()).hexdigest(),
           "oracle_seconds": dt}
    with open(os.path.join(ROOT, "tests", "golden", "fullsize_cfg5_classic_bench.json"), "w") as f:
        json.dump(out, f, indent=0)
    print("cfg5_classic_bench", r.iters, r.outcome, f"{dt:.0f}s", flush=True)


def main(names):
    for name in names:
        if name == "cfg5_classic_bench":
            cfg5_classic_bench()
            continue
        cfg = problems.configs()[name]
        st = cfg.stencil
        A = orc.stencil_csr(st.dim, st.nx, st.ny, st.nz, st.coef)
        xs = problems.x_star(A.n, 0)
        b = orc.spmv(A, xs)
        t0 = time.time()
        r = orc.pbicgstab(A, b, tol=cfg.tol, maxit=cfg.maxit, rr_period=cfg.rr_period)
        dt = time.time() - t0
        out = {
            "config": name, "desc": cfg.desc, "n": int(A.n), "tol": cfg.tol,
            "maxit": cfg.maxit, "rr_period": cfg.rr_period, "x_star_seed": 0,
            "generator": "scripts/make_golden_fullsize.py (oracle/oracle.c orc_pbicgstab)",
            "iters": int(r.iters), "outcome": r.outcome,
            "rnorm_hex": [float(v).hex() for v in r.rnorm],
            "gap_hex": [float(v).hex() for v in r.gap],
            "err": float(np.linalg.norm(r.x - xs) / np.linalg.norm(xs)),
            "x_sha256": hashlib.sha256(np.ascontiguousarray(r.x).tobytes()).hexdigest(),
            "oracle_seconds": dt,
        }
        p = os.path.join(ROOT, "tests", "golden", f"fullsize_{name}.json")
        with open(p, "w") as f:
            json.dump(out, f, indent=0)
        print(name, r.iters, r.outcome, f"{dt:.0f}s", out["err"], flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["cfg2", "cfg3"])
