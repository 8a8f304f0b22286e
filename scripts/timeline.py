#!/usr/bin/env python
"""Per-CTA timeline of the stencil sweeps (experiments only).

Builds a variant of libpbicgstab.so with -DPBICG_TIMELINE (tile_sweeps.cuh: thread 0
of every CTA records %globaltimer at entry, after the PDL wait, when its first plane
has landed, after its unit loop and at exit), runs a short bench-mode solve per case
with CUDA graphs on, and prints, per sweep kind, where the time of one launch goes:
launch-to-launch period, the gap between the previous grid's last exit and this
grid's first wait return, first-plane latency, the spread of the unit loops, and the
grid-reduction tail.  The product library is untouched.

usage: python scripts/timeline.py [--build-only] [case ...]   (cases as ab_libs.py)
       env TL_OPTS="opt=value,...": solver options (e.g. defer=0)
"""
import ctypes
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1809_01948_b200 import _build  # noqa: E402

VAR = os.path.join(ROOT, "paper_1809_01948_b200", "build_tl")
LIB = os.path.join(VAR, "libpbicgstab_tl.so")


def build_variant():
    os.makedirs(VAR, exist_ok=True)
    if os.path.exists(LIB) and all(os.path.getmtime(s) < os.path.getmtime(LIB)
                                   for s in _build.sources()):
        return
    procs, objs = [], []
    for i, (src, defs) in enumerate(_build.UNITS):
        obj = os.path.join(VAR, f"unit{i}.o")
        cmd = [_build.nvcc(), *_build.NVCC_FLAGS, *defs, "-DPBICG_TIMELINE", "-c", "-o", obj,
               os.path.join(_build.CSRC, src)]
        procs.append(subprocess.Popen(cmd))
        objs.append(obj)
    if any(p.wait() != 0 for p in procs):
        raise SystemExit("variant build failed")
    subprocess.check_call([_build.nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                           "-o", LIB, *objs])


MODES = {0: "A", 1: "C", 2: "rr1", 3: "rr2", 5: "init1", 6: "init2", 18: "spB", 19: "spD"}


def analyse(rec, peak, n, bytes_per_row):
    import numpy as np
    rec = rec[np.argsort(rec[:, 1])]
    grid = (rec[:, 8] >> 16) & 0xFFFF
    launches, i = [], 0
    while i < len(rec):
        g = int(grid[i])
        launches.append(rec[i:i + g])
        i += g
    rows = {}
    prev_end = None
    prev_wait = None
    for L in launches:
        mc = int((L[0, 8] >> 32) & 0xFFFF)
        m = MODES.get(mc, str(mc))
        t0, t1, t2, t3, t4, t5, t6, t7 = (L[:, k].astype(np.int64) for k in range(8))
        last = np.nonzero(t5)[0]
        d = {"period": (t1.min() - prev_wait) if prev_wait is not None else None,
             "gap": (t1.min() - prev_end) if prev_end is not None else None,
             "wait_spread": t1.max() - t1.min(),
             "first": float(np.median(t2 - t1)), "first_max": (t2 - t1).max(),
             "loop_med": float(np.median(t3 - t2)), "loop_min": (t3 - t2).min(),
             "loop_max": (t3 - t2).max(),
             "loop_end_spread": t3.max() - t3.min(),
             "tail": t4.max() - t3.max(),
             "cta_exit": float(np.median(t4 - t3)),
             "last_reduce": (t5[last[0]] - t3[last[0]]) if len(last) else None,
             "last_publish": (t6[last[0]] - t5[last[0]]) if len(last) else None,
             "last_after": (t4[last[0]] - t6[last[0]]) if len(last) else None,
             "last_is_latest": bool(len(last) and t3[last[0]] == t3.max()),
             "busy": t4.max() - t1.min(),
             # deferred finalize: the redundant reduction + step after the prologue issue
             "df_fin": float(np.median(t7 - t1)) if t7.min() > 0 else None,
             "df_cnt": float(np.median(t5 - t1)) if t7.min() > 0 else None,
             "df_pre": float(np.median(t6 - t1)) if t7.min() > 0 else None}
        prev_end = t4.max()
        prev_wait = t1.min()
        rows.setdefault(m, []).append(d)
    out = {}
    for m, ds in rows.items():
        agg = {}
        for k in ds[0]:
            v = [float(x[k]) for x in ds[2:] if x[k] is not None]  # skip the first two launches
            if v:
                agg[k] = round(float(np.median(v)) / 1e3, 2)  # microseconds
        agg["launches"] = len(ds)
        if m in bytes_per_row:
            agg["ideal_us"] = round(bytes_per_row[m] * n / peak / 1e3, 2)
        out[m] = agg
    return out


def main():
    args = [a for a in sys.argv[1:]]
    build_variant()
    if "--build-only" in args:
        return
    import numpy as np  # noqa: F401
    import torch
    _build.LIB = LIB
    from paper_1809_01948_b200 import Solver, binding, problems
    L = binding.lib(build=False)
    L.pbicg_timeline_set.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint]
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    cases = [("cfg2", 2, 1024, 1024, 1, problems.cfg2_coef()),
             ("cfg3", 3, 256, 256, 256, problems.cfg34_coef()),
             ("cfg3/4", 3, 256, 256, 64, problems.cfg34_coef()),
             ("cfg3/8", 3, 256, 256, 32, problems.cfg34_coef()),
             ("cfg4/8", 3, 512, 512, 64, problems.cfg34_coef())]
    only = {a for a in args if not a.startswith("--")}
    cap = 148 * 400
    buf = torch.zeros(cap, 10, dtype=torch.int64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    for name, dim, nx, ny, nz, coef in cases:
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
        for kv in filter(None, os.environ.get("TL_OPTS", "").split(",")):  # e.g. defer=0
            k, v = kv.split("=")
            S.set_option(k, int(v))
        for _ in range(3):
            S.solve(b, x0, tol=0.0, maxit=100, rr_period=0, gap=False, x_out=x)
        torch.cuda.synchronize()
        cnt.zero_()
        assert L.pbicg_timeline_set(buf.data_ptr(), cnt.data_ptr(), cap) == 0
        S.solve(b, x0, tol=0.0, maxit=100, rr_period=0, gap=False, x_out=x)
        torch.cuda.synchronize()
        L.pbicg_timeline_set(None, None, 0)
        k = min(int(cnt.item()), cap)
        rec = buf[:k].cpu().numpy().view("uint64")
        res = analyse(rec, peak, n, {"A": 88, "C": 104})
        print(json.dumps({"case": name, "n": n, "records": k, **res}), flush=True)
        S.close()


if __name__ == "__main__":
    main()
