#!/usr/bin/env python
"""bench.py -- p-BiCGStab fp64 iterations/s and % of HBM roofline on B200.

Contract:
  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--config cfg4]

A step = one full solve of the configured workload through the public API
(init + `maxit` p-BiCGStab iterations in bench mode, replacement every
`rr_period`), inputs resident in HBM.  value = iterations/s of the whole job.
Rank 0 prints one JSON line.  `--impl reference` times the CPU oracle (the
reference arm of this tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1809_01948_b200 import problems  # noqa: E402

METRIC = "p-BiCGStab fp64 iterations/s and % of HBM roofline at 1/2/4/8 B200"
SCHEDULES = {
    "pbicgstab": "fused 2-sweep (stencil), TMA 2.5D sweeps",
    "bicgstab": "classic Alg. 1: 3 TMA sweeps (p,s | q,y dots | x,r), 3 reductions",
    "pipecg": "p-CG: 1 TMA sweep, 1 reduction (Laplacian coefficients: CG needs SPD)",
}
UNIT = "iterations/s"
L2_BYTES = 126 * 2 ** 20


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(config: str, kernel: str):
    """dram bytes per launch of `kernel` on `config` from the committed ncu --set full
    summaries (profiles/ncu_traffic.json; captured with the Jacobi preconditioner,
    the default schedule and periodic replacement)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        d = json.load(open(p))
        return d[config][kernel]["dram_bytes_per_launch"]
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, index: int = 0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


class CsrShape:
    """Stand-in for StencilProblem when the workload is the CSR band matrix (cfg5)."""

    def __init__(self, n):
        self.n = n
        self.dim = 0
        self.nx = n
        self.ny = self.nz = 1


def workload(cfg_name: str):
    cfg = problems.configs()[cfg_name]
    if cfg.kind == "csr":
        # cfg5: 200 fixed iterations (A23: converges in ~8), replacement every 100
        return cfg, CsrShape(cfg.csr_n), 200, cfg.rr_period
    st = cfg.stencil
    maxit = cfg.maxit if cfg.bench else 200
    rr = 50  # replacement every 50 iterations (cfg3's period) so every 8(a) row runs
    return cfg, st, maxit, rr


_CSR_CACHE = {}


def csr_matrix(cfg):
    if cfg.name not in _CSR_CACHE:
        _CSR_CACHE[cfg.name] = problems.csr_band(cfg.csr_n, nnz_row=27, band=4096, seed=1)
    return _CSR_CACHE[cfg.name]


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


class PinnedCore:
    """Pin the calling thread to one core (the oracle is single-threaded) for the
    duration of the sample, like `taskset -c <core>`; restores the old mask."""

    def __enter__(self):
        self.old = None
        self.core = None
        try:
            self.old = os.sched_getaffinity(0)
            self.core = max(self.old)  # the highest core: away from the driver threads
            os.sched_setaffinity(0, {self.core})
        except (AttributeError, OSError):
            self.old = None
        return self

    def __exit__(self, *a):
        if self.old is not None:
            os.sched_setaffinity(0, self.old)


def oracle_sample(st, maxit_sample: int, nz_sample: int, cfg=None, method="pbicgstab", block=1):
    """Time the oracle (1 core, pinned) on an nx*ny*nz_sample slab of the workload
    (CSR: the full matrix for maxit_sample iterations)."""
    with PinnedCore():
        return _oracle_sample(st, maxit_sample, nz_sample, cfg, method, block)


def _oracle_sample(st, maxit_sample, nz_sample, cfg, method, block):
    from oracle import oracle as orc
    solve = {"pbicgstab": orc.pbicgstab, "bicgstab": orc.bicgstab, "pipecg": orc.pipecg}[method]
    if isinstance(st, CsrShape):
        M = csr_matrix(cfg)
        A = orc.csr(M.row_ptr, M.col, M.val)
        xs = problems.x_star(A.n, 0)
        b = orc.spmv(A, xs)
        t0 = time.perf_counter()
        solve(A, b, tol=0.0, maxit=0, bench=True, gap=False, block=block)
        t_init = time.perf_counter() - t0
        t0 = time.perf_counter()
        r = solve(A, b, tol=0.0, maxit=maxit_sample, bench=True, gap=False, block=block)
        t = time.perf_counter() - t0 - t_init
        return A.n * r.iters / t, A.n, r.iters, t
    nzs = min(nz_sample, st.nz if st.dim == 3 else st.ny)
    coef = [2.0 * st.dim] + [-1.0] * 6 if method == "pipecg" else st.coef
    if st.dim == 3:
        A = orc.stencil_csr(3, st.nx, st.ny, nzs, coef)
    else:
        A = orc.stencil_csr(2, st.nx, nzs, 1, coef)
    xs = problems.x_star(A.n, 0)
    b = orc.spmv(A, xs)
    t0 = time.perf_counter()
    solve(A, b, tol=0.0, maxit=0, bench=True, gap=False, block=block)
    t_init = time.perf_counter() - t0
    t0 = time.perf_counter()
    r = solve(A, b, tol=0.0, maxit=maxit_sample, bench=True, gap=False, block=block)
    t = time.perf_counter() - t0 - t_init
    rows_per_s = A.n * r.iters / t
    return rows_per_s, A.n, r.iters, t


def sample_desc(st, cfg):
    if isinstance(st, CsrShape):
        return f"the full {cfg.name} CSR matrix"
    return f"a {st.nx}x{st.ny}x64 slab of {cfg.name}"


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    cfg, st, maxit, rr = workload(args.config)
    n_full = st.n
    vals, secs = [], []
    sample = None
    for s in range(args.warmup + args.steps):
        rows_per_s, n_s, its, t = oracle_sample(st, 6 if st.dim else 3, 64, cfg)
        if s >= args.warmup:
            vals.append(rows_per_s / n_full)
            secs.append(t)
            sample = (f"oracle p-BiCGStab (C, 1 core) on {sample_desc(st, cfg)} "
                      f"({n_s} rows), {its} iterations per step, scaled by rows to {n_full} rows")
    v = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            # a step is one bounded sample (wall time as measured); value scales its
            # iterations by rows to the full workload
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * statistics.median(secs),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": bench_config(args, cfg, st, maxit, rr, world),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": sample, "cpu": cpu_model(),
                             "pinning": "sched_setaffinity to one core (taskset -c)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def bench_config(args, cfg, st, maxit, rr, world):
    """The workload description both arms print (identical config => comparable lines)."""
    n = st.n // world  # rows per rank
    return {"workload": f"{cfg.name}: {cfg.desc}", "n": st.n,
            "grid": [st.nx, st.ny, st.nz] if st.dim else "csr 27 nnz/row, band 4096",
            "maxit_per_step": maxit, "rr_period": rr, "gap_tracking": bool(args.gap),
            "rr_auto": bool(args.rr_auto),
            "preconditioner": ("jacobi" if args.block == 1 else args.block.upper()
                               if isinstance(args.block, str) else f"block-jacobi {args.block}"),
            "method": args.method,
            "schedule": (("split 4-phase (stencil), stand-alone TMA SpMVs the reductions "
                          "hide behind" if args.schedule == 2 else SCHEDULES[args.method])
                         if st.dim else "split 4-phase (CSR as ELL), reduction #1 overlapped"),
            "l2": ("inputs larger than L2 (%.1f GB per GPU)" % (14 * 8 * n / 1e9)
                   if 14 * 8 * n > 4 * 126e6 else
                   "working set %.0f MB, about the 126 MB L2: not flushed (this "
                   "config is L2-resident by construction)" % (14 * 8 * n / 1e6)),
            "timed_region": ("CUDA events around every kernel on the solver stream "
                             "(graphs off: per-kernel durations for the roofline); "
                             "e2e runs with CUDA graphs" if args.kernel_timing else
                             "CUDA graphs, no per-kernel events"),
            "parallelism": (f"z-slab x{world}" if st.dim else f"row-block x{world}") +
                           (" (NCCL halo + rank-row all-gather)" if world > 1 else ""),
            "overlap": bool(args.overlap) if world > 1 else None,
            "transport": (["nccl", "peer-memory"][args.transport] if world > 1 else None)}


def method_coef(args, st):
    """p-CG needs an SPD operator: --method pipecg runs the same grid with the
    pure-diffusion (Laplacian) coefficients; the other solvers use the config's."""
    if args.method == "pipecg" and not isinstance(st, CsrShape):
        return [2.0 * st.dim] + [-1.0] * 6
    return st.coef


def setup_solver(args, cfg, st, rank, world, dev, stream):
    """One handle per process; NCCL communicators for world > 1 (ids broadcast
    over the torch process group)."""
    import torch
    from paper_1809_01948_b200 import Solver, binding
    if world == 1:
        if isinstance(st, CsrShape):
            M = csr_matrix(cfg)
            return Solver.csr(st.n, M.row_ptr, M.col, M.val, stream=stream, block=args.block)
        return Solver.stencil(st.dim, st.nx, st.ny, st.nz, method_coef(args, st), stream=stream,
                              block=args.block)
    ids = [binding.nccl_unique_id(), binding.nccl_unique_id()] if rank == 0 else [None, None]
    torch.distributed.broadcast_object_list(ids, src=0)
    dist = binding.make_dist(world, rank, ids[0], ids[1])
    if isinstance(st, CsrShape):
        M = csr_matrix(cfg)
        lo, hi = st.n * rank // world, st.n * (rank + 1) // world
        rp = M.row_ptr[lo:hi + 1] - M.row_ptr[lo]
        sl = slice(int(M.row_ptr[lo]), int(M.row_ptr[hi]))
        return Solver.csr(st.n, rp, M.col[sl], M.val[sl], row_begin=lo, stream=stream, dist=dist,
                          block=args.block)
    return Solver.stencil(st.dim, st.nx, st.ny, st.nz, method_coef(args, st), stream=stream,
                          dist=dist, block=args.block)


def run_ours(args, rank, world):
    import torch

    dev = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(dev)
    cfg, st, maxit, rr = workload(args.config)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{dev}"))
    stream = torch.cuda.Stream()
    S = setup_solver(args, cfg, st, rank, world, dev, stream)
    from paper_1809_01948_b200.binding import METHODS
    S.set_option("method", METHODS[args.method])
    if args.method != "pbicgstab":
        rr = 0  # residual replacement is an Alg. 2 feature
    if args.rr_auto:
        S.set_option("rr_auto", 1)  # automated replacement instead of the period
        rr = 0
    n = S.n_local
    xs_full = problems.x_star(st.n, seed=0)
    xs = torch.from_numpy(xs_full[S.row_begin:S.row_begin + n]).to(f"cuda:{dev}")
    del xs_full
    b = S.apply(xs)
    x0 = torch.zeros_like(b)
    x = torch.empty_like(b)
    S.set_option("bench", 1)
    S.set_option("graphs", 1)
    S.set_option("overlap", args.overlap)
    if args.schedule:
        S.set_option("schedule", args.schedule)
    S.set_option("csr_tma", args.csr_tma)  # CSR sweeps / the stencil split schedule's sweeps
    if world > 1:
        S.set_option("transport", args.transport)  # collective: every rank sets it
    gap = bool(args.gap)

    def step():
        return S.solve(b, x0, tol=0.0, maxit=maxit, rr_period=rr, gap=gap, x_out=x)

    breakdown_at = None
    r = step()
    if r.outcome == "breakdown" and r.iters > 1:
        # bench mode runs past convergence; a comparison solver can hit an exact
        # breakdown in the rounding-noise regime (e.g. classic BiCGStab on cfg5 at
        # iteration 115).  The trajectory is deterministic, so a step of the
        # iterations before it is a fixed, complete unit of work.
        breakdown_at = r.iters
        maxit = r.iters - 1
        r = step()
    for _ in range(args.warmup - 1):
        r = step()
    assert r.iters == maxit, (r.iters, r.outcome)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=f"cuda:{dev}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    # ---- timed region: device time with CUDA events on the solver's stream
    # events around every kernel (graphs off; the headline's launches are ms-long)
    S.set_option("timing", 1 if args.kernel_timing else 0)
    S.kernel_time("all", reset=True)
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clk:
        e0.record(stream)
        iters = 0
        for _ in range(args.steps):
            iters += step().iters
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1))
    launches, _ = S.kernel_time("all")
    per_kernel = {}
    for k in ("sweepA", "sweepC", "spmvB", "spmvD", "rr1", "rr2", "gap", "init", "apply", "fin",
              "cl1", "cl2", "cl3", "pcg", "prec"):
        nk, tk = S.kernel_time(k)
        if nk:
            per_kernel[k] = {"launches": nk, "avg_ms": tk / nk if args.kernel_timing else None,
                             "bytes": S.kernel_bytes(k)}
    S.set_option("timing", 0)

    # ---- end to end: host (pinned) b, x0 -> solve -> host x, through the C ABI
    hb = torch.empty(n, dtype=torch.float64, pin_memory=True)
    hb.copy_(b.cpu())
    hx0 = torch.zeros(n, dtype=torch.float64, pin_memory=True)
    hx = torch.empty(n, dtype=torch.float64, pin_memory=True)
    hbn, hx0n, hxn = hb.numpy(), hx0.numpy(), hx.numpy()
    S.solve_host(hbn, hx0n, tol=0.0, maxit=maxit, rr_period=rr, gap=gap, x_out=hxn)  # warm
    barrier()
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    e2e_iters = 0
    e2e_steps = max(1, args.steps // 2)
    for _ in range(e2e_steps):
        e2e_iters += S.solve_host(hbn, hx0n, tol=0.0, maxit=maxit, rr_period=rr, gap=gap,
                                  x_out=hxn).iters
    f1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(f0.elapsed_time(f1))
    if rank != 0:
        return 0

    peak, peak_src = measured_peak()
    # strong scaling: every rank advances the same global iterations
    value = iters / (ms / 1000.0)
    # dominant kernel = largest share of the timed region
    if args.kernel_timing:
        dom = max(per_kernel, key=lambda k: per_kernel[k]["avg_ms"] * per_kernel[k]["launches"])
        k_avg_s = per_kernel[dom]["avg_ms"] / 1000.0
    else:
        dom, k_avg_s = "sweepC", float("nan")
    kb = per_kernel[dom]["bytes"]
    achieved = kb / k_avg_s / 1e9
    it_bytes = S.kernel_bytes("iteration") * world  # all ranks' algorithmic bytes per iteration
    profiled = (world == 1 and args.block == 1 and not args.rr_auto and args.schedule == 0
                and not args.loopback and (st.dim or args.method == "pbicgstab"))
    traffic = ncu_traffic(cfg.name, dom) if profiled else None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded x* ~ U[-1,1], b = A x* on device)",
        "config": {**bench_config(args, cfg, st, maxit, rr, world),
                   **({"breakdown_at": breakdown_at} if breakdown_at else {})},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "algorithmic_bytes_per_launch": kb, "peak_source": peak_src,
                     "iteration_frac": (it_bytes * value / world / 1e9) / peak,
                     # SURVEY 8(d)'s model of the 4-phase schedule (256 B/row stencil,
                     # 944 B/row CSR): the fused schedule moves fewer bytes, so > 1
                     "iteration_frac_4phase_model": ((256 if st.dim else 944) * st.n * value / world
                                                     / 1e9) / peak
                                                    if args.method == "pbicgstab" else None},
        "kernels": per_kernel,
        "gpu_launches": launches,
        "e2e": {"value": e2e_iters / (e2e_ms / 1000.0), "unit": UNIT,
                "h2d_bytes_per_step": 2 * 8 * n * world,
                "d2h_bytes_per_step": 8 * n * world + 8 * (maxit + 1) * (2 if gap else 1)},
        "clocks": clk.summary(),
    }
    if not args.no_cpu_baseline and world == 1:
        rows_per_s, n_s, its, t = oracle_sample(st, 6 if st.dim else 3, 64, cfg, args.method,
                                                args.block)
        line["cpu_baseline"] = {
            "value": rows_per_s / st.n, "unit": UNIT, "cores": 1, "kind": "oracle",
            "cpu": cpu_model(), "pinning": "sched_setaffinity to one core (taskset -c)",
            "sample": f"oracle {args.method} (C, 1 core) on {sample_desc(st, cfg)} "
                      f"({n_s} rows), {its} iterations in {t:.1f} s, scaled by rows to {st.n}"}
    print(json.dumps(line), flush=True)
    return 0


def run_loopback(args):
    """--loopback P: the multi-rank code path (partition, halos, rank-row
    reductions, finalize kernels) with P ranks emulated on ONE GPU.  Not a
    scaling number: it measures the overhead of the distributed schedule."""
    import torch
    from paper_1809_01948_b200 import binding
    cfg, st, maxit, rr = workload(args.config)
    P = args.loopback
    G = binding.LoopbackGroup.stencil(P, st.dim, st.nx, st.ny, st.nz, st.coef)
    xs = torch.from_numpy(problems.x_star(st.n, 0)).cuda()
    bs = G.apply(G.split(xs))
    del xs
    G.set_option("bench", 1)
    G.set_option("overlap", args.overlap)
    G.set_option("transport", args.transport)
    if args.schedule:
        G.set_option("schedule", args.schedule)
    for _ in range(args.warmup):
        G.solve(bs, tol=0.0, maxit=maxit, rr_period=rr, gap=bool(args.gap))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        r = G.solve(bs, tol=0.0, maxit=maxit, rr_period=rr, gap=bool(args.gap))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(json.dumps({"mode": f"loopback x{P} on 1 GPU", "config": cfg.name,
                      "iterations_per_s": args.steps * maxit / dt, "iters": r.iters}), flush=True)
    G.close()
    return 0


def relaunch_under_torchrun(n: int, need_gpus: bool = True) -> int:
    """`bench.py --gpus N` started without torchrun: re-exec this command as N ranks
    (one process per GPU, NCCL over NVLink) exactly as the driver launches it;
    rank 0 prints the JSON line.  NCCL's own log level is left to the caller."""
    import socket
    try:
        import torch
        have = torch.cuda.device_count()
    except Exception:
        have = 0
    if need_gpus and have < n:
        print(f"bench.py: --gpus {n} needs {n} visible GPUs, found {have}", file=sys.stderr)
        return 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--method", choices=["pbicgstab", "bicgstab", "pipecg"], default="pbicgstab",
                    help="solver: p-BiCGStab (the headline), classic BiCGStab or p-CG")
    ap.add_argument("--gap", type=int, default=0)
    ap.add_argument("--block", type=lambda v: int(v) if v.isdigit() else v, default=1,
                    help="preconditioner: block-Jacobi block size (1 = Jacobi; CSR 2..32, "
                         "stencils 2|4|8), or ilu0 / icc0 (reading A34)")
    ap.add_argument("--rr-auto", type=int, default=0,
                    help="automated residual replacement (bound f^r + eq:criterion) instead of "
                         "the periodic schedule")
    ap.add_argument("--schedule", type=int, default=0,
                    help="stencil p-BiCGStab: 0 auto (fused), 1 fused 2-sweep, 2 the paper's split "
                         "4-phase pipeline")
    ap.add_argument("--transport", type=int, default=0,
                    help="P > 1 reductions: 0 NCCL all-reduce, 1 peer-memory stores + flags")
    ap.add_argument("--overlap", type=int, default=1,
                    help="P > 1: dot-product reductions overlap the halo exchange / SpMV (1) "
                         "or block the compute stream (0)")
    ap.add_argument("--csr-tma", type=int, default=1,
                    help="point-wise sweeps (CSR; stencil --schedule 2) on the TMA chunk ring "
                         "(1, default) or per-row loads (0)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--kernel-timing", type=int, default=1,
                    help="1: CUDA events around every kernel in the timed region (graphs off); "
                         "0: CUDA-graph replay, no per-kernel times")
    ap.add_argument("--loopback", type=int, default=0,
                    help="emulate P ranks on one GPU (multi-rank code path check)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("note: warmup raised to 3 (timing rules)", file=sys.stderr)
        args.warmup = 3
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_under_torchrun(args.gpus, need_gpus=args.impl == "ours")
    if args.gpus != world:
        print(f"note: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if args.loopback:
        return run_loopback(args)
    return run_ours(args, rank, world)


if __name__ == "__main__":
    sys.exit(main())
