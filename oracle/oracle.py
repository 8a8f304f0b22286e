"""TEST INFRASTRUCTURE ONLY -- ctypes binding of oracle.c.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use this
module.  Builds ``oracle/liboracle.so`` with gcc (-O2 -ffp-contract=off, no fast
math) the first time it is needed.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

BENCH = 1
PLAIN_DOT = 2
GAP = 4
AUTO_RR = 8
ILU0 = 16
NTRACE = 15
TRACE_NAMES = ["x", "r", "k", "w", "m", "t", "g", "s", "l", "z", "q", "u", "y", "n", "v"]
OUTCOMES = {0: "converged", 1: "maxit", 2: "breakdown"}


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (plain C, no contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
             "-shared", "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        P = ctypes.c_void_p
        i64, i32, f64 = ctypes.c_int64, ctypes.c_int32, ctypes.c_double
        L.orc_dot2.restype = f64
        L.orc_dot2.argtypes = [i64, P, P]
        L.orc_dot_plain.restype = f64
        L.orc_dot_plain.argtypes = [i64, P, P]
        L.orc_spmv.restype = None
        L.orc_spmv.argtypes = [i64, P, P, P, P, P]
        L.orc_jacobi_dinv.restype = ctypes.c_int
        L.orc_jacobi_dinv.argtypes = [i64, P, P, P, P]
        L.orc_stencil_csr.restype = i64
        L.orc_stencil_csr.argtypes = [ctypes.c_int, i64, i64, i64, P, P, P, P]
        L.orc_pbicgstab.restype = ctypes.c_int
        L.orc_pbicgstab.argtypes = [i64, P, P, P, P, P, f64, i32, i32, i32, P, P, P, P, P, P, P,
                                    P, P, P]
        L.orc_anorm_bound.restype = f64
        L.orc_anorm_bound.argtypes = [i64, P, P, P]
        L.orc_prec_apply.restype = ctypes.c_int
        L.orc_prec_apply.argtypes = [i64, P, P, P, i32, P, P]
        L.orc_ilu0_factor.restype = ctypes.c_int
        L.orc_ilu0_factor.argtypes = [i64, P, P, P, P, P]
        L.orc_set_prec_matrix.restype = None
        L.orc_set_prec_matrix.argtypes = [i64, P, P, P]
        L.orc_gauss_jordan.restype = ctypes.c_int
        L.orc_gauss_jordan.argtypes = [ctypes.c_int, P, P]
        L.orc_bicgstab.restype = ctypes.c_int
        L.orc_bicgstab.argtypes = [i64, P, P, P, P, P, f64, i32, i32, P, P, P, P, P, P]
        for name in ("orc_pcg", "orc_pipecg"):
            f = getattr(L, name)
            f.restype = ctypes.c_int
            f.argtypes = [i64, P, P, P, P, P, f64, i32, i32, P, P, P, P, P]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


@dataclass
class CSR:
    n: int
    rp: np.ndarray  # int64 [n+1]
    ci: np.ndarray  # int64 [nnz], ascending per row
    va: np.ndarray  # float64 [nnz]

    def dense(self) -> np.ndarray:
        A = np.zeros((self.n, self.n))
        for i in range(self.n):
            for p in range(self.rp[i], self.rp[i + 1]):
                A[i, self.ci[p]] += self.va[p]
        return A


def csr(rp, ci, va) -> CSR:
    rp = np.ascontiguousarray(rp, dtype=np.int64)
    return CSR(len(rp) - 1, rp, np.ascontiguousarray(ci, dtype=np.int64), _f64(va))


def stencil_csr(dim: int, nx: int, ny: int, nz: int, coef) -> CSR:
    """Stencil written out as CSR by the oracle (ascending columns, Dirichlet legs dropped)."""
    n = nx * ny * (nz if dim == 3 else 1)
    rp = np.zeros(n + 1, np.int64)
    ci = np.zeros(7 * n, np.int64)
    va = np.zeros(7 * n)
    c = _f64(coef)
    nnz = lib().orc_stencil_csr(dim, nx, ny, nz, _p(c), _p(rp), _p(ci), _p(va))
    return CSR(n, rp, ci[:nnz].copy(), va[:nnz].copy())


def dot2(x, y) -> float:
    x, y = _f64(x), _f64(y)
    return lib().orc_dot2(len(x), _p(x), _p(y))


def dot_plain(x, y) -> float:
    x, y = _f64(x), _f64(y)
    return lib().orc_dot_plain(len(x), _p(x), _p(y))


def spmv(A: CSR, x) -> np.ndarray:
    x = _f64(x)
    y = np.zeros(A.n)
    lib().orc_spmv(A.n, _p(A.rp), _p(A.ci), _p(A.va), _p(x), _p(y))
    return y


def jacobi_dinv(A: CSR) -> np.ndarray:
    d = np.zeros(A.n)
    if lib().orc_jacobi_dinv(A.n, _p(A.rp), _p(A.ci), _p(A.va), _p(d)) != 0:
        raise ValueError("zero or missing diagonal")
    return d


@dataclass
class Result:
    x: np.ndarray
    rnorm: np.ndarray   # ||r_i||, i = 0..iters
    gap: np.ndarray | None  # ||(b - A x_i) - r_i||, i = 0..iters
    iters: int
    outcome: str
    scalars: np.ndarray | None = None  # [iters, 4]: alpha, beta, omega, rho
    trace: np.ndarray | None = None    # [maxit+1, NTRACE, n]
    bounds: np.ndarray | None = None   # [iters+1, 4]: f^r_i, Dw_i, Ds_i, Dz_i (auto RR)
    rr_iters: list | None = None       # iterations i that replaced r_{i+1} (auto RR)


def _run(fn, A: CSR, b, x0, tol, maxit, flags, extra=(), want_sc=False, want_trace=False,
         gap=True, want_bounds=False):
    b = _f64(b)
    x0 = np.zeros(A.n) if x0 is None else _f64(x0)
    x = np.zeros(A.n)
    rh = np.full(maxit + 1, np.nan)
    gh = np.full(maxit + 1, np.nan) if gap else None
    if gap:
        flags |= GAP
    it = ctypes.c_int32(0)
    oc = ctypes.c_int32(0)
    args = [A.n, _p(A.rp), _p(A.ci), _p(A.va), _p(b), _p(x0), float(tol), int(maxit), *extra,
            int(flags), _p(x), _p(rh), _p(gh), ctypes.byref(it), ctypes.byref(oc)]
    sc = tr = None
    if fn in ("orc_pbicgstab", "orc_bicgstab"):
        # p-BiCGStab: alpha, beta, omega, rho + the raw dots (q,y), (y,y), (r0,w), (r0,s), (r0,z)
        sc = np.full((maxit + 1, 9 if fn == "orc_pbicgstab" else 4), np.nan) if want_sc else None
        args.append(_p(sc))
    bt = rl = None
    nrr = ctypes.c_int32(0)
    if fn == "orc_pbicgstab":
        tr = np.zeros((maxit + 1, NTRACE, A.n)) if want_trace else None
        args.append(_p(tr))
        bt = np.full((maxit + 1, 4), np.nan) if want_bounds else None
        rl = np.zeros(max(maxit, 1), np.int32)
        args += [_p(bt), _p(rl), ctypes.byref(nrr)]
    rc = getattr(lib(), fn)(*args)
    if rc != 0:
        raise ValueError(f"{fn} failed with code {rc}")
    n_it = it.value
    return Result(x, rh[: n_it + 1], None if gh is None else gh[: n_it + 1], n_it,
                  OUTCOMES[oc.value], None if sc is None else sc[:n_it + 1], tr,
                  None if bt is None else bt[:n_it + 1],
                  None if rl is None else [int(v) for v in rl[:nrr.value]])


def _blk(block) -> int:
    """Preconditioner flags: an int = block size of the block-Jacobi preconditioner in
    bits 8-15 (1 = Jacobi); "ilu0" / "icc0" = ILU(0) (ICC(0) for symmetric A, A34)."""
    if block in ("ilu0", "icc0"):
        return ILU0
    if not 1 <= block <= 255:
        raise ValueError("block size must be in 1..255")
    return (block if block > 1 else 0) << 8


class prec_matrix:
    """Context manager: the matrix whose ILU(0) defines M (default A itself), e.g.
    block_diagonal(A, cuts) for the multi-rank reading of A34."""

    def __init__(self, Mtx: "CSR | None"):
        self.M = Mtx

    def __enter__(self):
        if self.M is not None:
            lib().orc_set_prec_matrix(self.M.n, _p(self.M.rp), _p(self.M.ci), _p(self.M.va))
        return self

    def __exit__(self, *a):
        lib().orc_set_prec_matrix(-1, None, None, None)


def block_diagonal(A: "CSR", cuts) -> "CSR":
    """A with every entry coupling two different row blocks [cuts[r], cuts[r+1]) dropped."""
    part = np.searchsorted(np.asarray(cuts[1:], np.int64), np.arange(A.n), side="right")
    rows = np.repeat(np.arange(A.n), np.diff(A.rp))
    keep = part[rows] == part[A.ci]
    rp = np.concatenate([[0], np.cumsum(np.bincount(rows[keep], minlength=A.n))]).astype(np.int64)
    return CSR(A.n, rp, A.ci[keep].copy(), A.va[keep].copy())


def ilu0_factor(A: "CSR"):
    """The oracle's ILU(0) factors on A's pattern: (lu values aligned with A.ci:
    multipliers l_ik below the diagonal, u_ij on and above it; uinv = 1/u_ii)."""
    lu = np.zeros(len(A.va))
    uinv = np.zeros(A.n)
    if lib().orc_ilu0_factor(A.n, _p(A.rp), _p(A.ci), _p(A.va), _p(lu), _p(uinv)) != 0:
        raise ValueError("ILU(0): missing or zero pivot")
    return lu, uinv


def pbicgstab(A: CSR, b, x0=None, tol=0.0, maxit=100, rr_period=0, bench=False,
              plain_dot=False, gap=True, want_scalars=False, want_trace=False,
              auto_rr=False, block=1) -> Result:
    """Alg. 2 with periodic replacement or, with auto_rr, the
    automated replacement of P:609-623 (bound f^r_i history in .bounds, replacement
    iterations in .rr_iters), and the gap history.  block > 1: block-Jacobi
    preconditioner with block x block diagonal blocks (reading A33)."""
    flags = ((BENCH if bench else 0) | (PLAIN_DOT if plain_dot else 0) |
             (AUTO_RR if auto_rr else 0) | _blk(block))
    return _run("orc_pbicgstab", A, b, x0, tol, maxit, flags, extra=(int(rr_period),),
                want_sc=want_scalars, want_trace=want_trace, gap=gap, want_bounds=auto_rr)


def anorm_bound(A: CSR) -> float:
    """sqrt(||A||_1 ||A||_inf) >= ||A||_2, the ||A|| of the run-time bound (reading A29)."""
    return lib().orc_anorm_bound(A.n, _p(A.rp), _p(A.ci), _p(A.va))


def bicgstab(A: CSR, b, x0=None, tol=0.0, maxit=100, bench=False, plain_dot=False, gap=True,
             want_scalars=False, block=1) -> Result:
    """Alg. 1."""
    flags = (BENCH if bench else 0) | (PLAIN_DOT if plain_dot else 0) | _blk(block)
    return _run("orc_bicgstab", A, b, x0, tol, maxit, flags, want_sc=want_scalars, gap=gap)


def pcg(A: CSR, b, x0=None, tol=0.0, maxit=100, bench=False, gap=True, block=1) -> Result:
    return _run("orc_pcg", A, b, x0, tol, maxit, (BENCH if bench else 0) | _blk(block), gap=gap)


def pipecg(A: CSR, b, x0=None, tol=0.0, maxit=100, bench=False, gap=True, block=1) -> Result:
    return _run("orc_pipecg", A, b, x0, tol, maxit, (BENCH if bench else 0) | _blk(block),
                gap=gap)


def prec_apply(A: CSR, u, block=1) -> np.ndarray:
    """M^{-1} u with the oracle's preconditioner (Jacobi or block Jacobi, A3 / A33)."""
    u = _f64(u)
    v = np.zeros(A.n)
    if lib().orc_prec_apply(A.n, _p(A.rp), _p(A.ci), _p(A.va), _blk(block), _p(u), _p(v)) != 0:
        raise ValueError("preconditioner undefined (zero pivot / block size)")
    return v


def gauss_jordan(B) -> np.ndarray:
    """The oracle's Gauss-Jordan inverse of a small dense matrix (no pivoting)."""
    a = np.ascontiguousarray(B, dtype=np.float64).copy()
    e = np.zeros_like(a)
    if lib().orc_gauss_jordan(a.shape[0], _p(a), _p(e)) != 0:
        raise ValueError("zero pivot")
    return e
