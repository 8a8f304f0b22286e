"""Thin ctypes binding of include/pbicgstab.h (argument marshalling only).

Every step of the p-BiCGStab iteration runs in libpbicgstab.so's CUDA kernels;
torch only supplies device memory and the stream.  There is no CPU fallback:
if the library or a CUDA device is missing, calls raise.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import numpy as np

from . import _build

STATUS = {0: "OK", 1: "EINVAL", 2: "ECUDA", 3: "ENCCL", 4: "ENOMEM", 5: "ESTATE"}
OUTCOMES = {0: "converged", 1: "maxit", 2: "breakdown"}
KERNELS = ["init", "sweepA", "sweepC", "spmvB", "spmvD", "rr1", "rr2", "gap", "apply", "fin",
           "cl1", "cl2", "cl3", "pcg", "prec"]
# option "method": 0 p-BiCGStab (Alg. 2), 1 classic BiCGStab (Alg. 1), 2 p-CG (reading A19)


def prec_code(block) -> int:
    """pbicg_prec value: 1 = Jacobi, PBICG_PREC_BJ(b) = 0x100 | b (block Jacobi),
    "ilu0" = PBICG_PREC_ILU0 (2), "icc0" = PBICG_PREC_ICC0 (3) (reading A34)."""
    if block in ("ilu0", "icc0"):
        return 2 if block == "ilu0" else 3
    return 1 if block == 1 else 0x100 | int(block)
METHODS = {"pbicgstab": 0, "bicgstab": 1, "pipecg": 2}


class PbicgError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"pbicgstab error {STATUS.get(status, status)}: {msg}")
        self.status = status


class _Stencil(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("nx", ctypes.c_int64), ("ny", ctypes.c_int64),
                ("nz", ctypes.c_int64), ("coef", ctypes.c_double * 7)]


class _Csr(ctypes.Structure):
    _fields_ = [("n_global", ctypes.c_int64), ("row_begin", ctypes.c_int64),
                ("n_local", ctypes.c_int64), ("row_ptr", ctypes.c_void_p),
                ("col", ctypes.c_void_p), ("val", ctypes.c_void_p)]


class _Dist(ctypes.Structure):
    _fields_ = [("nranks", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("nccl_id_halo", ctypes.c_void_p), ("nccl_id_red", ctypes.c_void_p)]


SYMBOLS = ["pbicgstab_create_stencil", "pbicgstab_create_csr", "pbicgstab_create_stencil_loopback",
           "pbicgstab_create_csr_loopback", "pbicgstab_apply_loopback", "pbicgstab_solve_loopback",
           "pbicgstab_local_rows", "pbicgstab_stencil_partition",
           "pbicgstab_set_option", "pbicgstab_apply", "pbicgstab_solve", "pbicgstab_solve_host",
           "pbicgstab_kernel_time", "pbicgstab_kernel_bytes", "pbicgstab_rr_info",
           "pbicgstab_scalar_trace",
           "pbicgstab_get_unique_id",
           "pbicgstab_last_error", "pbicgstab_destroy"]

_lib = None


def lib(build: bool = True):
    """Load libpbicgstab.so (building it with nvcc if stale).  Raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if build:
        try:
            _build.build()
        except Exception:
            if not os.path.exists(_build.LIB):
                raise
    if not os.path.exists(_build.LIB):
        raise RuntimeError(f"CUDA extension missing: {_build.LIB} (run __graft_entry__.build())")
    L = ctypes.CDLL(_build.LIB)
    P, i32, i64, f64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    L.pbicgstab_create_stencil.argtypes = [ctypes.POINTER(_Stencil), ctypes.c_int,
                                           ctypes.POINTER(_Dist), P, ctypes.POINTER(P)]
    L.pbicgstab_create_csr.argtypes = [ctypes.POINTER(_Csr), ctypes.c_int,
                                       ctypes.POINTER(_Dist), P, ctypes.POINTER(P)]
    L.pbicgstab_create_stencil_loopback.argtypes = [ctypes.POINTER(_Stencil), ctypes.c_int, i32, P,
                                                    P]
    L.pbicgstab_create_csr_loopback.argtypes = [P, ctypes.c_int, i32, P, P]
    L.pbicgstab_apply_loopback.argtypes = [P, i32, P, P]
    L.pbicgstab_solve_loopback.argtypes = [P, i32, P, P, f64, i32, i32, P, P, P,
                                           ctypes.POINTER(i32), ctypes.POINTER(i32)]
    L.pbicgstab_local_rows.argtypes = [P, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    L.pbicgstab_stencil_partition.argtypes = [ctypes.POINTER(_Stencil), i32, i32,
                                              ctypes.POINTER(i64), ctypes.POINTER(i64)]
    L.pbicgstab_set_option.argtypes = [P, ctypes.c_char_p, i64]
    L.pbicgstab_apply.argtypes = [P, P, P]
    L.pbicgstab_solve.argtypes = [P, P, P, f64, i32, i32, P, P, P, ctypes.POINTER(i32),
                                  ctypes.POINTER(i32)]
    L.pbicgstab_solve_host.argtypes = L.pbicgstab_solve.argtypes
    L.pbicgstab_kernel_time.argtypes = [P, ctypes.c_char_p, ctypes.POINTER(i64),
                                        ctypes.POINTER(f64), i32]
    L.pbicgstab_kernel_bytes.argtypes = [P, ctypes.c_char_p, ctypes.POINTER(f64)]
    L.pbicgstab_rr_info.argtypes = [P, P, P, i32, ctypes.POINTER(i32)]
    L.pbicgstab_scalar_trace.argtypes = [P, P, i32]
    L.pbicgstab_get_unique_id.argtypes = [P]
    L.pbicgstab_last_error.argtypes = [P]
    L.pbicgstab_last_error.restype = ctypes.c_char_p
    L.pbicgstab_destroy.argtypes = [P]
    L.pbicgstab_destroy.restype = None
    for name in SYMBOLS:
        if name not in ("pbicgstab_last_error", "pbicgstab_destroy"):
            getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


def _check(st: int, h=None):
    if st != 0:
        msg = lib().pbicgstab_last_error(h)
        raise PbicgError(st, msg.decode() if msg else "")


def _dptr(t, n: int, name: str):
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64
            and t.is_contiguous() and t.numel() == n):
        raise ValueError(f"{name}: expected a contiguous CUDA float64 tensor of {n} elements")
    return ctypes.c_void_p(t.data_ptr())


def _stream_ptr(stream):
    if stream is None:
        return None
    return ctypes.c_void_p(int(stream.cuda_stream) if hasattr(stream, "cuda_stream") else int(stream))


def stencil_partition(dim: int, nx: int, ny: int, nz: int, nranks: int, rank: int):
    """Rows [row_begin, row_begin + n_local) the stencil handle of `rank` owns (host-only)."""
    st = _Stencil(dim, nx, ny, nz if dim == 3 else 1, (ctypes.c_double * 7)(1, 0, 0, 0, 0, 0, 0))
    rb, nl = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().pbicgstab_stencil_partition(ctypes.byref(st), nranks, rank, ctypes.byref(rb),
                                             ctypes.byref(nl)))
    return rb.value, nl.value


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId from the library's NCCL (rank 0 calls this)."""
    buf = ctypes.create_string_buffer(128)
    _check(lib().pbicgstab_get_unique_id(buf))
    return buf.raw


def make_dist(nranks: int, rank: int, uid_halo: bytes, uid_red: bytes | None = None):
    """pbicg_dist for one process of an NCCL job (keeps the id buffers alive)."""
    bh = ctypes.create_string_buffer(uid_halo, 128)
    br = ctypes.create_string_buffer(uid_red, 128) if uid_red else None
    d = _Dist(nranks, rank, ctypes.cast(bh, ctypes.c_void_p),
              ctypes.cast(br, ctypes.c_void_p) if br is not None else None)
    d._keep = (bh, br)
    return d


@dataclass
class SolveResult:
    x: object            # torch tensor (device) or numpy (host solve)
    rnorm: np.ndarray    # ||r_i||, i = 0..iters
    gap: np.ndarray | None
    iters: int
    outcome: str


class Solver:
    """One p-BiCGStab handle (pbicg_handle)."""

    def __init__(self, handle: ctypes.c_void_p):
        self._h = handle
        rb, nl = ctypes.c_int64(), ctypes.c_int64()
        _check(lib().pbicgstab_local_rows(self._h, ctypes.byref(rb), ctypes.byref(nl)), self._h)
        self.row_begin, self.n_local = rb.value, nl.value

    # -- construction -----------------------------------------------------
    @classmethod
    def stencil(cls, dim: int, nx: int, ny: int, nz: int, coef, stream=None, dist=None,
                block: int = 1):
        st = _Stencil(dim, nx, ny, nz if dim == 3 else 1, (ctypes.c_double * 7)(*[float(c) for c in coef]))
        h = ctypes.c_void_p()
        d = ctypes.byref(dist) if dist is not None else None
        _check(lib().pbicgstab_create_stencil(ctypes.byref(st), prec_code(block), d,
                                              _stream_ptr(stream), ctypes.byref(h)))
        return cls(h)

    @classmethod
    def csr(cls, n_global: int, row_ptr, col, val, row_begin: int = 0, stream=None, dist=None,
            block: int = 1):
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(col, dtype=np.int32)
        va = np.ascontiguousarray(val, dtype=np.float64)
        c = _Csr(n_global, row_begin, len(rp) - 1, rp.ctypes.data, ci.ctypes.data, va.ctypes.data)
        h = ctypes.c_void_p()
        d = ctypes.byref(dist) if dist is not None else None
        _check(lib().pbicgstab_create_csr(ctypes.byref(c), prec_code(block), d,
                                          _stream_ptr(stream), ctypes.byref(h)))
        return cls(h)

    # -- API ------------------------------------------------------------------
    def set_option(self, key: str, value: int):
        _check(lib().pbicgstab_set_option(self._h, key.encode(), int(value)), self._h)

    def apply(self, x, y=None):
        import torch
        if y is None:
            y = torch.empty_like(x)
        _check(lib().pbicgstab_apply(self._h, _dptr(x, self.n_local, "x"),
                                     _dptr(y, self.n_local, "y")), self._h)
        return y

    def solve(self, b, x0=None, tol: float = 1e-10, maxit: int = 1000, rr_period: int = 0,
              gap: bool = True, x_out=None) -> SolveResult:
        import torch
        n = self.n_local
        if x0 is None:
            x0 = torch.zeros_like(b)
        if x_out is None:
            x_out = torch.empty_like(b)
        rh = np.full(maxit + 1, np.nan)
        gh = np.full(maxit + 1, np.nan) if gap else None
        it, oc = ctypes.c_int32(), ctypes.c_int32()
        _check(lib().pbicgstab_solve(
            self._h, _dptr(b, n, "b"), _dptr(x0, n, "x0"), float(tol), int(maxit),
            int(rr_period), _dptr(x_out, n, "x_out"), rh.ctypes.data_as(ctypes.c_void_p),
            None if gh is None else gh.ctypes.data_as(ctypes.c_void_p),
            ctypes.byref(it), ctypes.byref(oc)), self._h)
        k = it.value
        return SolveResult(x_out, rh[:k + 1], None if gh is None else gh[:k + 1], k,
                           OUTCOMES[oc.value])

    def solve_host(self, b: np.ndarray, x0: np.ndarray | None = None, tol: float = 1e-10,
                   maxit: int = 1000, rr_period: int = 0, gap: bool = True,
                   x_out: np.ndarray | None = None) -> SolveResult:
        n = self.n_local
        b = np.ascontiguousarray(b, dtype=np.float64)
        x0 = np.zeros(n) if x0 is None else np.ascontiguousarray(x0, dtype=np.float64)
        if b.size != n or x0.size != n:
            raise ValueError("b / x0 size mismatch")
        x = np.empty(n) if x_out is None else x_out
        rh = np.full(maxit + 1, np.nan)
        gh = np.full(maxit + 1, np.nan) if gap else None
        it, oc = ctypes.c_int32(), ctypes.c_int32()
        vp = lambda a: a.ctypes.data_as(ctypes.c_void_p)
        _check(lib().pbicgstab_solve_host(
            self._h, vp(b), vp(x0), float(tol), int(maxit), int(rr_period), vp(x), vp(rh),
            None if gh is None else vp(gh), ctypes.byref(it), ctypes.byref(oc)), self._h)
        k = it.value
        return SolveResult(x, rh[:k + 1], None if gh is None else gh[:k + 1], k, OUTCOMES[oc.value])

    def rr_info(self, iters: int):
        """(f^r history [iters+1] (NaN without rr_auto), replacement iterations) of the
        last solve (pbicgstab_rr_info)."""
        fr = np.full(iters + 1, np.nan)
        cap = max(iters, 1)
        rl = np.zeros(cap, np.int32)
        n = ctypes.c_int32()
        _check(lib().pbicgstab_rr_info(self._h, fr.ctypes.data_as(ctypes.c_void_p),
                                       rl.ctypes.data_as(ctypes.c_void_p), cap,
                                       ctypes.byref(n)), self._h)
        return fr, [int(v) for v in rl[:min(n.value, cap)]]

    def scalar_trace(self, iters: int) -> np.ndarray:
        """[iters, 9]: alpha_i, beta_i, omega_i, rho_i, (q,y), (y,y), (r0,w), (r0,s), (r0,z)
        of the last p-BiCGStab solve (pbicgstab_scalar_trace; the oracle's `scalars`)."""
        out = np.full((max(iters, 1), 9), np.nan)
        _check(lib().pbicgstab_scalar_trace(self._h, out.ctypes.data_as(ctypes.c_void_p),
                                            int(iters)), self._h)
        return out[:iters]

    def kernel_time(self, name: str = "all", reset: bool = False) -> tuple[int, float]:
        n, ms = ctypes.c_int64(), ctypes.c_double()
        _check(lib().pbicgstab_kernel_time(self._h, name.encode(), ctypes.byref(n),
                                           ctypes.byref(ms), int(reset)), self._h)
        return n.value, ms.value

    def kernel_bytes(self, name: str) -> float:
        b = ctypes.c_double()
        _check(lib().pbicgstab_kernel_bytes(self._h, name.encode(), ctypes.byref(b)), self._h)
        return b.value

    def close(self):
        if self._h:
            lib().pbicgstab_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


class LoopbackGroup:
    """P ranks of the multi-GPU path emulated on one device (loopback transport):
    the same partition, halo plan, rank-row reductions and finalize kernels as
    the NCCL path, with device-to-device copies in place of NCCL."""

    def __init__(self, handles):
        self._hs = handles  # ctypes array of c_void_p
        self.P = len(handles)
        self.ranks = [Solver(ctypes.c_void_p(h)) for h in handles]

    @classmethod
    def stencil(cls, nranks: int, dim: int, nx: int, ny: int, nz: int, coef, stream=None,
                block: int = 1):
        st = _Stencil(dim, nx, ny, nz if dim == 3 else 1,
                      (ctypes.c_double * 7)(*[float(c) for c in coef]))
        hs = (ctypes.c_void_p * nranks)()
        _check(lib().pbicgstab_create_stencil_loopback(ctypes.byref(st), prec_code(block), nranks,
                                                       _stream_ptr(stream), hs))
        return cls(hs)

    @classmethod
    def csr(cls, blocks, n_global: int, stream=None, block: int = 1):
        """blocks: list of (row_begin, row_ptr, col, val) per rank, contiguous."""
        keep = []
        arr = (_Csr * len(blocks))()
        for r, (rb, rp, ci, va) in enumerate(blocks):
            rp = np.ascontiguousarray(rp, dtype=np.int64)
            ci = np.ascontiguousarray(ci, dtype=np.int32)
            va = np.ascontiguousarray(va, dtype=np.float64)
            keep += [rp, ci, va]
            arr[r] = _Csr(n_global, rb, len(rp) - 1, rp.ctypes.data, ci.ctypes.data, va.ctypes.data)
        hs = (ctypes.c_void_p * len(blocks))()
        _check(lib().pbicgstab_create_csr_loopback(arr, prec_code(block), len(blocks),
                                                   _stream_ptr(stream), hs))
        return cls(hs)

    def set_option(self, key, value):
        self.ranks[0].set_option(key, value)  # applies to every member

    def split(self, v):
        return [v[s.row_begin:s.row_begin + s.n_local].contiguous() for s in self.ranks]

    def apply(self, xs):
        import torch
        ys = [torch.empty_like(x) for x in xs]
        xa = (ctypes.c_void_p * self.P)(*[_dptr(x, s.n_local, "x").value for x, s in zip(xs, self.ranks)])
        ya = (ctypes.c_void_p * self.P)(*[_dptr(y, s.n_local, "y").value for y, s in zip(ys, self.ranks)])
        _check(lib().pbicgstab_apply_loopback(self._hs, self.P, xa, ya), self._hs[0])
        return ys

    def solve(self, bs, x0s=None, tol=1e-10, maxit=1000, rr_period=0, gap=True):
        import torch
        if x0s is None:
            x0s = [torch.zeros_like(b) for b in bs]
        xs = [torch.empty_like(b) for b in bs]
        ptr = lambda ts, nm: (ctypes.c_void_p * self.P)(
            *[_dptr(t, s.n_local, nm).value for t, s in zip(ts, self.ranks)])
        rh = np.full(maxit + 1, np.nan)
        gh = np.full(maxit + 1, np.nan) if gap else None
        it, oc = ctypes.c_int32(), ctypes.c_int32()
        _check(lib().pbicgstab_solve_loopback(
            self._hs, self.P, ptr(bs, "b"), ptr(x0s, "x0"), float(tol), int(maxit),
            int(rr_period), ptr(xs, "x"), rh.ctypes.data_as(ctypes.c_void_p),
            None if gh is None else gh.ctypes.data_as(ctypes.c_void_p),
            ctypes.byref(it), ctypes.byref(oc)), self._hs[0])
        k = it.value
        return SolveResult(torch.cat(xs), rh[:k + 1], None if gh is None else gh[:k + 1], k,
                           OUTCOMES[oc.value])

    def close(self):
        for s in reversed(self.ranks):
            s.close()
        self.ranks = []
