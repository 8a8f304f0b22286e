"""Seeded synthetic inputs shaped like the paper's workloads.

This module is the ONLY code shared by the CUDA path and the oracle.  It holds
none of the method's arithmetic: it only defines operators (stencil coefficient
tables, random CSR band matrices) and draws the exact solution x*.  The right-hand
side b = A x* is computed by each side with its own SpMV (the GPU through
``pbicgstab_apply``, the oracle through ``orc_spmv``).

Paper workloads (Table 1): constant-coefficient 5-point / 7-point
stencils with Dirichlet boundaries, x-fastest natural ordering.  BASELINE.json
substitutes Jacobi, a seeded uniform x* and upwind convection-diffusion; the
readings are A15 (discretisation), A17 (CSR generator), A18 (x*, b).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

# coef order everywhere: {centre, -x, +x, -y, +y, -z, +z}  (include/pbicgstab.h)


def poisson2d_coef() -> list[float]:
    """TP1 stencil (Table 1): 4 centre, -1 neighbours."""
    return [4.0, -1.0, -1.0, -1.0, -1.0, 0.0, 0.0]


def poisson3d_coef() -> list[float]:
    return [6.0, -1.0, -1.0, -1.0, -1.0, -1.0, -1.0]


def convdiff_coef(dim: int, beta_h: tuple[float, ...]) -> list[float]:
    """-Lap u + beta . grad u, h^2-scaled, first-order upwind for beta > 0 (reading A15).

    beta_h[d] = beta_d * h = 2 * (cell Peclet number in direction d).
    Upwind difference beta_d (u_c - u_{-d}) / h adds beta_d*h to the centre and
    -beta_d*h to the upstream (-d) leg.  Centre accumulated in the order
    ((2*dim + b_x) + b_y) + b_z.
    """
    centre = float(2 * dim)
    for bh in beta_h:
        centre = centre + bh
    c = [centre, -(1.0 + beta_h[0]), -1.0, -(1.0 + beta_h[1]), -1.0, 0.0, 0.0]
    if dim == 3:
        c[5] = -(1.0 + beta_h[2])
        c[6] = -1.0
    return c


def cfg2_coef() -> list[float]:
    """cfg2: 2D upwind CD, cell Peclet 0.5 in x and y => beta*h = 1 (A15a): (6; -2,-1,-2,-1)."""
    return convdiff_coef(2, (1.0, 1.0))


def cfg34_coef() -> list[float]:
    """cfg3/cfg4: beta = c (1, 0.5, 0.25), max cell Peclet 0.8 => beta*h = (1.6, 0.8, 0.4) (A15b)."""
    return convdiff_coef(3, (1.6, 0.8, 0.4))


def x_star(n: int, seed: int = 0) -> np.ndarray:
    """Exact solution x* = default_rng(seed).uniform(-1, 1, n), global natural order (A18)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


@dataclass
class StencilProblem:
    dim: int
    nx: int
    ny: int
    nz: int
    coef: list[float]

    @property
    def n(self) -> int:
        return self.nx * self.ny * (self.nz if self.dim == 3 else 1)


@dataclass
class CSRProblem:
    n: int
    row_ptr: np.ndarray  # int64 [n+1]
    col: np.ndarray      # int32 [nnz], ascending per row, global ids
    val: np.ndarray      # float64 [nnz]


def csr_band(n: int, nnz_row: int = 27, band: int = 4096, dom: float = 1.2,
             seed: int = 1) -> CSRProblem:
    """cfg5 generator (reading A17).

    Row i: the diagonal plus (nnz_row - 1) distinct off-diagonal columns drawn
    uniformly without replacement from {j : |i - j| <= band, j != i, 0 <= j < n};
    off-diagonal values uniform[-1, 1]; a_ii = dom * sum_j |a_ij| summed in
    ascending column order.  Columns sorted ascending.  Seeded, vectorised.
    """
    rng = np.random.default_rng(seed)
    k = nnz_row - 1
    rows = np.arange(n, dtype=np.int64)
    lo = np.maximum(rows - band, 0)
    hi = np.minimum(rows + band, n - 1)
    width = hi - lo  # number of candidate off-diagonal columns
    if np.any(width < k):
        raise ValueError("band too narrow for the requested nnz per row")
    cols = np.empty((n, k), dtype=np.int64)
    todo = rows
    while todo.size:
        u = (rng.random((todo.size, k)) * width[todo, None]).astype(np.int64)
        u.sort(axis=1)
        ok = np.all(u[:, 1:] != u[:, :-1], axis=1)
        c = lo[todo, None] + u
        c += (c >= todo[:, None])  # skip the diagonal
        cols[todo[ok]] = c[ok]
        todo = todo[~ok]
    vals = rng.uniform(-1.0, 1.0, (n, k))
    s = np.zeros(n)
    for j in range(k):  # ascending column order
        s = s + np.abs(vals[:, j])
    diag = dom * s
    pos = (cols < rows[:, None]).sum(axis=1)
    C = np.empty((n, nnz_row), dtype=np.int32)
    V = np.empty((n, nnz_row))
    for j in range(nnz_row):
        before = j < pos
        at = j == pos
        jm = max(j - 1, 0)
        src_c = np.where(before, cols[:, min(j, k - 1)], cols[:, jm])
        src_v = np.where(before, vals[:, min(j, k - 1)], vals[:, jm])
        C[:, j] = np.where(at, rows, src_c)
        V[:, j] = np.where(at, diag, src_v)
    row_ptr = np.arange(n + 1, dtype=np.int64) * nnz_row
    return CSRProblem(n, row_ptr, C.reshape(-1), V.reshape(-1))


@dataclass
class Config:
    name: str
    kind: str                     # "stencil" | "csr"
    desc: str
    tol: float
    maxit: int
    rr_period: int
    bench: bool = False
    stencil: StencilProblem | None = None
    csr_n: int = 0
    extra: dict = field(default_factory=dict)


def configs() -> dict[str, Config]:
    """BASELINE.json configs[0..4] as concrete synthetic inputs."""
    return {
        "cfg1": Config("cfg1", "stencil", "2D Poisson 5-pt 100x100, Jacobi, 500 its",
                       0.0, 500, 0, bench=True,
                       stencil=StencilProblem(2, 100, 100, 1, poisson2d_coef())),
        "cfg2": Config("cfg2", "stencil", "2D upwind conv-diff 1024^2, Pe 0.5, tol 1e-10",
                       1e-10, 6000, 0,
                       stencil=StencilProblem(2, 1024, 1024, 1, cfg2_coef())),
        "cfg3": Config("cfg3", "stencil", "3D upwind conv-diff 256^3, Pe 0.8, RR 50",
                       1e-10, 3000, 50,
                       stencil=StencilProblem(3, 256, 256, 256, cfg34_coef())),
        "cfg4": Config("cfg4", "stencil", "3D upwind conv-diff 512^3, 200 fixed its",
                       0.0, 200, 0, bench=True,
                       stencil=StencilProblem(3, 512, 512, 512, cfg34_coef())),
        "cfg5": Config("cfg5", "csr", "CSR band N=2^23, 27 nnz/row, bw 4096, RR 100",
                       1e-10, 1000, 100, csr_n=1 << 23),
    }
