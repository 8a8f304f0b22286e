"""Pins for the oracle's building blocks (SpMV, stencils, Jacobi, Dot2).

Each pin checks the oracle against something other than itself: exact rational
sums, closed-form eigenpairs of the discrete operators, brute-force dense builds
and a hand-checkable example.
"""
import math
from fractions import Fraction as F

import numpy as np
import pytest

from paper_1809_01948_b200 import problems

EPS = 2.0 ** -53


def exact_dot(x, y):
    return sum((F(float(a)) * F(float(b)) for a, b in zip(x, y)), F(0))


def test_dot_examples(orc):
    # SPEC S:100 examples: (1,1,1,1).(1,2,3,4) = 10; e1.e1 = 1; e1.e2 = 0
    assert orc.dot2([1, 1, 1, 1], [1, 2, 3, 4]) == 10.0
    assert orc.dot_plain([1, 1, 1, 1], [1, 2, 3, 4]) == 10.0
    assert orc.dot2([1, 0], [1, 0]) == 1.0
    assert orc.dot2([1, 0], [0, 1]) == 0.0
    assert orc.dot2([], []) == 0.0


@pytest.mark.parametrize("seed", range(6))
def test_dot2_correctly_rounded_well_conditioned(orc, seed):
    """Dot2 (reading A6) equals the exactly rounded dot for well-conditioned data
    (Ogita-Rump-Oishi: error <= eps|s| + gamma_n^2 sum|x y|)."""
    rng = np.random.default_rng(seed)
    n = 1000 + 137 * seed
    x, y = rng.uniform(0, 1, n), rng.uniform(0, 1, n)
    assert orc.dot2(x, y) == float(exact_dot(x, y))


@pytest.mark.parametrize("seed", range(4))
def test_dot2_bound_ill_conditioned(orc, seed):
    """Heavy cancellation: Dot2 stays within eps|s| + gamma_n^2 sum|x_i y_i|, while
    a plain sum loses all digits."""
    rng = np.random.default_rng(100 + seed)
    n = 2000
    x = rng.uniform(-1, 1, n) * 2.0 ** rng.integers(-30, 30, n)
    y = rng.uniform(-1, 1, n)
    # append the negated products to force cancellation down to a tiny residue
    x = np.concatenate([x, x, [1e-20]])
    y = np.concatenate([y, -y, [1.0]])
    ex = exact_dot(x, y)
    d2 = orc.dot2(x, y)
    nn = len(x)
    gam = nn * EPS / (1 - nn * EPS)
    bound = EPS * abs(float(ex)) + gam * gam * float(sum(abs(F(a) * F(b)) for a, b in zip(x, y)))
    assert abs(F(d2) - ex) <= F(bound)
    assert d2 == pytest.approx(1e-20, rel=1e-12)


def test_spmv_1d_laplacian_example(orc):
    # 5x5 1D Laplacian [-1,2,-1] times (1,2,3,4,5) = (0,0,0,0,6)
    rp, ci, va = [0], [], []
    for i in range(5):
        for j in (i - 1, i, i + 1):
            if 0 <= j < 5:
                ci.append(j)
                va.append(2.0 if j == i else -1.0)
        rp.append(len(ci))
    A = orc.csr(rp, ci, va)
    assert list(orc.spmv(A, [1, 2, 3, 4, 5])) == [0, 0, 0, 0, 6]


def brute_dense_stencil(dim, nx, ny, nz, c):
    """Dense operator from the stencil definition (Dirichlet legs dropped)."""
    nz = nz if dim == 3 else 1
    n = nx * ny * nz
    A = np.zeros((n, n))
    for z in range(nz):
        for y in range(ny):
            for x in range(nx):
                row = x + nx * (y + ny * z)
                A[row, row] = c[0]
                for (dx, dy, dz, cc) in ((-1, 0, 0, c[1]), (1, 0, 0, c[2]), (0, -1, 0, c[3]),
                                         (0, 1, 0, c[4]), (0, 0, -1, c[5]), (0, 0, 1, c[6])):
                    xx, yy, zz = x + dx, y + dy, z + dz
                    if 0 <= xx < nx and 0 <= yy < ny and 0 <= zz < nz and (dim == 3 or dz == 0):
                        A[row, xx + nx * (yy + ny * zz)] = cc
    return A


@pytest.mark.parametrize("dim,nx,ny,nz,coef", [
    (2, 5, 4, 1, problems.poisson2d_coef()),
    (2, 6, 3, 1, problems.cfg2_coef()),
    (3, 4, 3, 5, problems.cfg34_coef()),
    (3, 3, 3, 3, problems.poisson3d_coef()),
])
def test_stencil_csr_matches_dense_definition(orc, dim, nx, ny, nz, coef):
    A = orc.stencil_csr(dim, nx, ny, nz, coef)
    D = brute_dense_stencil(dim, nx, ny, nz, coef)
    assert np.array_equal(A.dense(), D)
    for i in range(A.n):  # ascending columns (reading A5)
        cols = A.ci[A.rp[i]:A.rp[i + 1]]
        assert np.all(np.diff(cols) > 0)


def tridiag_eig_1d(n, a, c, b, j):
    """Eigenpair j of tridiag(a (sub), c, b (super)) of size n: lambda = c + 2 sqrt(ab) cos(j pi/(n+1)),
    v_i = (a/b)^(i/2) sin(i j pi/(n+1)), i = 1..n  (closed form)."""
    th = j * math.pi / (n + 1)
    lam = c + 2.0 * math.copysign(math.sqrt(a * b), a) * math.cos(th)
    i = np.arange(1, n + 1)
    v = (a / b) ** (i / 2.0) * np.sin(i * th)
    return lam, v


@pytest.mark.parametrize("name,dim,nx,ny,nz,coef,modes", [
    ("poisson2d", 2, 30, 20, 1, problems.poisson2d_coef(), [(1, 1, 0), (3, 5, 0), (29, 19, 0)]),
    ("cd2d", 2, 24, 17, 1, problems.cfg2_coef(), [(1, 2, 0), (7, 3, 0)]),
    ("cd3d", 3, 9, 8, 7, problems.cfg34_coef(), [(1, 1, 1), (2, 5, 3)]),
])
def test_stencil_closed_form_eigenpairs(orc, name, dim, nx, ny, nz, coef, modes):
    """Separable constant-coefficient operator: A v = lambda v with v the tensor
    product of 1D eigenvectors of tridiag(c_-d, ., c_+d); this fixes both the
    coefficients and their orientation (the -x leg multiplies x_{i-1})."""
    A = orc.stencil_csr(dim, nx, ny, nz, coef)
    sizes = [nx, ny] + ([nz] if dim == 3 else [])
    legs = [(coef[1], coef[2]), (coef[3], coef[4]), (coef[5], coef[6])][:dim]
    for mode in modes:
        lam = coef[0]
        v = np.ones(1)
        for d in range(dim):
            a, b = legs[d]
            l1, v1 = tridiag_eig_1d(sizes[d], a, 0.0, b, mode[d])
            lam += l1
            v = np.kron(v1, v)  # x fastest
        Av = orc.spmv(A, v)
        assert np.linalg.norm(Av - lam * v) <= 1e-13 * np.linalg.norm(v) * abs(coef[0])


def test_jacobi_dinv(orc):
    A = orc.stencil_csr(3, 3, 3, 3, problems.cfg34_coef())
    d = orc.jacobi_dinv(A)
    assert np.all(d == 1.0 / 8.8)
    B = orc.csr([0, 1, 2], [0, 1], [2.0, 0.0])
    with pytest.raises(ValueError):
        orc.jacobi_dinv(B)


def test_csr_band_generator_invariants(orc):
    P = problems.csr_band(3000, nnz_row=27, band=200, seed=3)
    rp, col, val = P.row_ptr, P.col.astype(np.int64), P.val
    assert rp[-1] == 27 * 3000
    for i in range(0, 3000, 7):
        c = col[rp[i]:rp[i + 1]]
        v = val[rp[i]:rp[i + 1]]
        assert np.all(np.diff(c) > 0)
        assert np.all(np.abs(c - i) <= 200)
        d = v[c == i]
        assert len(d) == 1
        off = v[c != i]
        assert np.all(np.abs(off) <= 1.0)
        s = 0.0
        for a in off:
            s = s + abs(a)
        assert d[0] == 1.2 * s  # strictly dominant diagonal (A17)
    # determinism
    Q = problems.csr_band(3000, nnz_row=27, band=200, seed=3)
    assert np.array_equal(P.col, Q.col) and np.array_equal(P.val, Q.val)


def test_stencil_spmv_equals_generic_csr_bitwise(orc):
    """The same operator as a stencil-generated CSR and as an independently
    built CSR gives bitwise-equal products (ascending-column order, A5)."""
    dim, nx, ny, nz = 3, 5, 4, 3
    coef = problems.cfg34_coef()
    A = orc.stencil_csr(dim, nx, ny, nz, coef)
    D = brute_dense_stencil(dim, nx, ny, nz, coef)
    rp, ci, va = [0], [], []
    for i in range(D.shape[0]):
        nz_ = np.nonzero(D[i])[0]
        ci += list(nz_)
        va += list(D[i, nz_])
        rp.append(len(ci))
    B = orc.csr(rp, ci, va)
    x = problems.x_star(A.n, seed=5)
    assert np.array_equal(orc.spmv(A, x), orc.spmv(B, x))


def test_table1_golden_stencils(orc):
    """Golden: Table 1 stencils.  Interior rows of TP1 sum to 0
    (SPEC S:56 example), TP3/TP5 interior rows sum to -eps (shifted Laplacians)."""
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "table1_stencils.json")))
    A = orc.stencil_csr(2, 7, 7, 1, g["TP1"]["coef"])
    s = orc.spmv(A, np.ones(A.n)).reshape(7, 7)
    assert np.all(s[1:-1, 1:-1] == 0.0) and np.all(s[0] > 0)
    for tp, dim in (("TP3", 2), ("TP5", 3)):
        e = g[tp]["eps"]
        c0 = g[tp]["coef_centre_minus_eps"] - e
        nb = g[tp]["neighbours"]
        coef = [c0, nb, nb, nb, nb, nb if dim == 3 else 0.0, nb if dim == 3 else 0.0]
        B = orc.stencil_csr(dim, 5, 5, 5, coef)
        s = orc.spmv(B, np.ones(B.n))
        interior = s.reshape((5, 5, 5) if dim == 3 else (5, 5))[(slice(1, -1),) * dim]
        assert np.allclose(interior, -e, rtol=0, atol=1e-15)
        D = B.dense()
        assert np.array_equal(D, D.T)  # symmetric (Table 1 "Sym.: Yes")
