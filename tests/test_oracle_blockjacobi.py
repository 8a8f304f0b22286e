"""Pins of the oracle's block-Jacobi preconditioner ("block
preconditioners" P:741; reading A33): M = the b x b diagonal blocks of A,
inverted by Gauss-Jordan elimination, applied as a block-diagonal matvec.

1. Gauss-Jordan: exact on matrices whose inverse is exactly representable,
   within the condition-number bound of LAPACK's inverse otherwise;
2. b = 1 is the Jacobi preconditioner bitwise; M (M^{-1} u) = u to rounding, and
   M^{-1} u equals an independent per-block LAPACK solve to rounding;
3. exact-rational replay: Alg. 1 and Alg. 2 with the same (exact) block-diagonal
   M^{-1} produce identical iterates, and the fp64 oracle follows them;
4. converged solutions agree with dense LU; block Jacobi accelerates the 2D
   Poisson solve (fewer iterations than Jacobi).
"""
from fractions import Fraction as F

import numpy as np
import pytest

from oracle import rational as R
from paper_1809_01948_b200 import problems


def test_gauss_jordan(orc):
    D = np.diag([2.0, -4.0, 0.5, 8.0])
    assert np.array_equal(orc.gauss_jordan(D), np.diag([0.5, -0.25, 2.0, 0.125]))
    P = np.array([[0, 2.0, 0], [0, 0, 4.0], [-1.0, 0, 0]])  # scaled permutation
    with pytest.raises(ValueError):  # no pivoting: a zero leading pivot is refused
        orc.gauss_jordan(P)
    rng = np.random.default_rng(0)
    for b in (1, 2, 3, 4, 8, 16):
        B = rng.uniform(-1, 1, (b, b))
        B += np.diag(np.abs(B).sum(1) + 0.5)
        inv = orc.gauss_jordan(B)
        ref = np.linalg.inv(B)
        cond = np.linalg.cond(B)
        assert np.linalg.norm(inv - ref) <= 20 * b * cond * 2.0 ** -52 * np.linalg.norm(ref)
        assert np.linalg.norm(B @ inv - np.eye(b)) <= 20 * b * cond * 2.0 ** -52
    assert orc.gauss_jordan(np.array([[3.0]]))[0, 0] == 1.0 / 3.0


def test_prec_apply(orc):
    P = problems.csr_band(512, nnz_row=27, band=40, seed=4)
    A = orc.csr(P.row_ptr, P.col, P.val)
    D = A.dense()
    u = problems.x_star(A.n, 7)
    assert np.array_equal(orc.prec_apply(A, u, 1), orc.jacobi_dinv(A) * u)
    for b in (2, 4, 8, 32):
        v = orc.prec_apply(A, u, b)
        ref = np.concatenate([np.linalg.solve(D[k:k + b, k:k + b], u[k:k + b])
                              for k in range(0, A.n, b)])
        assert np.linalg.norm(v - ref) <= 1e-14 * np.linalg.norm(ref)
        Mv = np.concatenate([D[k:k + b, k:k + b] @ v[k:k + b] for k in range(0, A.n, b)])
        assert np.linalg.norm(Mv - u) <= 1e-14 * np.linalg.norm(u)
    with pytest.raises(ValueError):
        orc.prec_apply(orc.csr(P.row_ptr[:11], P.col[:P.row_ptr[10]], P.val[:P.row_ptr[10]]),
                       u[:10], 4)  # n not a multiple of b


def _block_inverse_exact(orc, A, b):
    """The oracle's fp64 block inverse, as exact rationals (columns M^{-1} e_j)."""
    n = A.n
    cols = [orc.prec_apply(A, np.eye(n)[j], b) for j in range(n)]
    return [[F(float(cols[j][i])) for j in range(n)] for i in range(n)]


@pytest.mark.parametrize("seed", [0, 2])
def test_alg1_equals_alg2_exactly_block_jacobi(orc, seed):
    from test_oracle_rational import dense_to_csr, small_unsym
    n, b = 8, 4
    A = small_unsym(n, seed)
    Ac = dense_to_csr(orc, A)
    Minv = _block_inverse_exact(orc, Ac, b)
    rng = np.random.default_rng(10 + seed)
    xs = rng.integers(-5, 6, n).astype(float)
    bf = R.fvec(A @ xs)
    Af = R.fmat(A)
    x0 = [F(0)] * n
    c = R.bicgstab(Af, Minv, bf, x0, 4)
    p = R.pbicgstab(Af, Minv, bf, x0, 4)
    for i in range(4):
        assert c[i + 1]["x"] == p[i + 1]["x"]
        assert c[i + 1]["r"] == p[i + 1]["r"]
    # the fp64 oracle follows the exact iterates
    res = orc.pbicgstab(Ac, A @ xs, tol=0.0, maxit=4, bench=True, block=b, want_trace=True)
    for i in range(3):
        xe = np.array([float(v) for v in p[i + 1]["x"]])
        assert np.linalg.norm(res.trace[i + 1, 0] - xe) <= 1e-12 * np.linalg.norm(xe)


@pytest.mark.parametrize("b", [2, 4, 8])
def test_block_jacobi_solutions_dense_lu(orc, b):
    for A in (orc.stencil_csr(2, 16, 16, 1, problems.cfg2_coef()),
              orc.csr(*[getattr(problems.csr_band(2048, nnz_row=27, band=64, seed=5), k)
                        for k in ("row_ptr", "col", "val")])):
        xs = problems.x_star(A.n, 1)
        bb = orc.spmv(A, xs)
        xl = np.linalg.solve(A.dense(), bb)
        for solve in (orc.pbicgstab, orc.bicgstab):
            r = solve(A, bb, tol=1e-13, maxit=600, block=b)
            assert r.outcome == "converged"
            assert np.linalg.norm(r.x - xl) <= 1e-8 * np.linalg.norm(xl)


def test_block_jacobi_accelerates_poisson(orc):
    st = problems.configs()["cfg1"].stencil
    A = orc.stencil_csr(2, st.nx, st.ny, 1, st.coef)
    xs = problems.x_star(A.n, 0)
    b = orc.spmv(A, xs)
    its = {blk: orc.pbicgstab(A, b, tol=1e-10, maxit=2000, block=blk).iters for blk in (1, 4, 20)}
    pcg = {blk: orc.pipecg(A, b, tol=1e-10, maxit=2000, block=blk).iters for blk in (1, 4, 20)}
    assert its[4] < its[1] and its[20] < its[4]
    assert pcg[4] < pcg[1] and pcg[20] < pcg[4]
