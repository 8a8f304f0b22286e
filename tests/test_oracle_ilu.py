"""Pins of the oracle's ILU(0) / ICC(0) preconditioner (Table 1 "Precond." ICC(0),
P:659-697; "Incomplete Cholesky preconditioner with zero fill-in (ICC(0))", P:745;
SURVEY 8(f) NEXT-4; reading A34).  Nothing here re-types oracle.c's loops; each
pin checks the factorisation or its application against something else:

1. the defining property of an incomplete factorisation with zero fill: the
   product L U equals A on A's sparsity pattern.  Checked exactly: an exact-
   rational IKJ factorisation satisfies it with equality, and the fp64 factors
   of the oracle agree with the exact ones to a few ulps (a dropped update, a
   wrong operand or index leaves O(1) errors on the pattern);
2. for symmetric positive definite A the root-free ILU(0) is the incomplete
   Cholesky factorisation: L U equals L~ L~^T of the textbook IC(0) with square
   roots (a different algorithm, written below) to rounding;
3. where no fill is dropped (tridiagonal, block-diagonal tridiagonal) ILU(0) is the
   exact LU factorisation, so M^{-1} v is the dense LAPACK solve with A;
4. M^{-1} v (forward then backward substitution) equals a dense solve with the
   matrix L U to rounding;
5. exact-rational replay: Alg. 1 and Alg. 2 with the same exact ILU(0) M^{-1}
   generate identical iterates (P:4) and the fp64 oracle follows them;
6. converged solutions agree with dense LU, ICC(0) needs far fewer iterations
   than Jacobi on the 2D Poisson problem (TP1's setting), and the
   multi-rank reading (block-diagonal part) reduces to the one-rank one for one
   block and to block Jacobi's blocks being exactly LU-factorised when the blocks
   are tridiagonal.
"""
from fractions import Fraction as F

import numpy as np
import pytest

from oracle import rational as R
from paper_1809_01948_b200 import problems


def _pattern(A):
    return [(i, int(A.ci[p])) for i in range(A.n) for p in range(A.rp[i], A.rp[i + 1])]


def _lu_dense(A, lu):
    """Unit lower L (multipliers) and upper U from the oracle's lu values."""
    n = A.n
    L, U = np.eye(n), np.zeros((n, n))
    for i in range(n):
        for p in range(A.rp[i], A.rp[i + 1]):
            j = int(A.ci[p])
            if j < i:
                L[i, j] = lu[p]
            else:
                U[i, j] = lu[p]
    return L, U


def _ilu_exact(A):
    """Exact-rational ILU(0) (IKJ, restricted to the pattern) of a small CSR."""
    n = A.n
    rows = [{int(A.ci[p]): F(float(A.va[p])) for p in range(A.rp[i], A.rp[i + 1])}
            for i in range(n)]
    for i in range(n):
        for k in sorted(c for c in rows[i] if c < i):
            rows[i][k] = rows[i][k] / rows[k][k]
            for j in sorted(c for c in rows[k] if c > k):
                if j in rows[i]:
                    rows[i][j] = rows[i][j] - rows[i][k] * rows[k][j]
    return rows


def _small_cases(orc):
    out = [orc.stencil_csr(2, 5, 4, 1, problems.poisson2d_coef()),
           orc.stencil_csr(2, 4, 5, 1, problems.cfg2_coef()),
           orc.stencil_csr(3, 3, 3, 2, problems.cfg34_coef())]
    P = problems.csr_band(24, nnz_row=6, band=5, seed=3)
    out.append(orc.csr(P.row_ptr, P.col, P.val))
    return out


def test_lu_equals_a_on_the_pattern(orc):
    for A in _small_cases(orc):
        rows = _ilu_exact(A)
        # exact: (L U)_ij = a_ij on the pattern (the zero-fill property)
        for (i, j) in _pattern(A):
            lu_ij = sum((rows[i][k] if k < i else F(1)) * rows[k][j]
                        for k in range(min(i, j) + 1)
                        if (k == i or k in rows[i]) and j in rows[k])
            assert lu_ij == F(float(A.va[[int(A.ci[p]) for p in range(A.rp[i], A.rp[i + 1])].index(j) + A.rp[i]]))
        # fp64 factors of the oracle = exact factors to rounding
        lu, uinv = orc.ilu0_factor(A)
        for i in range(A.n):
            for p in range(A.rp[i], A.rp[i + 1]):
                ex = rows[i][int(A.ci[p])]
                assert abs(F(float(lu[p])) - ex) <= F(1, 2 ** 44) * (abs(ex) + 1)
            assert abs(F(float(uinv[i])) - 1 / rows[i][i]) <= F(1, 2 ** 44) * abs(1 / rows[i][i])
        L, U = _lu_dense(A, lu)
        D = A.dense()
        M = L @ U
        on = np.zeros_like(D, dtype=bool)
        for (i, j) in _pattern(A):
            on[i, j] = True
        assert np.max(np.abs((M - D)[on])) <= 1e-13 * np.max(np.abs(D))


def _ic0_textbook(D):
    """IC(0) with square roots (Golub & Van Loan / Saad "incomplete Cholesky"),
    right-looking, on the lower pattern of the symmetric matrix D (dense in,
    dense lower factor out)."""
    n = D.shape[0]
    pat = D != 0
    L = np.tril(D).copy()
    for k in range(n):
        L[k, k] = np.sqrt(L[k, k])
        for i in range(k + 1, n):
            if pat[i, k]:
                L[i, k] = L[i, k] / L[k, k]
        for j in range(k + 1, n):
            for i in range(j, n):
                if pat[i, j] and pat[i, k] and pat[j, k]:
                    L[i, j] = L[i, j] - L[i, k] * L[j, k]
    return L


def test_icc0_is_incomplete_cholesky(orc):
    st = orc.stencil_csr(2, 9, 7, 1, problems.poisson2d_coef())
    st3 = orc.stencil_csr(3, 4, 3, 5, [6.0, -1, -1, -1, -1, -1, -1])
    # symmetric band matrix: (B + B^T)/2 made diagonally dominant
    P = problems.csr_band(60, nnz_row=7, band=9, seed=8)
    Bd = orc.csr(P.row_ptr, P.col, P.val).dense()
    S = 0.5 * (Bd + Bd.T)
    np.fill_diagonal(S, 0.0)
    S = S + np.diag(np.abs(S).sum(1) * 1.1 + 1.0)
    Sc = orc.csr(*_dense_to_csr_arrays(S))
    for A in (st, st3, Sc):
        D = A.dense()
        assert np.array_equal(D, D.T)
        Lt = _ic0_textbook(D)
        lu, _ = orc.ilu0_factor(A)
        L, U = _lu_dense(A, lu)
        M_ic, M_ilu = Lt @ Lt.T, L @ U
        assert np.max(np.abs(M_ilu - M_ic)) <= 1e-13 * np.max(np.abs(D))
        # the dropped fill is real (IC(0) is not the exact Cholesky factorisation)
        assert np.max(np.abs(M_ilu - D)) > 1e-3


def _dense_to_csr_arrays(D):
    n = D.shape[0]
    rp, ci, va = [0], [], []
    for i in range(n):
        for j in range(n):
            if D[i, j] != 0.0:
                ci.append(j)
                va.append(D[i, j])
        rp.append(len(ci))
    return np.array(rp, np.int64), np.array(ci, np.int64), np.array(va)


def test_exact_lu_where_no_fill(orc):
    rng = np.random.default_rng(1)
    # 1D (tridiagonal) and 2D stencils with nx = 1 / ny = 1 are tridiagonal: no fill
    for A in (orc.stencil_csr(2, 40, 1, 1, problems.cfg2_coef()),
              orc.stencil_csr(2, 1, 33, 1, problems.poisson2d_coef()),
              orc.stencil_csr(3, 1, 1, 17, problems.cfg34_coef())):
        u = rng.uniform(-1, 1, A.n)
        v = orc.prec_apply(A, u, "ilu0")
        ref = np.linalg.solve(A.dense(), u)
        assert np.linalg.norm(v - ref) <= 1e-13 * np.linalg.norm(ref)


def test_apply_is_forward_backward_substitution(orc):
    rng = np.random.default_rng(2)
    P = problems.csr_band(300, nnz_row=11, band=20, seed=6)
    for A in (orc.stencil_csr(2, 13, 11, 1, problems.cfg2_coef()),
              orc.stencil_csr(3, 6, 5, 4, problems.cfg34_coef()),
              orc.csr(P.row_ptr, P.col, P.val)):
        lu, _ = orc.ilu0_factor(A)
        L, U = _lu_dense(A, lu)
        u = rng.uniform(-1, 1, A.n)
        v = orc.prec_apply(A, u, "ilu0")
        ref = np.linalg.solve(L @ U, u)
        assert np.linalg.norm(v - ref) <= 1e-12 * np.linalg.norm(ref)
        y = np.linalg.solve(L, u)  # the intermediate of the forward substitution
        assert np.linalg.norm(U @ v - y) <= 1e-12 * np.linalg.norm(y)
    with pytest.raises(ValueError):  # zero pivot
        Z = orc.csr(np.array([0, 2, 4]), np.array([0, 1, 0, 1]), np.array([1.0, 1.0, 1.0, 1.0]))
        orc.prec_apply(Z, np.ones(2), "ilu0")


def _ilu_minv_exact(A):
    """Exact M^{-1} = (L U)^{-1} of the exact ILU(0) factors, as rational rows."""
    n = A.n
    rows = _ilu_exact(A)
    M = [[sum((rows[i][k] if k < i else F(1)) * rows[k][j]
              for k in range(min(i, j) + 1) if (k == i or k in rows[i]) and j in rows[k])
          for j in range(n)] for i in range(n)]
    # Gauss-Jordan in rationals
    E = [[F(int(i == j)) for j in range(n)] for i in range(n)]
    for p in range(n):
        piv = M[p][p]
        M[p] = [a / piv for a in M[p]]
        E[p] = [a / piv for a in E[p]]
        for r in range(n):
            if r != p and M[r][p] != 0:
                f = M[r][p]
                M[r] = [a - f * b for a, b in zip(M[r], M[p])]
                E[r] = [a - f * b for a, b in zip(E[r], E[p])]
    return E


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_alg1_equals_alg2_exactly_ilu0(orc, seed):
    from test_oracle_rational import dense_to_csr, small_unsym
    n = 8
    A = small_unsym(n, seed)
    Ac = dense_to_csr(orc, A)
    Minv = _ilu_minv_exact(Ac)
    rng = np.random.default_rng(20 + seed)
    xs = rng.integers(-5, 6, n).astype(float)
    bf = R.fvec(A @ xs)
    Af = R.fmat(A)
    x0 = [F(0)] * n
    c = R.bicgstab(Af, Minv, bf, x0, 4)
    p = R.pbicgstab(Af, Minv, bf, x0, 4)
    for i in range(min(len(c), len(p)) - 1):
        assert c[i + 1]["x"] == p[i + 1]["x"]
        assert c[i + 1]["r"] == p[i + 1]["r"]
    # the fp64 oracle follows the exact iterates
    res = orc.pbicgstab(Ac, A @ xs, tol=0.0, maxit=4, bench=True, block="ilu0", want_trace=True)
    for i in range(3):
        xe = np.array([float(v) for v in p[i + 1]["x"]])
        assert np.linalg.norm(res.trace[i + 1, 0] - xe) <= 1e-11 * np.linalg.norm(xe)


def test_pcg_equals_pipecg_exactly_icc0(orc):
    n = 7
    D = np.diag([6.0] * n) + np.diag([-1.0] * (n - 1), 1) + np.diag([-1.0] * (n - 1), -1)
    D[0, 3] = D[3, 0] = -2.0
    D[2, 6] = D[6, 2] = -1.0
    Ac = orc.csr(*_dense_to_csr_arrays(D))
    Minv = _ilu_minv_exact(Ac)
    xs = np.arange(1, n + 1, dtype=float) - 3.0
    bf = R.fvec(D @ xs)
    x0 = [F(0)] * n
    a = R.pcg(R.fmat(D), Minv, bf, x0, 4)
    b = R.pipecg(R.fmat(D), Minv, bf, x0, 4)
    for i in range(min(len(a), len(b)) - 1):
        assert a[i + 1]["x"] == b[i + 1]["x"]


def test_ilu_solutions_dense_lu_and_acceleration(orc):
    P = problems.csr_band(2048, nnz_row=27, band=64, seed=5)
    for A in (orc.stencil_csr(2, 16, 16, 1, problems.cfg2_coef()),
              orc.stencil_csr(3, 8, 7, 6, problems.cfg34_coef()),
              orc.csr(P.row_ptr, P.col, P.val)):
        xs = problems.x_star(A.n, 1)
        bb = orc.spmv(A, xs)
        xl = np.linalg.solve(A.dense(), bb)
        for solve in (orc.pbicgstab, orc.bicgstab):
            r = solve(A, bb, tol=1e-13, maxit=600, block="ilu0")
            assert r.outcome == "converged"
            assert np.linalg.norm(r.x - xl) <= 1e-8 * np.linalg.norm(xl)
    st = problems.configs()["cfg1"].stencil
    A = orc.stencil_csr(2, st.nx, st.ny, 1, st.coef)
    xs = problems.x_star(A.n, 0)
    b = orc.spmv(A, xs)
    for solve in (orc.pbicgstab, orc.bicgstab, orc.pipecg):
        jac = solve(A, b, tol=1e-10, maxit=2000).iters
        icc = solve(A, b, tol=1e-10, maxit=2000, block="icc0").iters
        assert icc < 0.6 * jac, (solve.__name__, icc, jac)


def test_block_diagonal_reading(orc):
    """Multi-rank reading of A34: M = ILU(0) of A's block-diagonal part over the row
    blocks.  One block is plain ILU(0); with tridiagonal blocks (a 1D operator) the
    blocks are factorised exactly, so M^{-1} is the block-diagonal solve."""
    A = orc.stencil_csr(2, 12, 10, 1, problems.cfg2_coef())
    u = problems.x_star(A.n, 4)
    one = orc.block_diagonal(A, [0, A.n])
    with orc.prec_matrix(one):
        v1 = orc.prec_apply(A, u, "ilu0")
    assert np.array_equal(v1, orc.prec_apply(A, u, "ilu0"))
    T = orc.stencil_csr(2, 30, 1, 1, problems.cfg2_coef())  # tridiagonal
    ut = problems.x_star(T.n, 5)
    cuts = [0, 11, 19, 30]
    Bd = orc.block_diagonal(T, cuts)
    with orc.prec_matrix(Bd):
        vb = orc.prec_apply(T, ut, "ilu0")
    D = T.dense()
    ref = np.concatenate([np.linalg.solve(D[a:b, a:b], ut[a:b]) for a, b in zip(cuts, cuts[1:])])
    assert np.linalg.norm(vb - ref) <= 1e-13 * np.linalg.norm(ref)
