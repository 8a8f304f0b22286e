"""Exact breakdowns (reading A9) pinned in rationals, on small integer systems whose
scalars are exact in fp64 (power-of-two diagonals, small integers):

* BD_ALPHA0: (r^0, w_0) = 0, so alpha_0 = rho_0 / 0 (Alg. 2 line 3);
* BD_DEN: the alpha denominator (d_w + beta d_s) - (beta omega) d_z of line 26
   is exactly 0 at the end of iteration 0 while ||r_1|| > 0 -- a true
  breakdown, not a converged run.

The exact-rational replay of Alg. 2 (oracle/rational.py) meets the zero, and the
fp64 oracle reports BREAKDOWN at the same iteration with the iterate x and history
of the last completed step.  tests/test_gpu_breakdown.py holds the GPU to the same.
(The systems were found by a random search over such matrices with the oracle.)
"""
from fractions import Fraction as F

import numpy as np
import pytest

from oracle import rational as R

BD_ALPHA0 = (np.array([[1.0, -4.0], [0.0, 2.0]]), np.array([3.0, 0.5]))
BD_DEN = (np.array([[2.0, 1.0, 0.0], [-2.0, -2.0, 0.0], [0.0, -1.0, -1.0]]),
          np.array([-1.0, 1.0, 0.0]))


def dense_csr(orc, D):
    n = D.shape[0]
    rp, ci, va = [0], [], []
    for i in range(n):
        for j in range(n):
            if D[i, j] != 0.0 or i == j:
                ci.append(j)
                va.append(D[i, j])
        rp.append(len(ci))
    return orc.csr(np.array(rp), np.array(ci), np.array(va))


def test_alpha0_denominator_zero(orc):
    D, xs = BD_ALPHA0
    b = D @ xs
    dinv = [F(1) / F(D[i, i]) for i in range(2)]
    r0 = R.fvec(b)
    k0 = R.prec(dinv, r0)
    w0 = R.matvec(R.fmat(D), k0)
    assert R.dot(r0, w0) == 0 and R.dot(r0, r0) != 0  # alpha_0 = rho_0 / 0
    for solve in (orc.pbicgstab, orc.bicgstab):
        res = solve(dense_csr(orc, D), b, tol=0.0, maxit=5, bench=True)
        assert res.outcome == "breakdown" and res.iters == 0
        assert np.array_equal(res.x, np.zeros(2))


def test_alpha_denominator_zero_mid_run(orc):
    D, xs = BD_DEN
    b = D @ xs
    dinv = [F(1) / F(D[i, i]) for i in range(3)]
    with pytest.raises(ZeroDivisionError):  # line 26 divides by an exact zero
        R.pbicgstab(R.fmat(D), dinv, R.fvec(b), [F(0)] * 3, 2)
    # x_1, r_1 of the exact iteration (Alg. 1 generates the same iterates)
    st = R.bicgstab(R.fmat(D), dinv, R.fvec(b), [F(0)] * 3, 1)
    x1 = np.array([float(v) for v in st[1]["x"]])
    r1 = st[1]["r"]
    assert any(v != 0 for v in r1)  # not converged: a true breakdown
    res = orc.pbicgstab(dense_csr(orc, D), b, tol=0.0, maxit=5, bench=True)
    assert res.outcome == "breakdown" and res.iters == 1
    assert np.allclose(res.x, x1, rtol=1e-15, atol=0.0)  # the last iterate is returned
    assert res.rnorm[1] == pytest.approx(R.norm(r1), rel=1e-14)
