"""Solver-level pins of the fp64 oracle (no GPU).

* dense-LU brute force on small stencil / CSR systems (converged x);
* fp64 Alg. 2 vs fp64 Alg. 1 agreement over the first iterations (two different
  algorithms equal in exact arithmetic);
* residual replacement: the gap is exactly 0 right after a replacement
  (eq:rr P:598-601 with eq:res_gap P:113), replacing every iteration keeps the
  gap at rounding level;
* the paper's qualitative claims on the TP1-shaped cfg1;
* degenerate cases: identity system, zero rhs, maxit = 0, lucky breakdown.
"""
import numpy as np
import pytest

from paper_1809_01948_b200 import problems

EPS = 2.0 ** -53


def _stencil(orc, dim, nx, ny, nz, coef, seed=0):
    A = orc.stencil_csr(dim, nx, ny, nz, coef)
    xs = problems.x_star(A.n, seed)
    return A, xs, orc.spmv(A, xs)


@pytest.mark.parametrize("case", ["cd2d", "cd3d", "poisson2d", "csr"])
@pytest.mark.parametrize("solver", ["pbicgstab", "bicgstab", "pbicgstab_rr"])
def test_converged_solution_matches_dense_lu(orc, case, solver):
    if case == "cd2d":
        A, xs, b = _stencil(orc, 2, 16, 16, 1, problems.cfg2_coef())
    elif case == "cd3d":
        A, xs, b = _stencil(orc, 3, 7, 6, 5, problems.cfg34_coef())
    elif case == "poisson2d":
        A, xs, b = _stencil(orc, 2, 20, 20, 1, problems.poisson2d_coef())
    else:
        P = problems.csr_band(600, nnz_row=27, band=64, seed=1)
        A = orc.csr(P.row_ptr, P.col, P.val)
        xs = problems.x_star(A.n, 0)
        b = orc.spmv(A, xs)
    xlu = np.linalg.solve(A.dense(), b)
    if solver == "pbicgstab":
        res = orc.pbicgstab(A, b, tol=1e-13, maxit=2000)
    elif solver == "pbicgstab_rr":
        res = orc.pbicgstab(A, b, tol=1e-13, maxit=2000, rr_period=10)
    else:
        res = orc.bicgstab(A, b, tol=1e-13, maxit=2000)
    assert res.outcome == "converged"
    assert np.linalg.norm(res.x - xlu) <= 1e-8 * np.linalg.norm(xlu)
    # stopping rule (A7): first iteration with ||r_i|| <= tol ||b||
    nb = np.sqrt(orc.dot2(b, b))
    assert res.rnorm[res.iters] <= 1e-13 * nb
    assert np.all(res.rnorm[:res.iters] > 1e-13 * nb)


@pytest.mark.parametrize("solver", ["pcg", "pipecg"])
def test_cg_family_dense_lu(orc, solver):
    A, xs, b = _stencil(orc, 2, 20, 20, 1, problems.poisson2d_coef())
    res = getattr(orc, solver)(A, b, tol=1e-12, maxit=1000)
    assert res.outcome == "converged"
    xlu = np.linalg.solve(A.dense(), b)
    assert np.linalg.norm(res.x - xlu) <= 1e-8 * np.linalg.norm(xlu)


@pytest.mark.parametrize("case", ["cd2d", "poisson2d", "cd3d"])
def test_fp64_alg2_tracks_alg1(orc, case):
    """Alg. 1 and Alg. 2 are identical in exact arithmetic; in fp64 they
    agree to rounding over the first iterations."""
    if case == "cd2d":
        A, xs, b = _stencil(orc, 2, 32, 32, 1, problems.cfg2_coef())
    elif case == "cd3d":
        A, xs, b = _stencil(orc, 3, 10, 10, 10, problems.cfg34_coef())
    else:
        A, xs, b = _stencil(orc, 2, 30, 30, 1, problems.poisson2d_coef())
    p = orc.pbicgstab(A, b, maxit=10, bench=True)
    c = orc.bicgstab(A, b, maxit=10, bench=True)
    assert np.all(np.abs(p.rnorm - c.rnorm) <= 1e-10 * c.rnorm)


def test_replacement_zeroes_gap(orc):
    A, xs, b = _stencil(orc, 2, 40, 40, 1, problems.cfg2_coef())
    P = 7
    res = orc.pbicgstab(A, b, tol=0.0, maxit=60, rr_period=P, bench=True)
    rr_its = [i + 1 for i in range(res.iters) if (i + 1) % P == 0
              and res.rnorm[i] >= np.sqrt(EPS) * res.rnorm[0]]
    assert len(rr_its) >= 3
    for it in rr_its:
        assert res.gap[it] == 0.0, it
    assert res.gap[0] == 0.0
    # replacing every iteration keeps the gap at rounding level
    res1 = orc.pbicgstab(A, b, tol=0.0, maxit=40, rr_period=1, bench=True)
    nb = np.sqrt(orc.dot2(b, b))
    assert np.max(res1.gap) <= 100 * np.sqrt(A.n) * EPS * nb


def test_replacement_stops_below_sqrt_eps(orc):
    """replacements stop for good once ||r_i|| < sqrt(eps) ||r_0|| (A12)."""
    A, xs, b = _stencil(orc, 2, 20, 20, 1, problems.cfg2_coef())
    res = orc.pbicgstab(A, b, tol=0.0, maxit=200, rr_period=5, bench=True)
    h = res.rnorm
    first = int(np.argmax(h < np.sqrt(EPS) * h[0]))
    assert first > 0
    # after the latch no replacement: gap stays nonzero at later multiples of 5
    later = [it for it in range(first + 5, res.iters + 1) if it % 5 == 0]
    assert later and all(res.gap[it] != 0.0 for it in later)


def test_cfg1_qualitative_paper_claims(orc):
    """cfg1 (TP1-shaped Poisson 100^2, Jacobi, 500 its):
    classic BiCGStab only accumulates rounding errors;
    the p-BiCGStab gap grows orders of magnitude above it;
    periodic replacement restores classic-level accuracy."""
    cfg = problems.configs()["cfg1"]
    st = cfg.stencil
    A, xs, b = _stencil(orc, st.dim, st.nx, st.ny, st.nz, st.coef)
    nb = np.sqrt(orc.dot2(b, b))
    c = orc.bicgstab(A, b, maxit=500, bench=True)
    p = orc.pbicgstab(A, b, maxit=500, bench=True)
    prr = orc.pbicgstab(A, b, maxit=500, rr_period=50, bench=True)
    gc, gp, grr = c.gap[-1] / nb, p.gap[-1] / nb, prr.gap[-1] / nb
    assert gc < 1e-13
    assert gp > 100 * gc
    assert grr < 1e-12
    err = lambda r: np.linalg.norm(r.x - xs) / np.linalg.norm(xs)
    assert err(prr) < 1e-2 * err(p)


def test_replacement_can_delay_convergence(orc):
    """explicitly recomputed vectors are not orthogonal to the Krylov
    basis built so far, so frequent replacement delays convergence."""
    A, xs, b = _stencil(orc, 2, 128, 128, 1, problems.cfg2_coef())
    its = {rr: orc.pbicgstab(A, b, tol=1e-10, maxit=5000, rr_period=rr, gap=False).iters
           for rr in (0, 50, 20)}
    assert its[0] < its[50] < its[20]


def test_identity_system_one_iteration(orc):
    """A = I: r1 = 0 after one iteration (y0 = 0 => omega := 0 guard, A9)."""
    n = 10
    A = orc.csr(np.arange(n + 1), np.arange(n), np.ones(n))
    b = problems.x_star(n, 4)
    res = orc.pbicgstab(A, b, tol=1e-14, maxit=5)
    assert res.outcome == "converged" and res.iters == 1
    assert np.array_equal(res.x, b)


def test_degenerate_inputs(orc):
    A, xs, b = _stencil(orc, 2, 8, 8, 1, problems.cfg2_coef())
    z = np.zeros(A.n)
    r = orc.pbicgstab(A, z, tol=1e-10, maxit=10)
    assert r.outcome == "converged" and r.iters == 0 and np.all(r.x == 0)
    r = orc.pbicgstab(A, b, tol=1e-10, maxit=0)
    assert r.outcome == "maxit" and r.iters == 0 and r.rnorm.shape == (1,)
    # x0 = exact solution of a system with exact integer data => r0 = 0
    xi = np.arange(A.n, dtype=float)
    bi = orc.spmv(A, xi)
    r = orc.pbicgstab(A, bi, x0=xi, tol=0.0, maxit=3)
    assert r.rnorm[0] == 0.0


def test_oracle_deterministic(orc):
    A, xs, b = _stencil(orc, 2, 30, 30, 1, problems.cfg2_coef())
    r1 = orc.pbicgstab(A, b, maxit=50, rr_period=10, bench=True)
    r2 = orc.pbicgstab(A, b, maxit=50, rr_period=10, bench=True)
    assert np.array_equal(r1.x, r2.x) and np.array_equal(r1.rnorm, r2.rnorm)
    assert np.array_equal(r1.gap, r2.gap, equal_nan=True)
