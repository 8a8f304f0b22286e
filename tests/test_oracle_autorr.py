"""Pins of the oracle's automated residual replacement (
P:609-623): the run-time gap bound f^r_i (eq:DDr_bound P:613-616) propagated over
the gap recurrences eq:Dr-eq:Dz with the local-error bounds
eq:errbounds1-4, and the criterion eq:criterion.

What pins it:
1. dominance -- the paper's defining property ||Delta^r_i|| <= f^r_i, and
   the same for the auxiliary bounds of Delta^s, Delta^w, Delta^z (eq:DsDwDz),
   against the EXACT gaps of the oracle's fp64 iterates (rational arithmetic);
2. structure -- f^r dominates the triangle-inequality recursion built from the
   exact local errors delta (a bound with a recurrence term dropped falls below
   it as soon as that term's exact contribution matters);
3. ||A|| bound -- sqrt(||A||_1 ||A||_inf) >= ||A||_2, and equals the closed form
   for the 2D Poisson stencil's interior-dominated norms;
4. the criterion's decisions -- exactly the crossings of f^r_i over tau ||r_i||,
   gap = 0 right after each replacement, few replacements, and an attainable
   accuracy far better than without replacement.
"""
from fractions import Fraction as F

import numpy as np
import pytest

from oracle import rational as R
from paper_1809_01948_b200 import problems

EPS = 2.0 ** -53
TAU = np.sqrt(EPS)
NAMES = ["x", "r", "k", "w", "m", "t", "g", "s", "l", "z", "q", "u", "y", "n", "v"]


def nrm(v):
    return float(np.sqrt(float(sum(a * a for a in v))))


def _run(orc, dim, nx, ny, nz, coef, iters, seed=2):
    A = orc.stencil_csr(dim, nx, ny, nz, coef)
    xs = problems.x_star(A.n, seed=seed)
    b = orc.spmv(A, xs)
    res = orc.pbicgstab(A, b, tol=0.0, maxit=iters, bench=True, want_trace=True,
                        want_scalars=True, auto_rr=True)
    assert res.iters == iters
    return A, b, res


@pytest.mark.parametrize("case", [(2, 6, 5, 1, "cd2", 14), (3, 3, 3, 4, "cd3", 14),
                                  (2, 7, 7, 1, "poisson", 16)])
def test_bounds_dominate_exact_gaps(orc, case):
    dim, nx, ny, nz, kind, iters = case
    coef = {"cd2": problems.cfg2_coef(), "cd3": problems.cfg34_coef(),
            "poisson": problems.poisson2d_coef()}[kind]
    A, b, res = _run(orc, dim, nx, ny, nz, coef, iters)
    Af = R.fmat(A.dense())
    bf = R.fvec(b)
    T = res.trace
    idx = {nm: j for j, nm in enumerate(NAMES)}
    V = lambda i, nm: R.fvec(T[i, idx[nm]])
    Ax = lambda v: R.matvec(Af, v)
    B = res.bounds
    rr = set(res.rr_iters)
    for i in range(iters):
        x, r, k, w = V(i, "x"), V(i, "r"), V(i, "k"), V(i, "w")
        Dr = nrm(R.sub(R.sub(bf, Ax(x)), r))
        Dw = nrm(R.sub(Ax(k), w))
        assert Dr <= B[i, 0], ("f^r", i, Dr, B[i, 0])
        assert Dw <= B[i, 1], ("Dw", i, Dw, B[i, 1])
        if i in rr:  # s_i, l_i, z_i were replaced after the trace was taken
            continue
        g, s, l, z = V(i, "g"), V(i, "s"), V(i, "l"), V(i, "z")
        assert nrm(R.sub(Ax(g), s)) <= B[i, 2], ("Ds", i)
        assert nrm(R.sub(Ax(l), z)) <= B[i, 3], ("Dz", i)
    assert np.all(B[1:, 0] > B[0, 0])  # the bound grows from its initial value


def test_bound_dominates_exact_delta_recursion(orc):
    """f^r_i >= the same triangle-inequality recursion driven by the EXACT local
    errors (eq:auxrec, measured as in reading A21) instead of their bounds."""
    A, b, res = _run(orc, 2, 6, 5, 1, problems.cfg2_coef(), 8)
    assert res.rr_iters == []  # first crossing is later: pure recursion
    n = A.n
    Af = R.fmat(A.dense())
    dinv = R.fvec(orc.jacobi_dinv(A))
    bf = R.fvec(b)
    T = res.trace
    idx = {nm: j for j, nm in enumerate(NAMES)}
    V = lambda i, nm: R.fvec(T[i, idx[nm]])
    Ax = lambda v: R.matvec(Af, v)
    zero = [F(0)] * n
    x0 = V(0, "x")
    f = nrm(R.sub(R.sub(bf, Ax(x0)), V(0, "r")))
    Dw = nrm(R.sub(Ax(V(0, "k")), V(0, "w")))
    Ds = Dz = 0.0
    for i in range(res.iters - 1):
        al, be, om, _ = [F(float(a)) for a in res.scalars[i, :4]]
        om_prev = F(float(res.scalars[i - 1, 2])) if i > 0 else F(0)
        x, r, k, w = V(i, "x"), V(i, "r"), V(i, "k"), V(i, "w")
        g, s, l, z, q, u, y = (V(i, nm) for nm in "g s l z q u y".split())
        gp, sp, lp, zp = ((V(i - 1, nm) if i > 0 else zero) for nm in "g s l z".split())
        x1, r1, k1, w1 = V(i + 1, "x"), V(i + 1, "r"), V(i + 1, "k"), V(i + 1, "w")
        Mw, Mz, Mzp = R.prec(dinv, w), R.prec(dinv, z), R.prec(dinv, zp)
        d_x = R.sub(x1, R.add(R.add(x, R.scal(al, g)), R.scal(om, u)))
        d_r = R.sub(r1, R.sub(q, R.scal(om, y)))
        d_q = R.sub(q, R.sub(r, R.scal(al, s)))
        d_u = R.sub(u, R.sub(k, R.scal(al, l)))
        d_y = R.sub(y, R.sub(w, R.scal(al, z)))
        d_g = R.sub(g, R.add(k, R.scal(be, R.sub(gp, R.scal(om_prev, lp)))))
        d_s = R.sub(s, R.add(w, R.scal(be, R.sub(sp, R.scal(om_prev, zp)))))
        d_l = R.sub(l, R.add(Mw, R.scal(be, R.sub(lp, R.scal(om_prev, Mzp)))))
        d_z = R.sub(z, R.add(Ax(Mw), R.scal(be, R.sub(zp, R.scal(om_prev, Ax(Mzp))))))
        d_k = R.sub(k1, R.sub(u, R.scal(om, R.sub(Mw, R.scal(al, Mz)))))
        d_w = R.sub(w1, R.sub(y, R.scal(om, R.sub(Ax(Mw), R.scal(al, Ax(Mz))))))
        ab, abw = abs(float(be)), abs(float(be * om_prev))
        aa, aw, awa = abs(float(al)), abs(float(om)), abs(float(om * al))
        Dz_n = ab * Dz + nrm(Ax(d_l)) + nrm(d_z)
        Ds_n = Dw + ab * Ds + abw * Dz + nrm(Ax(d_g)) + nrm(d_s)
        Dw_n = Dw + aa * Dz_n + nrm(Ax(d_k)) + nrm(d_w) + nrm(Ax(d_u)) + nrm(d_y)
        f_n = (f + aa * Ds_n + aw * Dw + awa * Dz_n + nrm(Ax(d_x)) + nrm(d_r)
               + aw * nrm(Ax(d_u)) + nrm(d_q) + aw * nrm(d_y))
        f, Dw, Ds, Dz = f_n, Dw_n, Ds_n, Dz_n
        B = res.bounds
        assert Dz <= B[i, 3] and Ds <= B[i, 2], i
        assert Dw <= B[i + 1, 1] and f <= B[i + 1, 0], i


def test_anorm_bound(orc):
    for dim, nx, ny, nz, coef in [(2, 9, 7, 1, problems.poisson2d_coef()),
                                  (2, 8, 11, 1, problems.cfg2_coef()),
                                  (3, 5, 4, 6, problems.cfg34_coef()),
                                  (3, 1, 2, 1, problems.cfg34_coef())]:
        A = orc.stencil_csr(dim, nx, ny, nz, coef)
        bnd = orc.anorm_bound(A)
        D = A.dense()
        assert bnd >= np.linalg.norm(D, 2) * (1 - 1e-14)
        assert bnd == pytest.approx(np.sqrt(np.abs(D).sum(0).max() * np.abs(D).sum(1).max()),
                                    rel=1e-15)
    # 2D Poisson with interior points: ||A||_1 = ||A||_inf = 4 + 4 = 8 exactly
    assert orc.anorm_bound(orc.stencil_csr(2, 9, 7, 1, problems.poisson2d_coef())) == 8.0


@pytest.mark.parametrize("case", [("cfg1", None), ("cd2", (2, 64, 64, 1)), ("cd3", (3, 20, 20, 20))])
def test_criterion_decisions_and_accuracy(orc, case):
    name, shape = case
    if name == "cfg1":
        st = problems.configs()["cfg1"].stencil
        dim, nx, ny, nz, coef = st.dim, st.nx, st.ny, st.nz, st.coef
    else:
        dim, nx, ny, nz = shape
        coef = problems.cfg2_coef() if name == "cd2" else problems.cfg34_coef()
    A = orc.stencil_csr(dim, nx, ny, nz, coef)
    xs = problems.x_star(A.n, 0)
    b = orc.spmv(A, xs)
    res = orc.pbicgstab(A, b, tol=0.0, maxit=400, bench=True, auto_rr=True)
    ref = orc.pbicgstab(A, b, tol=0.0, maxit=400, bench=True)
    f, h = res.bounds[:, 0], res.rnorm
    # the replacements are exactly the crossings of eq:criterion (decided at the
    # end of iteration j-1 for iteration j, j >= 1)
    cross = [j for j in range(1, res.iters) if f[j - 1] <= TAU * h[j - 1] and f[j] > TAU * h[j]]
    assert res.rr_iters == cross
    assert 1 <= len(res.rr_iters) <= 10  # "no excess replacements" (P:787 counts)
    for j in res.rr_iters:
        assert res.gap[j + 1] == 0.0  # r_{j+1} = b - A x_{j+1} recomputed exactly
    # the bound dominates the measured gap throughout
    assert np.all(res.gap <= f)
    # replacement improves the attainable accuracy by orders of magnitude
    assert res.gap[-1] < 1e-2 * ref.gap[-1]


def test_auto_rr_off_is_unchanged(orc):
    """The bound bookkeeping never touches the iterates: with no crossing the auto
    run equals the plain run bitwise."""
    A = orc.stencil_csr(2, 30, 20, 1, problems.cfg2_coef())
    xs = problems.x_star(A.n, 0)
    b = orc.spmv(A, xs)
    r1 = orc.pbicgstab(A, b, tol=0.0, maxit=6, bench=True, auto_rr=True)
    r0 = orc.pbicgstab(A, b, tol=0.0, maxit=6, bench=True)
    assert r1.rr_iters == []
    assert np.array_equal(r1.rnorm, r0.rnorm) and np.array_equal(r1.x, r0.x)


def test_bounds_dominate_exact_gaps_block_jacobi(orc):
    """Same dominance with the block-Jacobi preconditioner (mu~ = b, ||M^-1|| bound
    over the inverse blocks, reading A33)."""
    A = orc.stencil_csr(2, 8, 5, 1, problems.cfg2_coef())
    xs = problems.x_star(A.n, seed=2)
    b = orc.spmv(A, xs)
    res = orc.pbicgstab(A, b, tol=0.0, maxit=14, bench=True, want_trace=True, auto_rr=True,
                        block=4)
    Af = R.fmat(A.dense())
    bf = R.fvec(b)
    idx = {nm: j for j, nm in enumerate(NAMES)}
    V = lambda i, nm: R.fvec(res.trace[i, idx[nm]])
    for i in range(res.iters):
        x, r, k, w = V(i, "x"), V(i, "r"), V(i, "k"), V(i, "w")
        assert nrm(R.sub(R.sub(bf, R.matvec(Af, x)), r)) <= res.bounds[i, 0]
        assert nrm(R.sub(R.matvec(Af, k), w)) <= res.bounds[i, 1]
