"""Exact-arithmetic pins (reading: P:4, "identical series of iterates";
eq:auxvars P:153-157; local-error bounds eq:errbounds1-4 P:226-251; gap
recurrences eq:Dr-eq:Dz P:264-293).

1. The rational transcriptions of Alg. 1 and Alg. 2 produce identical iterates
   and Alg. 2's recursively computed vectors equal their definitions exactly.
2. The fp64 C oracle follows those exact iterates to rounding level.
3. Every local rounding error of the C oracle's fp64 run, taken exactly in
   rationals, respects the paper's printed bound -- a dropped term, wrong sign
   or transposed operand in any recurrence of oracle.c violates it.
4. The gap recurrences derived in the paper hold exactly for that fp64 run.
"""
from fractions import Fraction as F

import numpy as np
import pytest

from oracle import rational as R
from paper_1809_01948_b200 import problems

EPS = 2.0 ** -53


def small_unsym(n, seed):
    """Random unsymmetric, strictly diagonally dominant integer matrix."""
    rng = np.random.default_rng(seed)
    A = rng.integers(-3, 4, (n, n)).astype(float)
    np.fill_diagonal(A, 0)
    np.fill_diagonal(A, np.abs(A).sum(1) + rng.integers(1, 4, n))
    return A


def dense_to_csr(orc, A):
    rp, ci, va = [0], [], []
    for i in range(A.shape[0]):
        nz = np.nonzero(A[i])[0]
        ci += list(nz)
        va += list(A[i, nz])
        rp.append(len(ci))
    return orc.csr(rp, ci, va)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_alg1_equals_alg2_exactly(seed):
    n = 7
    A = small_unsym(n, seed)
    rng = np.random.default_rng(10 + seed)
    xs = rng.integers(-5, 6, n)
    Af = R.fmat(A)
    dinv = [F(1) / Af[i][i] for i in range(n)]  # Jacobi in exact arithmetic
    b = R.matvec(Af, R.fvec(xs))
    x0 = [F(0)] * n
    c = R.bicgstab(Af, dinv, b, x0, 4)
    p = R.pbicgstab(Af, dinv, b, x0, 4)
    for i in range(min(len(c), len(p))):
        assert c[i]["x"] == p[i]["x"], f"x differs at {i}"
        assert c[i]["r"] == p[i]["r"], f"r differs at {i}"
        if "alpha" in c[i] and "alpha" in p[i]:
            assert c[i]["alpha"] == p[i]["alpha"]
            assert c[i]["omega"] == p[i]["omega"]
        if "beta" in c[i] and i + 1 < len(p) and "beta" in p[i + 1]:
            assert c[i]["beta"] == p[i + 1]["beta"]  # index shift of beta
    # eq:auxvars hold exactly for the recursive vectors
    for st in p[:-1]:
        assert st["k"] == R.prec(dinv, st["r"])
        assert st["w"] == R.matvec(Af, st["k"])
        assert st["m"] == R.prec(dinv, st["w"])
        assert st["t"] == R.matvec(Af, st["m"])
        assert st["s"] == R.matvec(Af, st["g"])
        assert st["l"] == R.prec(dinv, st["s"])
        assert st["z"] == R.matvec(Af, st["l"])
        assert st["u"] == R.prec(dinv, st["q"])
        assert st["y"] == R.matvec(Af, st["u"])
        assert st["r"] == R.sub(b, R.matvec(Af, st["x"]))
        # g_i = M^-1 p_i with p_i the classic search direction
    for i in range(min(len(c), len(p)) - 1):
        if "p" in c[i] and "g" in p[i]:
            assert p[i]["g"] == R.prec(dinv, c[i]["p"])


@pytest.mark.parametrize("seed", [0, 1])
def test_pcg_equals_pipecg_exactly(seed):
    """The reconstructed p-CG (reading A19) is exactly PCG in rationals."""
    n = 6
    rng = np.random.default_rng(seed)
    B = rng.integers(-2, 3, (n, n)).astype(float)
    A = B @ B.T + n * np.eye(n)
    Af = R.fmat(A)
    dinv = [F(1) / Af[i][i] for i in range(n)]
    b = R.matvec(Af, R.fvec(rng.integers(-4, 5, n)))
    x0 = [F(0)] * n
    c = R.pcg(Af, dinv, b, x0, 4)
    p = R.pipecg(Af, dinv, b, x0, 4)
    for i in range(min(len(c), len(p))):
        assert c[i]["x"] == p[i]["x"]
        assert c[i]["r"] == p[i]["r"]
        if "alpha" in c[i] and "alpha" in p[i]:
            assert c[i]["alpha"] == p[i]["alpha"]


@pytest.mark.parametrize("k", [1, 2, 3])
def test_finite_termination(k):
    """r0 in a k-dimensional invariant subspace of A M^-1 => r_k = 0 exactly."""
    n = 6
    rng = np.random.default_rng(7)
    S = np.tril(rng.integers(-2, 3, (n, n)), -1) + np.eye(n)  # unit lower triangular
    Sinv = np.round(np.linalg.inv(S))
    assert np.array_equal(S @ Sinv, np.eye(n))
    D = np.diag([2.0, 3.0, 5.0, 7.0, 11.0, 13.0])
    A = S @ D @ Sinv
    Af = R.fmat(A)
    dinv = [F(1)] * n  # M = I
    xs = [F(0)] * n
    for j in range(k):
        xs = R.add(xs, R.fvec(S[:, j]))
    b = R.matvec(Af, xs)
    p = R.pbicgstab(Af, dinv, b, [F(0)] * n, k + 2)
    assert p[k]["r"] == [F(0)] * n
    assert p[k]["x"] == xs
    for i in range(k):
        assert p[i]["r"] != [F(0)] * n


@pytest.mark.parametrize("seed", [0, 3])
def test_c_oracle_follows_exact_iterates(orc, seed):
    n = 8
    A = small_unsym(n, seed)
    Ac = dense_to_csr(orc, A)
    rng = np.random.default_rng(20 + seed)
    xs = rng.integers(-5, 6, n).astype(float)
    b = A @ xs  # exact in fp64 (small integers)
    Af = R.fmat(A)
    dinv = [F(x) for x in orc.jacobi_dinv(Ac)]  # the oracle's dinv, exactly
    ex = R.pbicgstab(Af, dinv, R.fvec(b), [F(0)] * n, 4)
    res = orc.pbicgstab(Ac, b, tol=0.0, maxit=4, bench=True, want_trace=True, want_scalars=True)
    for i in range(len(ex) - 1):
        xe = np.array([float(v) for v in ex[i + 1]["x"]])
        xc = res.trace[i + 1, 0] if i + 1 < 4 else res.x
        assert np.linalg.norm(xc - xe) <= 1e-12 * np.linalg.norm(xe)
        assert res.scalars[i, 0] == pytest.approx(float(ex[i]["alpha"]), rel=1e-12)
        assert res.scalars[i, 2] == pytest.approx(float(ex[i]["omega"]), rel=1e-12)


def _trace_problem(orc):
    nx, ny = 6, 5
    coef = problems.cfg2_coef()
    Ac = orc.stencil_csr(2, nx, ny, 1, coef)
    xs = problems.x_star(Ac.n, seed=2)
    b = orc.spmv(Ac, xs)
    iters = 6
    res = orc.pbicgstab(Ac, b, tol=0.0, maxit=iters, bench=True, want_trace=True,
                        want_scalars=True)
    assert res.iters == iters
    return Ac, b, res, iters


def test_local_errors_within_paper_bounds(orc):
    """eq:errbounds1-4: every delta of the C oracle's fp64 run, taken
    exactly, is below its printed bound (readings A21, A25: mu~ = 1; M^-1 is
    diag(dinv) exactly)."""
    Ac, b, res, iters = _trace_problem(orc)
    n = Ac.n
    Ad = Ac.dense()
    Af = R.fmat(Ad)
    dinv_f = orc.jacobi_dinv(Ac)
    dinv = R.fvec(dinv_f)
    normA = np.linalg.norm(Ad, 2)
    normM = float(np.max(np.abs(dinv_f)))
    mu = int(np.max(np.diff(Ac.rp)))
    mut = 1
    sq = np.sqrt(n)
    T = res.trace
    names = {nm: j for j, nm in enumerate(["x", "r", "k", "w", "m", "t", "g", "s", "l", "z",
                                            "q", "u", "y", "n", "v"])}

    def V(i, nm):
        return R.fvec(T[i, names[nm]])

    def nrm(v):
        return float(np.linalg.norm(np.array([float(a) for a in v])))

    def nf(v):  # float vector norm
        return float(np.linalg.norm(v))

    slack = 1.0 + 1e-6  # O(eps^2) terms are neglected by the paper
    worst = 0.0
    zero = [F(0)] * n
    for i in range(iters - 1):
        al, be, om, _ = [F(float(a)) for a in res.scalars[i, :4]]
        om_prev = F(float(res.scalars[i - 1, 2])) if i > 0 else F(0)
        k, w, m, t = V(i, "k"), V(i, "w"), V(i, "m"), V(i, "t")
        x, r = V(i, "x"), V(i, "r")
        g, s, l, z = V(i, "g"), V(i, "s"), V(i, "l"), V(i, "z")
        q, u, y, nn, v = V(i, "q"), V(i, "u"), V(i, "y"), V(i, "n"), V(i, "v")
        gp = V(i - 1, "g") if i > 0 else zero
        sp = V(i - 1, "s") if i > 0 else zero
        lp = V(i - 1, "l") if i > 0 else zero
        zp = V(i - 1, "z") if i > 0 else zero
        np_ = V(i - 1, "n") if i > 0 else zero
        vp = V(i - 1, "v") if i > 0 else zero
        x1, r1, k1, w1 = V(i + 1, "x"), V(i + 1, "r"), V(i + 1, "k"), V(i + 1, "w")
        Mw = R.prec(dinv, w)
        Mzp = R.prec(dinv, zp)
        Mz = R.prec(dinv, z)
        AMw = R.matvec(Af, Mw)
        AMzp = R.matvec(Af, Mzp)
        AMz = R.matvec(Af, Mz)
        fl = lambda a: float(a)
        checks = {
            # eq:errbounds1
            "g": (R.sub(g, R.add(k, R.scal(be, R.sub(gp, R.scal(om_prev, lp))))),
                  nrm(k) + 3 * abs(fl(be)) * nrm(gp) + 4 * abs(fl(be * om_prev)) * nrm(lp)),
            "x": (R.sub(x1, R.add(R.add(x, R.scal(al, g)), R.scal(om, u))),
                  2 * nrm(x) + 3 * abs(fl(al)) * nrm(g) + 2 * abs(fl(om)) * nrm(u)),
            "s": (R.sub(s, R.add(w, R.scal(be, R.sub(sp, R.scal(om_prev, zp))))),
                  nrm(w) + 3 * abs(fl(be)) * nrm(sp) + 4 * abs(fl(be * om_prev)) * nrm(zp)),
            "r": (R.sub(r1, R.sub(q, R.scal(om, y))), nrm(q) + 2 * abs(fl(om)) * nrm(y)),
            # eq:errbounds2 (l, z measured against exact M^-1 w, A M^-1 w: A21)
            "l": (R.sub(l, R.add(Mw, R.scal(be, R.sub(lp, R.scal(om_prev, Mzp))))),
                  nrm(m) + mut * sq * normM * nrm(w) + 3 * abs(fl(be)) * nrm(lp)
                  + 4 * abs(fl(be * om_prev)) * nrm(np_)
                  + mut * sq * normM * abs(fl(be * om_prev)) * nrm(zp)),
            "z": (R.sub(z, R.add(AMw, R.scal(be, R.sub(zp, R.scal(om_prev, AMzp))))),
                  nrm(t) + mu * sq * normA * nrm(m) + mut * sq * normA * normM * nrm(w)
                  + 3 * abs(fl(be)) * nrm(zp) + 4 * abs(fl(be * om_prev)) * nrm(vp)
                  + mu * sq * normA * abs(fl(be * om_prev)) * nrm(np_)
                  + mut * sq * normA * normM * abs(fl(be * om_prev)) * nrm(zp)),
            # eq:errbounds3
            "k": (R.sub(k1, R.sub(u, R.scal(om, R.sub(Mw, R.scal(al, Mz))))),
                  nrm(u) + 3 * abs(fl(om)) * nrm(m) + mut * sq * normM * abs(fl(om)) * nrm(w)
                  + 4 * abs(fl(om * al)) * nrm(nn) + mut * sq * normM * abs(fl(om * al)) * nrm(z)),
            "w": (R.sub(w1, R.sub(y, R.scal(om, R.sub(AMw, R.scal(al, AMz))))),
                  nrm(y) + 3 * abs(fl(om)) * nrm(t) + mu * sq * normA * abs(fl(om)) * nrm(m)
                  + mut * sq * normA * normM * abs(fl(om)) * nrm(w)
                  + 4 * abs(fl(om * al)) * nrm(v) + mu * sq * normA * abs(fl(om * al)) * nrm(nn)
                  + mut * sq * normA * normM * abs(fl(om * al)) * nrm(z)),
            # eq:errbounds4
            "q": (R.sub(q, R.sub(r, R.scal(al, s))), nrm(r) + 2 * abs(fl(al)) * nrm(s)),
            "u": (R.sub(u, R.sub(k, R.scal(al, l))), nrm(k) + 2 * abs(fl(al)) * nrm(l)),
            "y": (R.sub(y, R.sub(w, R.scal(al, z))), nrm(w) + 2 * abs(fl(al)) * nrm(z)),
        }
        for nm, (delta, bnd) in checks.items():
            d = nrm(delta)
            assert d <= bnd * EPS * slack, (nm, i, d, bnd * EPS)
            if bnd > 0:
                worst = max(worst, d / (bnd * EPS))
    assert worst > 0.0  # rounding did happen; the bound is not vacuous


def test_gap_recurrences_exact(orc):
    """eq:Dr, eq:Ds, eq:Dw, eq:Dz
    hold exactly for the oracle's fp64 iterates, with the deltas of eq:auxrec
    measured exactly (reading A21)."""
    Ac, b, res, iters = _trace_problem(orc)
    n = Ac.n
    Af = R.fmat(Ac.dense())
    dinv = R.fvec(orc.jacobi_dinv(Ac))
    bf = R.fvec(b)
    T = res.trace
    idx = {nm: j for j, nm in enumerate(["x", "r", "k", "w", "m", "t", "g", "s", "l", "z",
                                          "q", "u", "y", "n", "v"])}
    V = lambda i, nm: R.fvec(T[i, idx[nm]])
    A = lambda v: R.matvec(Af, v)
    zero = [F(0)] * n
    Ds_prev, Dz_prev = zero, zero
    for i in range(iters - 1):
        al, be, om, _ = [F(float(a)) for a in res.scalars[i, :4]]
        om_prev = F(float(res.scalars[i - 1, 2])) if i > 0 else F(0)
        x, r, k, w = V(i, "x"), V(i, "r"), V(i, "k"), V(i, "w")
        g, s, l, z, q, u, y = (V(i, nm) for nm in "g s l z q u y".split())
        gp = V(i - 1, "g") if i > 0 else zero
        sp = V(i - 1, "s") if i > 0 else zero
        lp = V(i - 1, "l") if i > 0 else zero
        zp = V(i - 1, "z") if i > 0 else zero
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
        d_z = R.sub(z, R.add(A(Mw), R.scal(be, R.sub(zp, R.scal(om_prev, A(Mzp))))))
        d_k = R.sub(k1, R.sub(u, R.scal(om, R.sub(Mw, R.scal(al, Mz)))))
        d_w = R.sub(w1, R.sub(y, R.scal(om, R.sub(A(Mw), R.scal(al, A(Mz))))))
        Dr = R.sub(R.sub(bf, A(x)), r)
        Dr1 = R.sub(R.sub(bf, A(x1)), r1)
        Ds = R.sub(A(g), s)
        Dw = R.sub(A(k), w)
        Dw1 = R.sub(A(k1), w1)
        Dz = R.sub(A(l), z)
        # eq:Dz
        assert Dz == R.sub(R.add(R.scal(be, Dz_prev), A(d_l)), d_z)
        # eq:Ds
        rhs = R.add(Dw, R.scal(be, Ds_prev))
        rhs = R.sub(rhs, R.scal(be * om_prev, Dz_prev))
        assert Ds == R.sub(R.add(rhs, A(d_g)), d_s)
        # eq:Dw
        rhs = R.sub(Dw, R.scal(al, Dz))
        rhs = R.add(rhs, A(d_k))
        rhs = R.sub(rhs, d_w)
        rhs = R.add(rhs, A(d_u))
        assert Dw1 == R.sub(rhs, d_y)
        # eq:Dr
        rhs = R.sub(Dr, R.scal(al, Ds))
        rhs = R.sub(rhs, R.scal(om, Dw))
        rhs = R.add(rhs, R.scal(om * al, Dz))
        rhs = R.sub(rhs, A(d_x))
        rhs = R.sub(rhs, d_r)
        rhs = R.sub(rhs, R.scal(om, A(d_u)))
        rhs = R.sub(rhs, d_q)
        rhs = R.add(rhs, R.scal(om, d_y))
        assert Dr1 == rhs
        Ds_prev, Dz_prev = Ds, Dz
