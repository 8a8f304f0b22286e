"""Per-term pins of the oracle's run-time gap bound f^r (eq:DDr_bound, P:613-616;
SURVEY 8(f) NEXT-1), answering "a dropped term or a changed coefficient passes the
dominance pins".

The bound the oracle propagates is rebuilt here from two independent sources and
compared with the oracle's bound trace (f_i, Dw_i, Ds_i, Dz_i) to 1e-12:

1. LOCAL error bounds (eq:errbounds1-4) are DERIVED, not re-typed: each
   recurrence of Alg. 2 (eq:auxrec) is written as the expression tree the
   oracle evaluates (left to right with the printed brackets), and the
   standard rounding model gives each leaf L with scalar coefficient kappa the term
   c * |kappa| * ||L|| with c = the number of rounded operations on its path to the
   root; a leaf that is itself an explicitly computed product fl(Op v) (m, n, t, v:
   eq:auxvars2) adds |kappa| (mu_Op sqrt(N) ||Op|| ||v|| + ||Op|| * (the same for v))
   -- the convention of reading A21.  The derivation reproduces every coefficient
   the paper prints (asserted below against a table of the printed ones), so a
   mutant coefficient or a dropped term in oracle.c no longer matches.
2. PROPAGATION is the paper's closed form: eq:DDr / eq:DDs / eq:DDw / eq:DDz
    as explicit sums with explicit products of |beta_k| (O(i^2)), with
   eq:DDs's local term A delta^g - delta^s (reading A20), instead of the oracle's
   one-step recursion.

scripts/mutate_oracle_bounds.py applies one mutation per term / coefficient of
oracle.c's bound code and checks that this file fails for every one of them.
"""
import math

import numpy as np
import pytest

from paper_1809_01948_b200 import problems

EPS = 2.0 ** -53
NAMES = ["x", "r", "k", "w", "m", "t", "g", "s", "l", "z", "q", "u", "y", "n", "v"]

# --- expression trees of eq:auxrec (leaves: vectors of iteration i; 'p' suffix =
# the previous iteration's vector; scalars: a = alpha_i, b = beta_i, w = omega_i,
# wp = omega_{i-1})
V = lambda n: ("v", n)
ADD = lambda a, b: ("add", a, b)
SUB = lambda a, b: ("sub", a, b)
MUL = lambda s, e: ("mul", s, e)
TREES = {
    "g": ADD(V("k"), MUL("b", SUB(V("gp"), MUL("wp", V("lp"))))),
    "s": ADD(V("w"), MUL("b", SUB(V("sp"), MUL("wp", V("zp"))))),
    "l": ADD(V("m"), MUL("b", SUB(V("lp"), MUL("wp", V("np"))))),
    "z": ADD(V("t"), MUL("b", SUB(V("zp"), MUL("wp", V("vp"))))),
    "q": SUB(V("r"), MUL("a", V("s"))),
    "u": SUB(V("k"), MUL("a", V("l"))),
    "y": SUB(V("w"), MUL("a", V("z"))),
    "x": ADD(ADD(V("x"), MUL("a", V("g"))), MUL("w", V("u"))),
    "r": SUB(V("q"), MUL("w", V("y"))),
    "k": SUB(V("u"), MUL("w", SUB(V("m"), MUL("a", V("n"))))),
    "wn": SUB(V("y"), MUL("w", SUB(V("t"), MUL("a", V("v"))))),
}
# explicitly computed products (eq:auxvars2): leaf -> (operator, operand)
PRODUCTS = {"m": ("Minv", "w"), "n": ("Minv", "z"), "np": ("Minv", "zp"),
            "t": ("A", "m"), "v": ("A", "n"), "vp": ("A", "np")}


def leaf_terms(e, scal=(), depth=0):
    """[(leaf, scalars on its path, rounded operations above it)]"""
    if e[0] == "v":
        return [(e[1], scal, depth)]
    if e[0] == "mul":
        return leaf_terms(e[2], scal + (e[1],), depth + 1)
    return leaf_terms(e[1], scal, depth + 1) + leaf_terms(e[2], scal, depth + 1)


def test_derived_coefficients_are_the_printed_ones():
    """The rounding-count derivation reproduces eq:errbounds1-4."""
    printed = {  # (leaf, |scalars|) -> coefficient, as printed in the paper
        "g": {("k", ()): 1, ("gp", ("b",)): 3, ("lp", ("b", "wp")): 4},
        "s": {("w", ()): 1, ("sp", ("b",)): 3, ("zp", ("b", "wp")): 4},
        "l": {("m", ()): 1, ("lp", ("b",)): 3, ("np", ("b", "wp")): 4},
        "z": {("t", ()): 1, ("zp", ("b",)): 3, ("vp", ("b", "wp")): 4},
        "x": {("x", ()): 2, ("g", ("a",)): 3, ("u", ("w",)): 2},
        "r": {("q", ()): 1, ("y", ("w",)): 2},
        "k": {("u", ()): 1, ("m", ("w",)): 3, ("n", ("w", "a")): 4},
        "wn": {("y", ()): 1, ("t", ("w",)): 3, ("v", ("w", "a")): 4},
        "q": {("r", ()): 1, ("s", ("a",)): 2},
        "u": {("k", ()): 1, ("l", ("a",)): 2},
        "y": {("w", ()): 1, ("z", ("a",)): 2},
    }
    for key, tree in TREES.items():
        got = {(leaf, s): c for leaf, s, c in leaf_terms(tree)}
        assert got == printed[key], key


def local_bound(key, N, sc, consts):
    """e^key / eps from the derivation: N = norms by name, sc = scalar values."""
    nA, muN, mutN = consts

    def prod_err(leaf):
        """error of an explicitly computed product, measured against the exact
        operator applied to the computed operand (reading A21)"""
        if leaf not in PRODUCTS:
            return 0.0
        op, inner = PRODUCTS[leaf]
        if op == "Minv":  # mu~ sqrt(N) ||M^-1|| ||inner||  (mutN carries ||M^-1||)
            return mutN * N[inner]
        return muN * nA * N[inner] + nA * prod_err(inner)

    tot = 0.0
    for leaf, scal, c in leaf_terms(TREES[key]):
        kap = math.prod(abs(sc[s]) for s in scal)
        tot += c * kap * N[leaf] + kap * prod_err(leaf)
    return tot


def closed_form_bounds(res, consts, nb, nx0, nk0):
    """f_i, Dw_i, Ds_i, Dz_i from eq:DDr/DDs/DDw/DDz as explicit sums."""
    nA, muN, mutN = consts
    T = res.trace
    S = res.scalars
    iters = res.iters
    idx = {n: j for j, n in enumerate(NAMES)}

    def norms(i):
        N = {n: float(np.linalg.norm(T[i, idx[n]])) for n in NAMES}
        for n in ("g", "s", "l", "z", "n", "v"):
            N[n + "p"] = float(np.linalg.norm(T[i - 1, idx[n]])) if i > 0 else 0.0
        return N

    eg, es, el, ez, ek, ew, eu, ey, ex, er, eq = ([] for _ in range(11))
    al, be, om = S[:iters, 0], S[:iters, 1], S[:iters, 2]
    for i in range(iters):
        N = norms(i)
        N["wn"] = 0.0
        sc = {"a": al[i], "b": be[i], "w": om[i], "wp": om[i - 1] if i > 0 else 0.0}
        for lst, key in ((eg, "g"), (es, "s"), (el, "l"), (ez, "z"), (ek, "k"), (ew, "wn"),
                         (eu, "u"), (ey, "y"), (ex, "x"), (er, "r"), (eq, "q")):
            lst.append(local_bound(key, N, sc, consts) * EPS)
    f0 = ((muN + 1.0) * nA * nx0 + nb) * EPS
    Dw0 = muN * nA * nk0 * EPS

    def P(lo, hi):  # prod_{k=lo..hi} |beta_k|
        return math.prod(abs(be[k]) for k in range(lo, hi + 1))

    Dz = [sum(P(j + 1, i) * (nA * el[j] + ez[j]) for j in range(i + 1)) for i in range(iters)]
    Dw = [Dw0 + sum(abs(al[j]) * Dz[j] + nA * ek[j] + ew[j] + nA * eu[j] + ey[j]
                    for j in range(i)) for i in range(iters + 1)]
    Ds = [sum(P(j + 1, i) * (Dw[j] + nA * eg[j] + es[j]) for j in range(i + 1))
          + sum(P(j + 1, i) * abs(be[j] * (om[j - 1] if j > 0 else 0.0)) * Dz[j - 1]
                for j in range(1, i + 1)) for i in range(iters)]
    f = [f0 + sum(abs(al[j]) * Ds[j] + abs(om[j]) * Dw[j] + abs(om[j] * al[j]) * Dz[j]
                  + nA * ex[j] + er[j] + abs(om[j]) * nA * eu[j] + eq[j] + abs(om[j]) * ey[j]
                  for j in range(i)) for i in range(iters + 1)]
    return f, Dw, Ds, Dz


CASES = [(2, 6, 5, 1, "cd2", 12), (3, 3, 3, 4, "cd3", 12), (2, 7, 7, 1, "poisson", 14)]


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("block", [1, 2])
def test_bound_trace_equals_derived_closed_form(orc, case, block):
    dim, nx, ny, nz, kind, iters = case
    coef = {"cd2": problems.cfg2_coef(), "cd3": problems.cfg34_coef(),
            "poisson": problems.poisson2d_coef()}[kind]
    A = orc.stencil_csr(dim, nx, ny, nz, coef)
    if A.n % block:
        pytest.skip("block size")
    xs = problems.x_star(A.n, seed=3)
    b = orc.spmv(A, xs)
    res = orc.pbicgstab(A, b, tol=0.0, maxit=iters, bench=True, want_trace=True,
                        want_scalars=True, auto_rr=True, block=block)
    # compare up to the first replacement (after it the recomputation restarts the
    # bounds: reading A31, pinned by test_oracle_autorr.py)
    last = min(res.iters, (res.rr_iters[0] if res.rr_iters else res.iters))
    mu = int(np.max(np.diff(A.rp)))
    nA = orc.anorm_bound(A)
    D = A.dense()
    if block == 1:
        minv = float(np.max(np.abs(1.0 / np.diag(D))))
    else:  # max over blocks of sqrt(||B^-1||_1 ||B^-1||_inf) (reading A33)
        minv = 0.0
        for k0 in range(0, A.n, block):
            Bi = np.linalg.inv(D[k0:k0 + block, k0:k0 + block])
            minv = max(minv, math.sqrt(np.abs(Bi).sum(0).max() * np.abs(Bi).sum(1).max()))
    consts = (nA, mu * math.sqrt(A.n), block * math.sqrt(A.n) * minv)
    nb = float(np.linalg.norm(b))
    T = res.trace
    nx0 = float(np.linalg.norm(T[0, 0]))
    nk0 = float(np.linalg.norm(T[0, 2]))
    f, Dw, Ds, Dz = closed_form_bounds(res, consts, nb, nx0, nk0)
    B = res.bounds
    for i in range(last + 1):
        assert B[i, 0] == pytest.approx(f[i], rel=1e-11, abs=0.0), ("f", i)
        assert B[i, 1] == pytest.approx(Dw[i], rel=1e-11, abs=0.0), ("Dw", i)
    for i in range(last):
        assert B[i, 2] == pytest.approx(Ds[i], rel=1e-11, abs=0.0), ("Ds", i)
        assert B[i, 3] == pytest.approx(Dz[i], rel=1e-11, abs=0.0), ("Dz", i)
