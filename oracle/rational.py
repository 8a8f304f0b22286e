"""TEST INFRASTRUCTURE ONLY -- exact-rational replay (the oracle's own oracle).

Dense, tiny, pure-Python ``fractions.Fraction`` transcriptions of
  * classic preconditioned BiCGStab, Algorithm 1,
  * preconditioned pipelined BiCGStab, Algorithm 2,
  * preconditioned CG and the reconstructed pipelined CG (reading A19),
with M^{-1} = diag(dinv) applied exactly.  In exact arithmetic Alg. 1 and Alg. 2
"generate identical series of iterates" (P:4) and the auxiliary
vectors satisfy eq:auxvars exactly; tests/test_oracle_rational.py
checks both, which pins these transcriptions, and then pins the C oracle
(oracle.c) against them.

Also: the fp64 local-error analysis helpers (eq:auxrec P:203-215, bounds
eq:errbounds1-4 P:226-251, gap recurrences eq:Dr-eq:Dz P:264-293).
"""
from __future__ import annotations

from fractions import Fraction as F

Vec = list
Mat = list


def fvec(v) -> Vec:
    return [F(float(a)) if not isinstance(a, F) else a for a in v]


def fmat(A) -> Mat:
    return [fvec(row) for row in A]


def matvec(A: Mat, x: Vec) -> Vec:
    return [sum((a * b for a, b in zip(row, x)), F(0)) for row in A]


def dot(x: Vec, y: Vec) -> F:
    return sum((a * b for a, b in zip(x, y)), F(0))


def axpy(a: F, x: Vec, y: Vec) -> Vec:  # y + a x
    return [yi + a * xi for xi, yi in zip(x, y)]


def scal(a: F, x: Vec) -> Vec:
    return [a * xi for xi in x]


def sub(x: Vec, y: Vec) -> Vec:
    return [a - b for a, b in zip(x, y)]


def add(x: Vec, y: Vec) -> Vec:
    return [a + b for a, b in zip(x, y)]


def prec(dinv, v: Vec) -> Vec:
    """M^{-1} v: diag(dinv) (Jacobi, a vector) or a dense matrix M^{-1} (a list of
    rows, e.g. the block-diagonal inverse of block Jacobi, reading A33)."""
    if dinv and isinstance(dinv[0], list):
        return matvec(dinv, v)
    return [d * a for d, a in zip(dinv, v)]


def bicgstab(A: Mat, dinv: Vec, b: Vec, x0: Vec, iters: int):
    """Algorithm 1 in exact arithmetic.  Returns the list of states
    {x, r, p, alpha, omega, beta} per iteration (state i = before iteration i)."""
    n = len(b)
    x = list(x0)
    r = sub(b, matvec(A, x))                 # line 2
    r0 = list(r)
    p = list(r)
    out = []
    for _ in range(iters):
        g = prec(dinv, p)                    # line 4
        s = matvec(A, g)                     # line 5
        rs = dot(r0, s)
        if rs == 0:
            break
        alpha = dot(r0, r) / rs              # line 7
        q = sub(r, scal(alpha, s))           # line 8
        u = prec(dinv, q)                    # line 9
        y = matvec(A, u)                     # line 10
        yy = dot(y, y)
        omega = F(0) if yy == 0 else dot(q, y) / yy   # line 12 (A9 guard)
        out.append(dict(x=list(x), r=list(r), p=list(p), g=g, s=s, q=q, u=u, y=y,
                        alpha=alpha, omega=omega))
        x = add(add(x, scal(alpha, g)), scal(omega, u))  # line 13
        rn = sub(q, scal(omega, y))          # line 14
        if all(a == 0 for a in rn):
            out.append(dict(x=list(x), r=rn))
            return out
        if omega == 0:
            out.append(dict(x=list(x), r=rn))
            return out
        beta = (alpha / omega) * dot(r0, rn) / dot(r0, r)   # line 16
        out[-1]["beta"] = beta
        p = add(rn, scal(beta, sub(p, scal(omega, s))))      # line 17
        r = rn
    out.append(dict(x=list(x), r=list(r), p=list(p)))
    return out


def pbicgstab(A: Mat, dinv: Vec, b: Vec, x0: Vec, iters: int):
    """Algorithm 2 in exact arithmetic, reading A1 for the i=-1
    vectors.  Returns states per iteration: dict with x,r,k,w,m,t (entering i),
    and g,s,l,z,q,u,y,n,v, alpha, beta, omega (iteration i)."""
    n = len(b)
    zero = [F(0)] * n
    x = list(x0)
    r = sub(b, matvec(A, x))                 # line 2
    r0 = list(r)
    k = prec(dinv, r)
    w = matvec(A, k)
    m = prec(dinv, w)
    t = matvec(A, m)                         # line 3
    alpha = dot(r0, r) / dot(r0, w)
    beta = F(0)
    omega = F(0)
    g, s, l, z, nn, v = zero, zero, zero, zero, zero, zero
    out = []
    for _ in range(iters):
        st = dict(x=list(x), r=list(r), k=list(k), w=list(w), m=list(m), t=list(t),
                  alpha=alpha, beta=beta)
        g = add(k, scal(beta, sub(g, scal(omega, l))))      # line 5
        s = add(w, scal(beta, sub(s, scal(omega, z))))      # line 6
        l = add(m, scal(beta, sub(l, scal(omega, nn))))     # line 7
        z = add(t, scal(beta, sub(z, scal(omega, v))))      # line 8
        q = sub(r, scal(alpha, s))                          # line 9
        u = sub(k, scal(alpha, l))                          # line 10
        y = sub(w, scal(alpha, z))                          # line 11
        qy, yy = dot(q, y), dot(y, y)                       # line 12
        nn = prec(dinv, z)                                  # line 13
        v = matvec(A, nn)                                   # line 14
        omega = F(0) if yy == 0 else qy / yy                # line 16 (A9)
        st.update(g=g, s=s, l=l, z=z, q=q, u=u, y=y, n=nn, v=v, omega=omega)
        out.append(st)
        x = add(add(x, scal(alpha, g)), scal(omega, u))     # line 17
        r = sub(q, scal(omega, y))                          # line 18
        k = sub(u, scal(omega, sub(m, scal(alpha, nn))))    # line 19
        w = sub(y, scal(omega, sub(t, scal(alpha, v))))     # line 20
        rho1, dw, ds, dz = dot(r0, r), dot(r0, w), dot(r0, s), dot(r0, z)  # line 21
        m = prec(dinv, w)                                   # line 22
        t = matvec(A, m)                                    # line 23
        if all(a == 0 for a in r) or omega == 0:
            break
        beta = (alpha / omega) * rho1 / dot(r0, st["r"])    # line 25
        alpha = rho1 / (dw + beta * ds - beta * omega * dz)  # line 26
    out.append(dict(x=list(x), r=list(r), k=list(k), w=list(w), m=list(m), t=list(t)))
    return out


def pcg(A: Mat, dinv: Vec, b: Vec, x0: Vec, iters: int):
    x = list(x0)
    r = sub(b, matvec(A, x))
    u = prec(dinv, r)
    p = list(u)
    gam = dot(r, u)
    out = [dict(x=list(x), r=list(r))]
    for _ in range(iters):
        s = matvec(A, p)
        alpha = gam / dot(p, s)
        x = add(x, scal(alpha, p))
        r = sub(r, scal(alpha, s))
        u = prec(dinv, r)
        gam1 = dot(r, u)
        out[-1]["alpha"] = alpha
        out.append(dict(x=list(x), r=list(r)))
        if gam1 == 0:
            break
        p = add(u, scal(gam1 / gam, p))
        gam = gam1
    return out


def pipecg(A: Mat, dinv: Vec, b: Vec, x0: Vec, iters: int):
    """Reconstructed preconditioned pipelined CG (reading A19), as in oracle.c."""
    n = len(b)
    zero = [F(0)] * n
    x = list(x0)
    r = sub(b, matvec(A, x))
    u = prec(dinv, r)
    w = matvec(A, u)
    z = q = s = p = zero
    out = [dict(x=list(x), r=list(r), u=list(u), w=list(w))]
    gam_old = alpha_old = None
    for i in range(iters):
        gam, dl = dot(r, u), dot(w, u)
        if gam == 0:
            break
        m = prec(dinv, w)
        nn = matvec(A, m)
        if i == 0:
            beta, alpha = F(0), gam / dl
        else:
            beta = gam / gam_old
            alpha = gam / (dl - beta * gam / alpha_old)
        z = add(nn, scal(beta, z))
        q = add(m, scal(beta, q))
        s = add(w, scal(beta, s))
        p = add(u, scal(beta, p))
        x = add(x, scal(alpha, p))
        r = sub(r, scal(alpha, s))
        u = sub(u, scal(alpha, q))
        w = sub(w, scal(alpha, z))
        out[-1]["alpha"] = alpha
        out.append(dict(x=list(x), r=list(r), u=list(u), w=list(w), p=list(p), s=list(s),
                        q=list(q), z=list(z)))
        gam_old, alpha_old = gam, alpha
    return out


def norm(v: Vec) -> float:
    """Euclidean norm of an exact vector, as a float (correctly rounded square
    of the sum, then sqrt in float -- used only for bounds)."""
    return float(dot(v, v)) ** 0.5
