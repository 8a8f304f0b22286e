"""GPU parity of the block-Jacobi preconditioner (reading A33)
on CSR operators and matrix-free stencils, against the oracle: the library inverts the diagonal blocks
with its own Gauss-Jordan (same textbook operations as the oracle's) and applies
them with warp shuffles, so the runs are expected bitwise equal.
"""
import numpy as np
import pytest

from paper_1809_01948_b200 import problems

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from test_gpu_parity import check_parity  # noqa: E402


@pytest.fixture(scope="module")
def S():
    from paper_1809_01948_b200 import Solver
    assert torch.cuda.is_available()
    return Solver


def case(S, orc, A, block, seed=0):
    solver = S.csr(A.n, A.rp, A.ci.astype(np.int32), A.va, block=block)
    xs = problems.x_star(A.n, seed)
    b_d = solver.apply(torch.from_numpy(xs).cuda())
    b = orc.spmv(A, xs)
    assert np.array_equal(b_d.cpu().numpy(), b)
    return solver, xs, b, b_d


def band(n, bw, seed):
    P = problems.csr_band(n, nnz_row=27, band=bw, seed=seed)
    from oracle import oracle as o
    return o.csr(P.row_ptr, P.col, P.val)


@pytest.mark.parametrize("block", [1, 2, 4, 8, 16, 32])
@pytest.mark.parametrize("bw", [300, 6000])  # window SpMV / gather SpMV
def test_bj_pbicgstab_parity(S, orc, block, bw):
    A = band(8192, bw, 1)
    solver, xs, b, b_d = case(S, orc, A, block)
    for rr in (0, 3):
        res = solver.solve(b_d, tol=1e-12, maxit=100, rr_period=rr, gap=True)
        ref = orc.pbicgstab(A, b, tol=1e-12, maxit=100, rr_period=rr, block=block)
        assert res.outcome == ref.outcome
        check_parity(res, ref, xs)


@pytest.mark.parametrize("block", [4, 8])
def test_bj_stencil_as_csr_all_methods(S, orc, block):
    """A 2D Poisson stencil written out as CSR (ragged rows): block Jacobi speeds
    up every solver; p-BiCGStab, classic BiCGStab and p-CG bitwise vs the oracle."""
    A = orc.stencil_csr(2, 40, 30, 1, problems.poisson2d_coef())
    solver, xs, b, b_d = case(S, orc, A, block)
    for method, ref in ((0, orc.pbicgstab(A, b, tol=1e-10, maxit=500, block=block)),
                        (1, orc.bicgstab(A, b, tol=1e-10, maxit=500, block=block)),
                        (2, orc.pipecg(A, b, tol=1e-10, maxit=500, block=block))):
        solver.set_option("method", method)
        res = solver.solve(b_d, tol=1e-10, maxit=500, gap=True)
        assert res.outcome == ref.outcome == "converged"
        check_parity(res, ref, xs)
        jac = {0: orc.pbicgstab, 1: orc.bicgstab, 2: orc.pipecg}[method](A, b, tol=1e-10, maxit=500)
        assert res.iters < jac.iters


def test_bj_auto_rr(S, orc):
    A = orc.stencil_csr(2, 64, 64, 1, problems.cfg2_coef())
    solver, xs, b, b_d = case(S, orc, A, 4)
    solver.set_option("bench", 1)
    solver.set_option("rr_auto", 1)
    res = solver.solve(b_d, tol=0.0, maxit=200, gap=True)
    fr, rrl = solver.rr_info(res.iters)
    ref = orc.pbicgstab(A, b, tol=0.0, maxit=200, bench=True, auto_rr=True, block=4)
    from test_gpu_autorr import check_auto
    check_auto(res, fr, rrl, ref, xs)


@pytest.mark.parametrize("method", [0, 1, 2])
def test_bj_loopback(S, orc, method):
    from paper_1809_01948_b200.binding import LoopbackGroup
    A = orc.stencil_csr(2, 64, 192, 1, problems.poisson2d_coef())
    n, P, blk = A.n, 3, 8
    rp, ci, va = A.rp, A.ci.astype(np.int32), A.va
    cuts = [0, 4096, 8192, n]
    blocks = [(cuts[r], rp[cuts[r]:cuts[r + 1] + 1] - rp[cuts[r]], ci[rp[cuts[r]]:rp[cuts[r + 1]]],
               va[rp[cuts[r]]:rp[cuts[r + 1]]]) for r in range(P)]
    G = LoopbackGroup.csr(blocks, n, block=blk)
    G.set_option("method", method)
    xs = problems.x_star(n, 0)
    b = orc.spmv(A, xs)
    bs = G.apply(G.split(torch.from_numpy(xs).cuda()))
    res = G.solve(bs, tol=1e-10, maxit=400, rr_period=0, gap=True)
    ref = {0: orc.pbicgstab, 1: orc.bicgstab, 2: orc.pipecg}[method](A, b, tol=1e-10, maxit=400,
                                                                      block=blk)
    check_parity(res, ref, xs)
    G.close()


STENCILS = [(2, 64, 48, 1, "cd2"), (2, 40, 30, 1, "poisson"), (3, 16, 12, 10, "cd3"),
            (3, 64, 64, 64, "cd3"), (3, 8, 5, 7, "cd3"),
            # one-line tiles with the widest halos that fit (3D nx = 840: the transform
            # stage's halo pairs take two rounds of the CTA), a tile of one block per line
            (3, 840, 3, 4, "cd3"), (3, 520, 5, 4, "cd3"), (2, 1024, 6, 1, "cd2"),
            (2, 8, 40, 1, "cd2")]


@pytest.mark.parametrize("block", [2, 4, 8])
@pytest.mark.parametrize("shape", STENCILS)
def test_bj_stencil_parity(S, orc, block, shape):
    """Matrix-free stencils with x-aligned blocks: tile kernels apply the common
    inverse block from shared memory (stencil legs) and by lane shuffles (k, l in
    the replacement / init steps); bitwise vs the oracle's CSR form."""
    from test_gpu_parity import coef_of
    dim, nx, ny, nz, kind = shape
    if nx % block:
        pytest.skip("nx % b != 0")
    coef = coef_of(kind)
    solver = S.stencil(dim, nx, ny, nz, coef, block=block)
    A = orc.stencil_csr(dim, nx, ny, nz, coef)
    xs = problems.x_star(A.n, 0)
    b_d = solver.apply(torch.from_numpy(xs).cuda())
    b = orc.spmv(A, xs)
    for rr in (0, 5):
        res = solver.solve(b_d, tol=1e-11, maxit=150, rr_period=rr, gap=True)
        ref = orc.pbicgstab(A, b, tol=1e-11, maxit=150, rr_period=rr, block=block)
        assert res.outcome == ref.outcome
        check_parity(res, ref, xs)
    solver.set_option("bench", 1)
    solver.set_option("rr_auto", 1)
    res = solver.solve(b_d, tol=0.0, maxit=120, gap=True)
    fr, rrl = solver.rr_info(res.iters)
    ref = orc.pbicgstab(A, b, tol=0.0, maxit=120, bench=True, auto_rr=True, block=block)
    from test_gpu_autorr import check_auto
    check_auto(res, fr, rrl, ref, xs)


@pytest.mark.parametrize("method", [1, 2])
@pytest.mark.parametrize("block", [2, 4, 8])
@pytest.mark.parametrize("shape", STENCILS)
def test_bj_stencil_methods(S, orc, block, shape, method):
    """Classic BiCGStab (Alg. 1: the derived p_i, q_i are derived then transformed once
    per staged element, g := M^-1 p by lane shuffles) and p-CG (m := M^-1 w from the
    stencil's block, u0 := M^-1 r0 by lane shuffles) with stencil block Jacobi, bitwise
    vs the oracle's CSR form; p-CG on the symmetric (Poisson) stencils only."""
    from test_gpu_parity import coef_of
    dim, nx, ny, nz, kind = shape
    if nx % block:
        pytest.skip("nx % b != 0")
    coef = coef_of(kind)
    if method == 2:  # p-CG needs a symmetric M and A
        coef = problems.poisson3d_coef() if dim == 3 else problems.poisson2d_coef()
    solver = S.stencil(dim, nx, ny, nz, coef, block=block)
    solver.set_option("method", method)
    A = orc.stencil_csr(dim, nx, ny, nz, coef)
    xs = problems.x_star(A.n, 0)
    b_d = solver.apply(torch.from_numpy(xs).cuda())
    b = orc.spmv(A, xs)
    fn = orc.bicgstab if method == 1 else orc.pipecg
    res = solver.solve(b_d, tol=1e-11, maxit=150, gap=True)
    ref = fn(A, b, tol=1e-11, maxit=150, block=block)
    assert res.outcome == ref.outcome
    check_parity(res, ref, xs)
    solver.set_option("bench", 1)  # bench mode: exactly maxit iterations
    res = solver.solve(b_d, tol=0.0, maxit=40, gap=True)
    ref = fn(A, b, tol=0.0, maxit=40, bench=True, block=block)
    assert res.outcome == ref.outcome
    check_parity(res, ref, xs)


@pytest.mark.parametrize("method", [1, 2])
@pytest.mark.parametrize("P", [2, 3])
def test_bj_stencil_methods_loopback(S, orc, P, method):
    from paper_1809_01948_b200.binding import LoopbackGroup
    dim, nx, ny, nz, blk = 3, 24, 10, 9, 4
    coef = problems.cfg34_coef() if method == 1 else problems.poisson3d_coef()
    A = orc.stencil_csr(dim, nx, ny, nz, coef)
    xs = problems.x_star(A.n, 0)
    b = orc.spmv(A, xs)
    G = LoopbackGroup.stencil(P, dim, nx, ny, nz, coef, block=blk)
    G.set_option("method", method)
    bs = G.apply(G.split(torch.from_numpy(xs).cuda()))
    res = G.solve(bs, tol=1e-11, maxit=200, rr_period=0, gap=True)
    fn = orc.bicgstab if method == 1 else orc.pipecg
    ref = fn(A, b, tol=1e-11, maxit=200, block=blk)
    check_parity(res, ref, xs)
    G.close()


@pytest.mark.parametrize("P", [2, 3])
def test_bj_stencil_loopback(S, orc, P):
    from paper_1809_01948_b200.binding import LoopbackGroup
    dim, nx, ny, nz, blk = 3, 24, 10, 9, 4
    coef = problems.cfg34_coef()
    A = orc.stencil_csr(dim, nx, ny, nz, coef)
    xs = problems.x_star(A.n, 0)
    b = orc.spmv(A, xs)
    G = LoopbackGroup.stencil(P, dim, nx, ny, nz, coef, block=blk)
    bs = G.apply(G.split(torch.from_numpy(xs).cuda()))
    res = G.solve(bs, tol=1e-11, maxit=200, rr_period=7, gap=True)
    ref = orc.pbicgstab(A, b, tol=1e-11, maxit=200, rr_period=7, block=blk)
    check_parity(res, ref, xs)
    G.close()


def test_bj_stencil_cfg3_fullsize_first_iterations(S, orc):
    st = problems.configs()["cfg3"].stencil
    solver = S.stencil(st.dim, st.nx, st.ny, st.nz, st.coef, block=4)
    A = orc.stencil_csr(st.dim, st.nx, st.ny, st.nz, st.coef)
    xs = problems.x_star(A.n, 0)
    b_d = solver.apply(torch.from_numpy(xs).cuda())
    b = orc.spmv(A, xs)
    res = solver.solve(b_d, tol=0.0, maxit=3, rr_period=2, gap=True)
    ref = orc.pbicgstab(A, b, tol=0.0, maxit=3, rr_period=2, block=4)
    check_parity(res, ref, xs)


def test_bj_errors(S, orc):
    from paper_1809_01948_b200.binding import PbicgError
    A = orc.stencil_csr(2, 10, 9, 1, problems.poisson2d_coef())  # n = 90
    with pytest.raises(PbicgError):  # n not a multiple of b
        S.csr(A.n, A.rp, A.ci.astype(np.int32), A.va, block=4)
    with pytest.raises(PbicgError):  # unsupported block size
        S.csr(A.n, A.rp, A.ci.astype(np.int32), A.va, block=3)
    with pytest.raises(PbicgError):  # stencil: nx % b != 0
        S.stencil(2, 10, 8, 1, problems.poisson2d_coef(), block=4)
    with pytest.raises(PbicgError):  # stencil: b <= 8
        S.stencil(2, 32, 8, 1, problems.poisson2d_coef(), block=16)
    with pytest.raises(PbicgError):  # x-segmented tiles (nx > 1024) have no block Jacobi
        S.stencil(2, 2048, 4, 1, problems.poisson2d_coef(), block=4)
    with pytest.raises(PbicgError):  # 3D planes too wide for full-line tiles: segmented
        S.stencil(3, 1024, 3, 4, problems.cfg34_coef(), block=4)
    st = S.stencil(2, 32, 8, 1, problems.poisson2d_coef(), block=4)
    with pytest.raises(PbicgError):  # line kernels have no block Jacobi
        st.set_option("tile", 0)
