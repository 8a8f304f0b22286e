"""The NCCL transport on one GPU: a one-rank NCCL job (pbicg_dist with nranks = 1
and a unique id) runs the multi-rank schedule -- ncclCommInitRank /
ncclCommInitRankConfig, the rank-row all-reduce on the high-priority side
stream, empty send/recv groups, k_fin finalize kernels, NCCL nodes inside the
captured CUDA graphs, and (transport 1) the IPC-handle all-gather and peer-memory
publication -- and must reproduce the oracle bitwise, exactly like the plain
single-GPU path.  (Several ranks on one GPU are not used: kernels of different
ranks would wait on one another; B200_PROFILING.md.)
"""
import numpy as np
import pytest

from paper_1809_01948_b200 import problems

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from test_gpu_parity import check_parity  # noqa: E402


def _dist1():
    from paper_1809_01948_b200 import binding as B
    return B.make_dist(1, 0, B.nccl_unique_id(), B.nccl_unique_id())


@pytest.mark.parametrize("graphs", [0, 1])
@pytest.mark.parametrize("overlap", [0, 1])
@pytest.mark.parametrize("transport", [0, 1])
def test_nccl_one_rank_stencil(orc, graphs, overlap, transport):
    from paper_1809_01948_b200 import Solver
    dim, nx, ny, nz = 3, 24, 19, 11
    coef = problems.cfg34_coef()
    A = orc.stencil_csr(dim, nx, ny, nz, coef)
    xs = problems.x_star(A.n, 3)
    b = orc.spmv(A, xs)
    ref = orc.pbicgstab(A, b, tol=1e-11, maxit=120, rr_period=10)
    S = Solver.stencil(dim, nx, ny, nz, coef, dist=_dist1())
    S.set_option("graphs", graphs)
    S.set_option("overlap", overlap)
    S.set_option("transport", transport)
    b_d = S.apply(torch.from_numpy(xs).cuda())
    assert np.array_equal(b_d.cpu().numpy(), b)
    S.kernel_time("all", reset=True)
    res = S.solve(b_d, tol=1e-11, maxit=120, rr_period=10, gap=True)
    check_parity(res, ref, xs, bitwise=True)
    nfin, _ = S.kernel_time("fin")
    assert nfin >= 2 * res.iters, "the rank-row finalize kernels must run"
    S.close()


@pytest.mark.parametrize("method", [0, 1, 2])
def test_nccl_one_rank_methods(orc, method):
    from paper_1809_01948_b200 import Solver
    dim, nx, ny = 2, 64, 40
    coef = problems.poisson2d_coef()
    A = orc.stencil_csr(dim, nx, ny, 1, coef)
    xs = problems.x_star(A.n, 5)
    b = orc.spmv(A, xs)
    solve = {0: orc.pbicgstab, 1: orc.bicgstab, 2: orc.pipecg}[method]
    ref = solve(A, b, tol=1e-11, maxit=200)
    S = Solver.stencil(dim, nx, ny, 1, coef, dist=_dist1())
    S.set_option("method", method)
    b_d = torch.from_numpy(b).cuda()
    res = S.solve(b_d, tol=1e-11, maxit=200, gap=True)
    check_parity(res, ref, xs, bitwise=True)
    S.close()


@pytest.mark.parametrize("method,block", [(0, 1), (1, 1), (2, 1), (0, 4)])
def test_nccl_one_rank_csr(orc, method, block):
    from paper_1809_01948_b200 import Solver
    if method == 2:  # p-CG needs SPD: the 2D Poisson stencil written out as CSR
        A0 = orc.stencil_csr(2, 80, 75, 1, problems.poisson2d_coef())
        n, rp, ci, va = A0.n, A0.rp, A0.ci.astype(np.int32), A0.va
    else:
        n = 6000 - 6000 % block
        M = problems.csr_band(n, nnz_row=11, band=300, seed=11)
        rp, ci, va = M.row_ptr, M.col, M.val
    A = orc.csr(rp, ci, va)
    xs = problems.x_star(n, 11)
    b = orc.spmv(A, xs)
    solve = {0: orc.pbicgstab, 1: orc.bicgstab, 2: orc.pipecg}[method]
    kw = dict(rr_period=5) if method == 0 else {}
    ref = solve(A, b, tol=1e-12, maxit=60, block=block, **kw)
    S = Solver.csr(n, rp, ci, va, dist=_dist1(), block=block)
    S.set_option("method", method)
    b_d = torch.from_numpy(b).cuda()
    res = S.solve(b_d, tol=1e-12, maxit=60, gap=True, **kw)
    check_parity(res, ref, xs, bitwise=True)
    S.close()


def test_nccl_one_rank_auto_rr(orc):
    from paper_1809_01948_b200 import Solver
    dim, nx, ny = 2, 50, 50
    coef = problems.poisson2d_coef()
    A = orc.stencil_csr(dim, nx, ny, 1, coef)
    xs = problems.x_star(A.n, 0)
    b = orc.spmv(A, xs)
    ref = orc.pbicgstab(A, b, tol=0.0, maxit=300, bench=True, auto_rr=True)
    S = Solver.stencil(dim, nx, ny, 1, coef, dist=_dist1())
    S.set_option("rr_auto", 1)
    S.set_option("bench", 1)
    res = S.solve(torch.from_numpy(b).cuda(), tol=0.0, maxit=300, gap=True)
    fr, rr = S.rr_info(res.iters)
    assert rr == list(ref.rr_iters)
    k = np.nonzero(ref.rnorm < 1e-16 * ref.rnorm[0])[0]
    k = int(k[0]) if k.size else res.iters + 1
    assert np.array_equal(res.rnorm[:k], ref.rnorm[:k])
    S.close()
