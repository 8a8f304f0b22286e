"""GPU parity of the automated residual replacement (SURVEY 8(f) NEXT-1, P:609-623;
option rr_auto) against the oracle.

The decisions (which iterations replace) are integers decided by the fp64 bound
f^r_i against tau ||r_i||: both sides decide in fp64 from the same formulas and
operation order, with every vector norm a Dot2 sum of squares (reading A30; the
GPU's per-thread Dot2 + fixed tree, the oracle's sequential Dot2), so f^r is
bitwise the oracle's and the replacement lists are identical by construction.
"""
import numpy as np
import pytest

from paper_1809_01948_b200 import problems

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from test_gpu_parity import check_parity, coef_of, stencil_case  # noqa: E402

@pytest.fixture(scope="module")
def S():
    from paper_1809_01948_b200 import Solver
    assert torch.cuda.is_available()
    return Solver


def check_auto(res, fr, rrl, ref, xs):
    """Decisions identical; north-star bars; bitwise iterates and f^r while
    ||r_i|| >= 1e-16 ||r_0||.  Below that the recursive residual is
    rounding noise: dot products of noise vectors are ill-conditioned beyond
    Dot2's guarantee, their rounding depends on the summation order, so the
    GPU's tree and the oracle's sequential sum may part (DESIGN.md parity rule)."""
    assert rrl == ref.rr_iters, (rrl, ref.rr_iters)
    check_parity(res, ref, xs, bitwise=False)
    assert res.iters == ref.iters
    noise = np.nonzero(ref.rnorm < 1e-16 * ref.rnorm[0])[0]
    k = int(noise[0]) if noise.size else ref.iters + 1
    assert np.array_equal(res.rnorm[:k], ref.rnorm[:k]), "rnorm not bitwise before the noise floor"
    if res.gap is not None and ref.gap is not None:
        assert np.array_equal(res.gap[:k], ref.gap[:k]), "gap not bitwise before the noise floor"
    if k > ref.iters:
        assert np.array_equal(res.x.cpu().numpy(), ref.x), "x not bitwise"
    assert np.array_equal(fr[:k], ref.bounds[:k, 0]), "f^r not bitwise"


CASES = [
    (2, 100, 100, 1, "poisson", 400),  # cfg1 shape
    (2, 64, 64, 1, "cd2", 300),
    (3, 20, 20, 20, "cd3", 200),
    (3, 13, 7, 19, "cd3", 200),        # ragged
    (2, 37, 53, 1, "cd2", 300),        # odd nx
]


@pytest.mark.parametrize("dim,nx,ny,nz,kind,maxit", CASES)
def test_auto_rr_parity(S, orc, dim, nx, ny, nz, kind, maxit):
    solver, A, xs, b, b_d = stencil_case(S, orc, dim, nx, ny, nz, coef_of(kind))
    solver.set_option("bench", 1)
    solver.set_option("rr_auto", 1)
    res = solver.solve(b_d, tol=0.0, maxit=maxit, gap=True)
    fr, rrl = solver.rr_info(res.iters)
    ref = orc.pbicgstab(A, b, tol=0.0, maxit=maxit, bench=True, auto_rr=True)
    assert len(ref.rr_iters) >= 1
    check_auto(res, fr, rrl, ref, xs)
    for j in rrl:
        assert res.gap[j + 1] == 0.0


def test_auto_rr_converging_and_graph_modes(S, orc):
    solver, A, xs, b, b_d = stencil_case(S, orc, 3, 24, 20, 18, problems.cfg34_coef())
    solver.set_option("rr_auto", 1)
    ref = orc.pbicgstab(A, b, tol=1e-13, maxit=600, auto_rr=True)
    out = []
    for graphs, timing in ((1, 0), (0, 0), (0, 1)):
        solver.set_option("graphs", graphs)
        solver.set_option("timing", timing)
        res = solver.solve(b_d, tol=1e-13, maxit=600, gap=True)
        fr, rrl = solver.rr_info(res.iters)
        assert res.outcome == ref.outcome
        check_auto(res, fr, rrl, ref, xs)
        out.append((res, fr))
    for res, fr in out[1:]:
        assert np.array_equal(fr, out[0][1])  # deterministic on the device


def test_periodic_rr_info_and_switching(S, orc):
    """rr_info also lists periodic replacements; switching rr_auto off restores the
    periodic schedule bitwise."""
    solver, A, xs, b, b_d = stencil_case(S, orc, 2, 64, 64, 1, problems.cfg2_coef())
    solver.set_option("bench", 1)
    ref = orc.pbicgstab(A, b, tol=0.0, maxit=200, rr_period=30, bench=True)
    for auto in (1, 0):
        solver.set_option("rr_auto", auto)
        if auto:
            solver.solve(b_d, tol=0.0, maxit=200, gap=True)
            continue
        res = solver.solve(b_d, tol=0.0, maxit=200, rr_period=30, gap=True)
        fr, rrl = solver.rr_info(res.iters)
        check_parity(res, ref, xs)
        assert rrl == ref.rr_iters
        assert np.all(np.isnan(fr))


def test_auto_rr_errors(S, orc):
    from paper_1809_01948_b200.binding import PbicgError
    solver, A, xs, b, b_d = stencil_case(S, orc, 2, 33, 17, 1, problems.cfg2_coef())
    solver.set_option("rr_auto", 1)
    with pytest.raises(PbicgError):
        solver.solve(b_d, tol=1e-10, maxit=10, rr_period=5)
    with pytest.raises(PbicgError):
        solver.set_option("method", 1)
    solver.set_option("rr_auto", 0)
    solver.set_option("method", 1)
    with pytest.raises(PbicgError):
        solver.set_option("rr_auto", 1)
    wide = S.stencil(2, 1501, 4, 1, problems.cfg2_coef())  # odd nx > 1024: line kernels
    with pytest.raises(PbicgError):
        wide.set_option("rr_auto", 1)


@pytest.mark.parametrize("band", [300, 6000])  # window / gather SpMV
def test_auto_rr_csr(S, orc, band):
    P = problems.csr_band(6000, nnz_row=27, band=band, seed=3)
    solver = S.csr(P.n, P.row_ptr, P.col, P.val)
    A = orc.csr(P.row_ptr, P.col, P.val)
    xs = problems.x_star(P.n, 0)
    b_d = solver.apply(torch.from_numpy(xs).cuda())
    b = orc.spmv(A, xs)
    solver.set_option("bench", 1)
    solver.set_option("rr_auto", 1)
    res = solver.solve(b_d, tol=0.0, maxit=60, gap=True)
    fr, rrl = solver.rr_info(res.iters)
    ref = orc.pbicgstab(A, b, tol=0.0, maxit=60, bench=True, auto_rr=True)
    check_auto(res, fr, rrl, ref, xs)


def test_auto_rr_csr_loopback(S, orc):
    from paper_1809_01948_b200.binding import LoopbackGroup
    A0 = orc.stencil_csr(2, 64, 192, 1, problems.cfg2_coef())  # CSR with stencil structure
    n, P = A0.n, 2
    rp, ci, va = A0.rp, A0.ci.astype(np.int32), A0.va
    cuts = [0, n // 2, n]
    blocks = [(cuts[r], rp[cuts[r]:cuts[r + 1] + 1] - rp[cuts[r]], ci[rp[cuts[r]]:rp[cuts[r + 1]]],
               va[rp[cuts[r]]:rp[cuts[r + 1]]]) for r in range(P)]
    G = LoopbackGroup.csr(blocks, n)
    G.set_option("bench", 1)
    G.set_option("rr_auto", 1)
    xs = problems.x_star(n, 0)
    b = orc.spmv(A0, xs)
    bs = G.apply(G.split(torch.from_numpy(xs).cuda()))
    res = G.solve(bs, tol=0.0, maxit=250, gap=True)
    fr, rrl = G.ranks[0].rr_info(res.iters)
    ref = orc.pbicgstab(A0, b, tol=0.0, maxit=250, bench=True, auto_rr=True)
    assert len(ref.rr_iters) >= 1
    check_auto(res, fr, rrl, ref, xs)
    G.close()


@pytest.mark.parametrize("P", [2, 3])
def test_auto_rr_loopback_multirank(S, orc, P):
    from paper_1809_01948_b200.binding import LoopbackGroup
    dim, nx, ny, nz = 3, 20, 17, 12
    coef = problems.cfg34_coef()
    A = orc.stencil_csr(dim, nx, ny, nz, coef)
    xs = problems.x_star(A.n, 0)
    b = orc.spmv(A, xs)
    G = LoopbackGroup.stencil(P, dim, nx, ny, nz, coef)
    G.set_option("bench", 1)
    G.set_option("rr_auto", 1)
    bs = G.apply(G.split(torch.from_numpy(xs).cuda()))
    res = G.solve(bs, tol=0.0, maxit=250, gap=True)
    fr, rrl = G.ranks[0].rr_info(res.iters)
    ref = orc.pbicgstab(A, b, tol=0.0, maxit=250, bench=True, auto_rr=True)
    assert len(ref.rr_iters) >= 1
    check_auto(res, fr, rrl, ref, xs)
    G.close()


def test_auto_rr_fullsize_cfg3_first_iterations(S, orc):
    """cfg3 at full size (256^3): 12 iterations with rr_auto; the bound history
    and the (empty or not) decision list match the oracle; iterates bitwise."""
    st = problems.configs()["cfg3"].stencil
    solver, A, xs, b, b_d = stencil_case(S, orc, st.dim, st.nx, st.ny, st.nz, st.coef)
    solver.set_option("bench", 1)
    solver.set_option("rr_auto", 1)
    res = solver.solve(b_d, tol=0.0, maxit=12, gap=False)
    fr, rrl = solver.rr_info(res.iters)
    ref = orc.pbicgstab(A, b, tol=0.0, maxit=12, bench=True, auto_rr=True, gap=False)
    check_auto(res, fr, rrl, ref, xs)


@pytest.mark.parametrize("block", [1, 2])
def test_auto_rr_csr_loopback_band_chain(S, orc, block):
    """Multi-rank CSR with rr_auto: the ||A|| bound's column sums are accumulated
    rank by rank (window hand-over, csr_bound_chain_step -- the code NCCL ranks run),
    with ranks of barely more than the halo so column sums span three ranks; the
    constants, hence f^r and the decisions, must be the one-process oracle's bitwise."""
    from paper_1809_01948_b200.binding import LoopbackGroup
    sizes = [4096 + 100, 4200, 4096 + 4]
    n = sum(sizes)
    M = problems.csr_band(n, nnz_row=9, band=4000, seed=12)
    A = orc.csr(M.row_ptr, M.col, M.val)
    cuts = np.concatenate([[0], np.cumsum(sizes)])
    blocks = [(int(cuts[r]), M.row_ptr[cuts[r]:cuts[r + 1] + 1] - M.row_ptr[cuts[r]],
               M.col[M.row_ptr[cuts[r]]:M.row_ptr[cuts[r + 1]]],
               M.val[M.row_ptr[cuts[r]]:M.row_ptr[cuts[r + 1]]]) for r in range(3)]
    G = LoopbackGroup.csr(blocks, n, block=block)
    G.set_option("bench", 1)
    G.set_option("rr_auto", 1)
    xs = problems.x_star(n, 4)
    b = orc.spmv(A, xs)
    bs = G.apply(G.split(torch.from_numpy(xs).cuda()))
    res = G.solve(bs, tol=0.0, maxit=40, gap=True)
    fr, rrl = G.ranks[0].rr_info(res.iters)
    ref = orc.pbicgstab(A, b, tol=0.0, maxit=40, bench=True, auto_rr=True, block=block)
    check_auto(res, fr, rrl, ref, xs)
    G.close()
