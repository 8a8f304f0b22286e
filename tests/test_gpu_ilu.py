"""GPU parity of the ILU(0) / ICC(0) preconditioner (Table 1 ICC(0), P:659-697;
P:745 TP1 with ICC(0); reading A34) against the oracle:
bitwise histories and x for all three methods, stencils (the pipelined line-
wavefront kernels: one tile, several tiles in y / z, ragged tiles) and general
CSR (the level-ordered row kernel), periodic replacement, loopback ranks with the
block-diagonal reading, the one-rank NCCL path, and the error cases.
"""
import os

import numpy as np
import pytest

from paper_1809_01948_b200 import problems

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from test_gpu_parity import check_parity  # noqa: E402

REF = {0: "pbicgstab", 1: "bicgstab", 2: "pipecg"}


def _ref(orc, method, A, b, **kw):
    return getattr(orc, REF[method])(A, b, block="ilu0", **kw)


def _bitwise_above_floor(res, ref, floor=1e-16):
    k = np.nonzero(ref.rnorm < floor * ref.rnorm[0])[0]
    k = int(k[0]) if k.size else min(res.iters, ref.iters) + 1
    assert np.array_equal(res.rnorm[:k], ref.rnorm[:k])
    return k


STENCILS = [
    (2, 100, 100, 1, "poisson", "icc0"),   # cfg1 / TP1 shape: one tile
    (2, 37, 300, 1, "cd2", "ilu0"),        # two tiles along y (256 lines per tile)
    (3, 13, 7, 19, "cd3", "ilu0"),         # ragged 3D, TA = 7
    (3, 40, 37, 33, "cd3", "ilu0"),        # 3 x 3 tiles of 16 x 16 lines
    (3, 5, 6, 1, "cd3", "ilu0"),           # one plane
    (2, 1, 9, 1, "poisson", "icc0"),       # single column (falls back to the CSR kernel)
]


def _coef(kind):
    return {"poisson": problems.poisson2d_coef(), "cd2": problems.cfg2_coef(),
            "cd3": problems.cfg34_coef()}[kind]


@pytest.mark.parametrize("dim,nx,ny,nz,kind,prec", STENCILS)
@pytest.mark.parametrize("method", [0, 1, 2])
def test_ilu_stencil_parity(orc, dim, nx, ny, nz, kind, prec, method):
    from paper_1809_01948_b200 import Solver
    coef = _coef(kind)
    if method == 2:
        if kind != "poisson":
            coef = [6.0 if dim == 3 else 4.0] + [-1.0] * 6
        prec = "icc0"
    A = orc.stencil_csr(dim, nx, ny, nz, coef)
    xs = problems.x_star(A.n, 1)
    b = orc.spmv(A, xs)
    S = Solver.stencil(dim, nx, ny, nz, coef, block=prec)
    S.set_option("method", method)
    b_d = S.apply(torch.from_numpy(xs).cuda())
    assert np.array_equal(b_d.cpu().numpy(), b)
    rr = 7 if method == 0 else 0
    res = S.solve(b_d, tol=1e-12, maxit=300, rr_period=rr, gap=True)
    ref = _ref(orc, method, A, b, tol=1e-12, maxit=300, **({"rr_period": rr} if method == 0 else {}))
    assert res.outcome == ref.outcome
    check_parity(res, ref, xs, bitwise=True)
    n, _ = S.kernel_time("prec")
    assert n > 0, "the ILU kernels must run"
    S.close()


def test_cfg1_icc0_three_solvers_500_iterations(orc):
    """The Fig. 1 / Fig. 2 setting (TP1-like 2D Poisson with ICC(0)) on
    cfg1's grid: 500 iterations in bench mode for p-BiCGStab (with and without
    replacement every 50), BiCGStab and p-CG.  Classic BiCGStab and p-CG are bitwise
    over all 500 iterations; p-BiCGStab is bitwise above the noise floor, and where
    it leaves the oracle (its recursive residual stagnates at ~1e-15 ||r_0|| without
    replacement) the first differing scalar is named and must be within a few ulps
    (SURVEY 8(c4)); the history of iterations is printed for the record."""
    from paper_1809_01948_b200 import Solver
    from test_gpu_parity import noise_floor_parity
    st = problems.configs()["cfg1"].stencil
    A = orc.stencil_csr(2, st.nx, st.ny, 1, st.coef)
    xs = problems.x_star(A.n, 0)
    b = orc.spmv(A, xs)
    S = Solver.stencil(2, st.nx, st.ny, 1, st.coef, block="icc0")
    S.set_option("bench", 1)
    b_d = torch.from_numpy(b).cuda()
    for method, rr in ((0, 0), (0, 50), (1, 0), (2, 0)):
        S.set_option("method", method)
        res = S.solve(b_d, tol=0.0, maxit=500, rr_period=rr, gap=True)
        kw = {"rr_period": rr} if method == 0 else {}
        ref = getattr(orc, REF[method])(A, b, tol=0.0, maxit=500, bench=True, block="icc0",
                                        want_scalars=(method < 2), **kw) \
            if method < 2 else orc.pipecg(A, b, tol=0.0, maxit=500, bench=True, block="icc0")
        if method > 0:
            assert np.array_equal(res.rnorm, ref.rnorm) and np.array_equal(res.gap, ref.gap)
            assert np.array_equal(res.x.cpu().numpy(), ref.x)
            continue
        rerun = (lambda m, rr=rr: orc.pbicgstab(A, b, tol=0.0, maxit=m, bench=True, block="icc0",
                                                rr_period=rr, want_trace=True))
        noise_floor_parity(S, res, ref, xs, tag=f" cfg1 ICC(0) p-BiCGStab rr={rr}", rerun=rerun)
    S.close()


@pytest.mark.parametrize("band", [8, 300, 5000])
@pytest.mark.parametrize("method", [0, 1])
def test_ilu_csr_parity(orc, band, method):
    from paper_1809_01948_b200 import Solver
    n = 6000
    M = problems.csr_band(n, nnz_row=min(13, band + 1), band=band, seed=band)
    A = orc.csr(M.row_ptr, M.col, M.val)
    xs = problems.x_star(n, 2)
    b = orc.spmv(A, xs)
    S = Solver.csr(n, M.row_ptr, M.col, M.val, block="ilu0")
    S.set_option("method", method)
    kw = {"rr_period": 5} if method == 0 else {}
    res = S.solve(torch.from_numpy(b).cuda(), tol=1e-12, maxit=80, gap=True, **kw)
    ref = _ref(orc, method, A, b, tol=1e-12, maxit=80, **kw)
    assert res.outcome == ref.outcome
    check_parity(res, ref, xs, bitwise=True)
    S.close()


def test_ilu_csr_pipecg_symmetric(orc):
    from paper_1809_01948_b200 import Solver
    A = orc.stencil_csr(3, 12, 11, 10, [6.0, -1, -1, -1, -1, -1, -1])
    xs = problems.x_star(A.n, 3)
    b = orc.spmv(A, xs)
    S = Solver.csr(A.n, A.rp, A.ci.astype(np.int32), A.va, block="icc0")
    S.set_option("method", 2)
    res = S.solve(torch.from_numpy(b).cuda(), tol=1e-12, maxit=100, gap=True)
    ref = _ref(orc, 2, A, b, tol=1e-12, maxit=100)
    check_parity(res, ref, xs, bitwise=True)
    S.close()


def _random_shapes():
    """Seeded 3D grids around the k_ilu_st tile geometry (16 x 16 lines per tile, blocks of
    8 steps): x shorter than a block, ragged last tiles in y / z, one to five tiles per
    direction, plus two fixed many-tile cases."""
    rng = np.random.default_rng(20181809 + int(os.environ.get("PBICG_FUZZ_OFFSET", "0")))
    shapes = [(96, 80, 72), (9, 70, 83)]
    for _ in range(int(os.environ.get("PBICG_ILU_SHAPES", "22"))):  # wide sweeps: more shapes
        shapes.append((int(rng.integers(2, 71)), int(rng.integers(2, 52)), int(rng.integers(2, 52))))
    return shapes


@pytest.mark.parametrize("case,shape", list(enumerate(_random_shapes())))
def test_ilu_stencil_random_shapes(orc, case, shape):
    """The 3D wavefront sweeps (transposed staging, loader / publisher warps, tile
    hand-over) on randomised grids: a short ILU(0) solve per shape, histories and x
    bitwise vs the oracle (any wrong row, stale boundary value or missed hand-over
    changes the first iterations' bits)."""
    from paper_1809_01948_b200 import Solver
    nx, ny, nz = shape
    method = case % 3
    coef = problems.cfg34_coef() if method != 2 else [6.0] + [-1.0] * 6
    prec = "ilu0" if method != 2 else "icc0"
    A = orc.stencil_csr(3, nx, ny, nz, coef)
    xs = problems.x_star(A.n, 100 + case)
    b = orc.spmv(A, xs)
    S = Solver.stencil(3, nx, ny, nz, coef, block=prec)
    S.set_option("method", method)
    b_d = S.apply(torch.from_numpy(xs).cuda())
    rr = 5 if method == 0 else 0
    for rep in range(2):  # the second solve reuses the epoch-stamped progress counters
        res = S.solve(b_d, tol=1e-13, maxit=12, rr_period=rr, gap=False)
        ref = _ref(orc, method, A, b, tol=1e-13, maxit=12, **({"rr_period": rr} if method == 0 else {}))
        assert res.outcome == ref.outcome
        k = min(res.iters, ref.iters) + 1
        assert np.array_equal(res.rnorm[:k], ref.rnorm[:k]), (shape, method, rep)
        assert np.array_equal(res.x.cpu().numpy(), ref.x), (shape, method, rep)
    n, _ = S.kernel_time("prec")
    assert n > 0, "the ILU kernels must run"
    S.close()


@pytest.mark.parametrize("case,shape", [(c, sh) for c, sh in enumerate(_random_shapes()) if c % 3 == 0])
def test_ilu_stencil_random_shapes_loopback(orc, case, shape):
    """The same sweeps on P = 2 / 3 loopback ranks (each rank's slab is its own tile grid,
    block-diagonal reading A35) for every third random shape, both transports."""
    from paper_1809_01948_b200.binding import LoopbackGroup, stencil_partition
    nx, ny, nz = shape
    P = 2 + (case // 3) % 2
    if nz < P:
        pytest.skip("fewer planes than ranks")
    coef = problems.cfg34_coef()
    A = orc.stencil_csr(3, nx, ny, nz, coef)
    xs = problems.x_star(A.n, 200 + case)
    b = orc.spmv(A, xs)
    cuts = [stencil_partition(3, nx, ny, nz, P, r)[0] for r in range(P)] + [A.n]
    with orc.prec_matrix(orc.block_diagonal(A, cuts)):
        ref = orc.pbicgstab(A, b, tol=1e-13, maxit=12, rr_period=5, block="ilu0")
    G = LoopbackGroup.stencil(P, 3, nx, ny, nz, coef, block="ilu0")
    for transport in (0, 1):
        G.set_option("transport", transport)
        bs = G.apply(G.split(torch.from_numpy(xs).cuda()))
        res = G.solve(bs, tol=1e-13, maxit=12, rr_period=5, gap=False)
        assert res.outcome == ref.outcome
        k = min(res.iters, ref.iters) + 1
        assert np.array_equal(res.rnorm[:k], ref.rnorm[:k]), (shape, P, transport)
        x = res.x.cpu().numpy() if hasattr(res.x, "cpu") else res.x
        assert np.array_equal(x, ref.x), (shape, P, transport)
    G.close()


def test_ilu_loopback_odd_plane_window_alignment(orc):
    """Regression (round 2): three loopback ranks of one 35 x 47 plane each -- an odd ghost
    width -- made the window SpMV's bulk copies misaligned ("misaligned address"); such
    handles now keep the gather SpMV.  Bitwise vs the oracle's block-diagonal reading."""
    from paper_1809_01948_b200.binding import LoopbackGroup, stencil_partition
    nx, ny, nz, P = 35, 47, 3, 3
    coef = problems.cfg34_coef()
    A = orc.stencil_csr(3, nx, ny, nz, coef)
    xs = problems.x_star(A.n, 7)
    b = orc.spmv(A, xs)
    cuts = [stencil_partition(3, nx, ny, nz, P, r)[0] for r in range(P)] + [A.n]
    with orc.prec_matrix(orc.block_diagonal(A, cuts)):
        ref = orc.pbicgstab(A, b, tol=1e-12, maxit=60, rr_period=9, block="ilu0")
    G = LoopbackGroup.stencil(P, 3, nx, ny, nz, coef, block="ilu0")
    bs = G.apply(G.split(torch.from_numpy(xs).cuda()))
    res = G.solve(bs, tol=1e-12, maxit=60, rr_period=9, gap=True)
    check_parity(res, ref, xs, bitwise=True)
    G.close()


@pytest.mark.parametrize("P", [2, 3])
def test_ilu_stencil_loopback_block_reading(orc, P):
    """P ranks: each factorises its own slab (the block-diagonal part of A, A34)."""
    from paper_1809_01948_b200.binding import LoopbackGroup, stencil_partition
    dim, nx, ny, nz = 3, 24, 18, 13
    coef = problems.cfg34_coef()
    A = orc.stencil_csr(dim, nx, ny, nz, coef)
    xs = problems.x_star(A.n, 4)
    b = orc.spmv(A, xs)
    cuts = [stencil_partition(dim, nx, ny, nz, P, r)[0] for r in range(P)] + [A.n]
    with orc.prec_matrix(orc.block_diagonal(A, cuts)):
        ref = orc.pbicgstab(A, b, tol=1e-12, maxit=200, rr_period=9, block="ilu0")
    G = LoopbackGroup.stencil(P, dim, nx, ny, nz, coef, block="ilu0")
    for transport in (0, 1):
        G.set_option("transport", transport)
        bs = G.apply(G.split(torch.from_numpy(xs).cuda()))
        res = G.solve(bs, tol=1e-12, maxit=200, rr_period=9, gap=True)
        check_parity(res, ref, xs, bitwise=True)
    G.close()


def test_ilu_csr_loopback_block_reading(orc):
    from paper_1809_01948_b200.binding import LoopbackGroup
    P, n = 3, 3 * 5000
    M = problems.csr_band(n, nnz_row=11, band=200, seed=9)
    A = orc.csr(M.row_ptr, M.col, M.val)
    xs = problems.x_star(n, 5)
    b = orc.spmv(A, xs)
    cuts = [0, 5000, 10000, n]
    blocks = [(cuts[r], M.row_ptr[cuts[r]:cuts[r + 1] + 1] - M.row_ptr[cuts[r]],
               M.col[M.row_ptr[cuts[r]]:M.row_ptr[cuts[r + 1]]],
               M.val[M.row_ptr[cuts[r]]:M.row_ptr[cuts[r + 1]]]) for r in range(P)]
    with orc.prec_matrix(orc.block_diagonal(A, cuts)):
        ref = orc.pbicgstab(A, b, tol=1e-12, maxit=100, rr_period=4, block="ilu0")
        ref1 = orc.bicgstab(A, b, tol=1e-12, maxit=100, block="ilu0")
    G = LoopbackGroup.csr(blocks, n, block="ilu0")
    for ov in (1, 0):
        G.set_option("overlap", ov)
        G.set_option("method", 0)
        bs = G.apply(G.split(torch.from_numpy(xs).cuda()))
        res = G.solve(bs, tol=1e-12, maxit=100, rr_period=4, gap=True)
        check_parity(res, ref, xs, bitwise=True)
        G.set_option("method", 1)
        res = G.solve(bs, tol=1e-12, maxit=100, gap=True)
        check_parity(res, ref1, xs, bitwise=True)
    G.close()


def test_ilu_nccl_one_rank(orc):
    from paper_1809_01948_b200 import Solver
    from paper_1809_01948_b200 import binding as B
    d = B.make_dist(1, 0, B.nccl_unique_id(), B.nccl_unique_id())
    A = orc.stencil_csr(2, 64, 48, 1, problems.poisson2d_coef())
    xs = problems.x_star(A.n, 6)
    b = orc.spmv(A, xs)
    S = Solver.stencil(2, 64, 48, 1, problems.poisson2d_coef(), dist=d, block="icc0")
    res = S.solve(torch.from_numpy(b).cuda(), tol=1e-12, maxit=200, rr_period=20, gap=True)
    ref = orc.pbicgstab(A, b, tol=1e-12, maxit=200, rr_period=20, block="icc0")
    check_parity(res, ref, xs, bitwise=True)
    S.close()


def test_ilu_errors():
    from paper_1809_01948_b200 import Solver
    from paper_1809_01948_b200.binding import PbicgError
    with pytest.raises(PbicgError):  # ICC(0) of an unsymmetric stencil
        Solver.stencil(3, 8, 8, 8, problems.cfg34_coef(), block="icc0")
    M = problems.csr_band(512, nnz_row=5, band=8, seed=1)
    with pytest.raises(PbicgError):  # ICC(0) of an unsymmetric CSR matrix
        Solver.csr(512, M.row_ptr, M.col, M.val, block="icc0")
    S = Solver.stencil(2, 16, 16, 1, problems.poisson2d_coef(), block="icc0")
    with pytest.raises(PbicgError):  # no automated replacement with ILU(0)
        S.set_option("rr_auto", 1)
    S.close()
