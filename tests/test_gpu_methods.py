"""GPU parity of the comparison solvers against the
oracle: classic preconditioned BiCGStab (Alg. 1; option method=1) and
preconditioned pipelined CG (reading A19; option method=2), stencil operators,
through the C ABI.  Same bars as tests/test_gpu_parity.py; the design target is
bitwise equality of ||r_i||, the gap history and x.
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


def ref_of(orc, method, A, b, **kw):
    return orc.bicgstab(A, b, **kw) if method == 1 else orc.pipecg(A, b, **kw)


SHAPES = [
    (2, 100, 100, 1, "poisson"),  # cfg1 shape
    (2, 37, 53, 1, "cd2"),        # ragged, odd nx (unpaired loads)
    (3, 13, 7, 19, "cd3"),        # ragged 3D
    (3, 40, 33, 31, "cd3"),
    (3, 64, 64, 64, "cd3"),       # several tiles per plane, several chunks
    (2, 1024, 64, 1, "cd2"),      # widest tile row
    (3, 5, 6, 7, "cd3"),          # nx < 32
    (3, 1, 1, 1, "cd3"),          # N = 1
]

SPD_SHAPES = [(2, 100, 100, 1), (2, 37, 53, 1), (3, 13, 7, 19), (3, 64, 64, 64), (3, 1, 1, 1)]


@pytest.mark.parametrize("dim,nx,ny,nz,kind", SHAPES)
def test_classic_bicgstab_parity(S, orc, dim, nx, ny, nz, kind):
    solver, A, xs, b, b_d = stencil_case(S, orc, dim, nx, ny, nz, coef_of(kind))
    solver.set_option("method", 1)
    res = solver.solve(b_d, tol=1e-10, maxit=150, gap=True)
    ref = orc.bicgstab(A, b, tol=1e-10, maxit=150)
    assert res.outcome == ref.outcome
    check_parity(res, ref, xs)


@pytest.mark.parametrize("dim,nx,ny,nz", SPD_SHAPES)
def test_pipecg_parity(S, orc, dim, nx, ny, nz):
    """p-CG on SPD Poisson operators (CG needs symmetry)."""
    coef = problems.poisson2d_coef() if dim == 2 else [6.0, -1, -1, -1, -1, -1, -1]
    solver, A, xs, b, b_d = stencil_case(S, orc, dim, nx, ny, nz, coef)
    solver.set_option("method", 2)
    res = solver.solve(b_d, tol=1e-10, maxit=400, gap=True)
    ref = orc.pipecg(A, b, tol=1e-10, maxit=400)
    assert res.outcome == ref.outcome
    check_parity(res, ref, xs)


def test_cfg1_three_solvers_500_iterations(S, orc):
    """cfg1: p-BiCGStab vs classic BiCGStab vs p-CG residual/gap histories over 500
    fixed iterations, all three on the GPU, each bitwise equal to its oracle."""
    st = problems.configs()["cfg1"].stencil
    solver, A, xs, b, b_d = stencil_case(S, orc, st.dim, st.nx, st.ny, st.nz, st.coef)
    solver.set_option("bench", 1)
    for method, ref in ((0, orc.pbicgstab(A, b, tol=0.0, maxit=500, bench=True)),
                        (1, orc.bicgstab(A, b, tol=0.0, maxit=500, bench=True)),
                        (2, orc.pipecg(A, b, tol=0.0, maxit=500, bench=True))):
        solver.set_option("method", method)
        res = solver.solve(b_d, tol=0.0, maxit=500, gap=True)
        assert res.iters == ref.iters, (method, res.iters, ref.iters, ref.outcome)
        check_parity(res, ref, xs)


def test_methods_switch_back_and_forth(S, orc):
    """Switching the method on one handle leaves no state behind."""
    solver, A, xs, b, b_d = stencil_case(S, orc, 3, 24, 20, 18, problems.cfg34_coef())
    runs = {}
    for method in (0, 1, 0, 1):
        solver.set_option("method", method)
        r = solver.solve(b_d, tol=1e-10, maxit=200, rr_period=0, gap=True)
        if method in runs:
            assert np.array_equal(r.rnorm, runs[method].rnorm)
            assert np.array_equal(r.x.cpu().numpy(), runs[method].x.cpu().numpy())
        runs[method] = r


def test_graphs_timing_host_entry_identical(S, orc):
    solver, A, xs, b, b_d = stencil_case(S, orc, 3, 20, 18, 16, problems.cfg34_coef())
    for method in (1, 2):
        if method == 2:
            solver, A, xs, b, b_d = stencil_case(S, orc, 3, 20, 18, 16, [6.0, -1, -1, -1, -1, -1, -1])
        solver.set_option("method", method)
        out = []
        for graphs, timing in ((1, 0), (0, 0), (0, 1)):
            solver.set_option("graphs", graphs)
            solver.set_option("timing", timing)
            out.append(solver.solve(b_d, tol=1e-10, maxit=300, gap=True))
        out.append(solver.solve_host(b, tol=1e-10, maxit=300, gap=True))
        for r in out[1:]:
            assert r.iters == out[0].iters
            assert np.array_equal(r.rnorm, out[0].rnorm)
            x = r.x.cpu().numpy() if hasattr(r.x, "cpu") else r.x
            assert np.array_equal(x, out[0].x.cpu().numpy())
        n, ms = solver.kernel_time("cl3" if method == 1 else "pcg")
        assert n > 0 and ms > 0


def test_degenerate_and_errors(S, orc):
    from paper_1809_01948_b200.binding import PbicgError
    solver, A, xs, b, b_d = stencil_case(S, orc, 2, 33, 17, 1, problems.cfg2_coef())
    for method in (1, 2):
        solver.set_option("method", method)
        z = torch.zeros_like(b_d)
        r = solver.solve(z, tol=1e-10, maxit=10)
        assert r.outcome == "converged" and r.iters == 0
        assert torch.count_nonzero(r.x).item() == 0
        r = solver.solve(b_d, tol=1e-10, maxit=0)
        ref = ref_of(orc, method, A, b, tol=1e-10, maxit=0)
        assert r.outcome == "maxit" and r.iters == 0 and r.rnorm[0] == ref.rnorm[0]
        with pytest.raises(PbicgError):
            solver.solve(b_d, tol=1e-10, maxit=10, rr_period=5)  # RR is Alg. 2 only
    # identity operator: Alg. 1 converges in one step (y = q => omega = 1... or lucky)
    ident = S.stencil(3, 8, 8, 8, [1, 0, 0, 0, 0, 0, 0])
    bi = problems.x_star(512, 3)
    A1 = orc.stencil_csr(3, 8, 8, 8, [1, 0, 0, 0, 0, 0, 0])
    for method in (1, 2):
        ident.set_option("method", method)
        r = ident.solve(torch.from_numpy(bi).cuda(), tol=1e-14, maxit=5)
        ref = ref_of(orc, method, A1, bi, tol=1e-14, maxit=5)
        assert (r.iters, r.outcome) == (ref.iters, ref.outcome)
        assert np.array_equal(r.rnorm, ref.rnorm)
        assert np.array_equal(r.x.cpu().numpy(), ref.x)
    # stencils with nx > 1024 reject methods 1/2 (tile kernels only)
    wide = S.stencil(2, 1501, 4, 1, problems.cfg2_coef())  # odd nx > 1024: line kernels only
    with pytest.raises(PbicgError):
        wide.set_option("method", 2)


@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("method", [1, 2])
def test_methods_loopback_multirank(S, orc, P, method):
    """The multi-rank path (slabs, halos of p/s/r or w, rank-row reductions,
    finalize kernels) reproduces the oracle bitwise for P emulated ranks."""
    from paper_1809_01948_b200.binding import LoopbackGroup
    dim, nx, ny, nz = 3, 20, 17, 9
    coef = problems.cfg34_coef() if method == 1 else [6.0, -1, -1, -1, -1, -1, -1]
    A = orc.stencil_csr(dim, nx, ny, nz, coef)
    xs = problems.x_star(A.n, 0)
    b = orc.spmv(A, xs)
    G = LoopbackGroup.stencil(P, dim, nx, ny, nz, coef)
    G.set_option("method", method)
    bs = G.apply(G.split(torch.from_numpy(xs).cuda()))
    assert np.array_equal(torch.cat(bs).cpu().numpy(), b)
    res = G.solve(bs, tol=1e-10, maxit=200, gap=True)
    ref = ref_of(orc, method, A, b, tol=1e-10, maxit=200)
    check_parity(res, ref, xs)
    G.close()


def test_classic_fullsize_cfg3_first_iterations(S, orc):
    """Alg. 1 on the full 256^3 cfg3 operator (several tiles per plane, many
    chunks, the bench launch configuration): the first 3 iterations bitwise
    against the oracle."""
    st = problems.configs()["cfg3"].stencil
    solver, A, xs, b, b_d = stencil_case(S, orc, st.dim, st.nx, st.ny, st.nz, st.coef)
    solver.set_option("bench", 1)
    solver.set_option("method", 1)
    res = solver.solve(b_d, tol=0.0, maxit=3, gap=True)
    ref = orc.bicgstab(A, b, tol=0.0, maxit=3, bench=True)
    check_parity(res, ref, xs)


def _csr_case(S, orc, spd, band, n=20000, seed=1):
    """CSR band matrix; spd => symmetrised (A + A^T)/2 with the dominant diagonal
    kept (p-CG needs SPD)."""
    P = problems.csr_band(n, nnz_row=27, band=band, seed=seed)
    rp, ci, va = P.row_ptr, P.col, P.val
    if spd:
        import scipy.sparse as sp
        M = sp.csr_matrix((va, ci, rp), shape=(n, n))
        M = ((M + M.T) * 0.5).tocsr()
        M.sort_indices()
        d = np.asarray(abs(M).sum(axis=1)).ravel()
        M.setdiag(0)
        M.eliminate_zeros()
        M = (M + sp.diags(1.2 * np.asarray(abs(M).sum(axis=1)).ravel() + 1.0)).tocsr()
        M.sort_indices()
        rp, ci, va = M.indptr.astype(np.int64), M.indices.astype(np.int32), M.data
    solver = S.csr(n, rp, ci, va)
    A = orc.csr(rp, ci, va)
    xs = problems.x_star(n, 0)
    b_d = solver.apply(torch.from_numpy(xs).cuda())
    b = orc.spmv(A, xs)
    assert np.array_equal(b_d.cpu().numpy(), b)
    return solver, A, xs, b, b_d, (rp, ci, va)


@pytest.mark.parametrize("band", [500, 6000])  # window SpMV / gather SpMV
@pytest.mark.parametrize("method", [1, 2])
def test_methods_csr_parity(S, orc, method, band):
    solver, A, xs, b, b_d, _ = _csr_case(S, orc, method == 2, band)
    solver.set_option("method", method)
    res = solver.solve(b_d, tol=1e-12, maxit=200, gap=True)
    ref = ref_of(orc, method, A, b, tol=1e-12, maxit=200)
    assert res.outcome == ref.outcome
    check_parity(res, ref, xs)


def test_methods_csr_ragged_rows_bench(S, orc):
    """Stencil written out as CSR (3-5 entries per row), 300 fixed iterations."""
    A0 = orc.stencil_csr(2, 23, 19, 1, problems.poisson2d_coef())
    solver = S.csr(A0.n, A0.rp, A0.ci.astype(np.int32), A0.va)
    xs = problems.x_star(A0.n, 1)
    b_d = solver.apply(torch.from_numpy(xs).cuda())
    b = orc.spmv(A0, xs)
    solver.set_option("bench", 1)
    for method in (1, 2):
        solver.set_option("method", method)
        res = solver.solve(b_d, tol=0.0, maxit=300, gap=True)
        ref = ref_of(orc, method, A0, b, tol=0.0, maxit=300, bench=True)
        check_parity(res, ref, xs, bitwise=False)
        k = np.nonzero(ref.rnorm < 1e-16 * ref.rnorm[0])[0]
        k = int(k[0]) if k.size else ref.iters + 1
        assert np.array_equal(res.rnorm[:k], ref.rnorm[:k])


@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("method", [1, 2])
def test_methods_csr_loopback(S, orc, P, method):
    from paper_1809_01948_b200.binding import LoopbackGroup
    n = 3 * 8192
    solver, A, xs, b, b_d, (rp, ci, va) = _csr_case(S, orc, method == 2, 1000, n=n)
    solver.close()
    cuts = [n * r // P for r in range(P + 1)]
    blocks = []
    for r in range(P):
        lo, hi = cuts[r], cuts[r + 1]
        blocks.append((lo, rp[lo:hi + 1] - rp[lo], ci[rp[lo]:rp[hi]], va[rp[lo]:rp[hi]]))
    G = LoopbackGroup.csr(blocks, n)
    G.set_option("method", method)
    overlap_runs = []
    for ov in (1, 0):
        G.set_option("overlap", ov)
        bs = G.apply(G.split(torch.from_numpy(xs).cuda()))
        res = G.solve(bs, tol=1e-12, maxit=150, gap=True)
        ref = ref_of(orc, method, A, b, tol=1e-12, maxit=150)
        check_parity(res, ref, xs)
        overlap_runs.append(res)
    assert np.array_equal(overlap_runs[0].rnorm, overlap_runs[1].rnorm)
    G.close()
