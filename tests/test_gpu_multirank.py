"""Multi-rank path on one GPU through the loopback transport.

pbicgstab_create_*_loopback builds P handles that partition the operator exactly
as P processes would (z-/y-slabs, CSR row blocks), exchange ghost planes and the
per-rank Dot2 rows with device copies (in place of NCCL send/recv/all-reduce),
and form the scalars with the rank-order finalize kernels.  Kernels of different
ranks never wait on each other (one stream).  Results must match the oracle
(north-star bars; bitwise expected) and the single-rank run.
"""
import numpy as np
import pytest

from paper_1809_01948_b200 import problems

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def B():
    from paper_1809_01948_b200 import binding
    assert torch.cuda.is_available()
    return binding


def _parity(res, ref, xs, bitwise=True):
    k = min(30, ref.iters, res.iters)
    rel = np.abs(res.rnorm[:k + 1] - ref.rnorm[:k + 1]) / np.maximum(ref.rnorm[:k + 1], 1e-300)
    assert np.all(rel <= 1e-9), rel.max()
    assert abs(res.iters - ref.iters) <= 2
    x = res.x.cpu().numpy()
    e, e0 = (np.linalg.norm(v - xs) / np.linalg.norm(xs) for v in (x, ref.x))
    assert e <= 10 * e0 + 1e-15
    if bitwise:
        assert res.iters == ref.iters
        assert np.array_equal(res.rnorm, ref.rnorm)
        assert np.array_equal(x, ref.x)
        if res.gap is not None:
            assert np.array_equal(res.gap, ref.gap)


@pytest.mark.parametrize("P", [2, 3, 4])
@pytest.mark.parametrize("dim,nx,ny,nz", [(3, 24, 20, 17), (2, 64, 37, 1), (3, 13, 7, 9)])
@pytest.mark.parametrize("tile,overlap", [(1, 1), (0, 1), (1, 0)])
def test_loopback_stencil_matches_oracle(B, orc, P, dim, nx, ny, nz, tile, overlap):
    coef = problems.cfg34_coef() if dim == 3 else problems.cfg2_coef()
    G = B.LoopbackGroup.stencil(P, dim, nx, ny, nz, coef)
    G.set_option("tile", tile)
    G.set_option("overlap", overlap)  # reductions behind the halo exchange, or blocking
    A = orc.stencil_csr(dim, nx, ny, nz, coef)
    xs = problems.x_star(A.n, 0)
    b = orc.spmv(A, xs)
    parts = G.split(torch.from_numpy(xs).cuda())
    assert sum(s.n_local for s in G.ranks) == A.n
    bd = G.apply(parts)
    assert np.array_equal(torch.cat(bd).cpu().numpy(), b)
    for rr in (0, 5):
        res = G.solve(bd, tol=1e-11, maxit=200, rr_period=rr, gap=True)
        ref = orc.pbicgstab(A, b, tol=1e-11, maxit=200, rr_period=rr)
        assert res.outcome == ref.outcome
        _parity(res, ref, xs)
    G.close()


def test_loopback_equals_single_rank_large(B, orc):
    """A 3D problem spanning several tiles per slab, RR and gap on, graphs on."""
    dim, nx, ny, nz = 3, 96, 80, 64
    coef = problems.cfg34_coef()
    xs = problems.x_star(nx * ny * nz, 0)
    S = B.Solver.stencil(dim, nx, ny, nz, coef)
    b1 = S.apply(torch.from_numpy(xs).cuda())
    r1 = S.solve(b1, tol=1e-10, maxit=400, rr_period=50, gap=True)
    for P in (2, 4):
        G = B.LoopbackGroup.stencil(P, dim, nx, ny, nz, coef)
        bd = G.split(b1)
        rp = G.solve(bd, tol=1e-10, maxit=400, rr_period=50, gap=True)
        assert rp.iters == r1.iters and rp.outcome == r1.outcome
        rel = np.abs(rp.rnorm - r1.rnorm) / r1.rnorm
        assert rel.max() <= 1e-9
        assert np.array_equal(rp.rnorm, r1.rnorm)
        assert np.array_equal(rp.x.cpu().numpy(), r1.x.cpu().numpy())
        G.close()


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("overlap", [1, 0])
def test_loopback_csr_matches_oracle(B, orc, P, overlap):
    n = 20000
    M = problems.csr_band(n, nnz_row=27, band=500, seed=1)
    A = orc.csr(M.row_ptr, M.col, M.val)
    xs = problems.x_star(n, 0)
    b = orc.spmv(A, xs)
    cuts = np.linspace(0, n, P + 1).astype(int)
    blocks = []
    for r in range(P):
        lo, hi = cuts[r], cuts[r + 1]
        rp = M.row_ptr[lo:hi + 1] - M.row_ptr[lo]
        sl = slice(M.row_ptr[lo], M.row_ptr[hi])
        blocks.append((int(lo), rp, M.col[sl], M.val[sl]))
    G = B.LoopbackGroup.csr(blocks, n)
    G.set_option("overlap", overlap)
    bd = G.apply(G.split(torch.from_numpy(xs).cuda()))
    assert np.array_equal(torch.cat(bd).cpu().numpy(), b)
    for rr in (0, 3):
        res = G.solve(bd, tol=1e-12, maxit=100, rr_period=rr, gap=True)
        ref = orc.pbicgstab(A, b, tol=1e-12, maxit=100, rr_period=rr)
        _parity(res, ref, xs)
    G.close()


def test_partition_is_balanced_slabs(B):
    G = B.LoopbackGroup.stencil(3, 3, 10, 10, 11, problems.cfg34_coef())
    nl = [s.n_local for s in G.ranks]
    rb = [s.row_begin for s in G.ranks]
    assert nl == [400, 400, 300] and rb == [0, 400, 800]
    G.close()


@pytest.mark.parametrize("P", [2, 3, 4])
@pytest.mark.parametrize("case", ["stencil", "stencil_auto", "stencil_bj", "stencil_split",
                                  "classic", "pipecg", "csr", "csr_pipecg"])
def test_peer_memory_transport(B, orc, P, case):
    """option transport=1: the producing kernels store their rank's Dot2 pairs into
    every rank's receive buffer and the finalize kernels wait on per-rank flags
    (no collective launch).  Results are those of the copy transport (and the
    oracle), bitwise, over repeated solves (the epoch counter persists)."""
    coef = problems.cfg34_coef()
    spd = [6.0, -1, -1, -1, -1, -1, -1]
    if case.startswith("csr"):
        n = 4096 * P
        M = problems.csr_band(n, nnz_row=15, band=900, seed=3)
        rp, ci, va = M.row_ptr, M.col, M.val
        if case == "csr_pipecg":
            A0 = orc.stencil_csr(2, 64, n // 64, 1, problems.poisson2d_coef())
            rp, ci, va = A0.rp, A0.ci.astype(np.int32), A0.va
        A = orc.csr(rp, ci, va)
        cuts = [n * r // P for r in range(P + 1)]
        blocks = [(cuts[r], rp[cuts[r]:cuts[r + 1] + 1] - rp[cuts[r]], ci[rp[cuts[r]]:rp[cuts[r + 1]]],
                   va[rp[cuts[r]]:rp[cuts[r + 1]]]) for r in range(P)]
        make = lambda: B.LoopbackGroup.csr(blocks, n)
    else:
        dim, nx, ny, nz = 3, 24, 10, 13
        cf = spd if case == "pipecg" else coef
        A = orc.stencil_csr(dim, nx, ny, nz, cf)
        blk = 4 if case == "stencil_bj" else 1
        make = lambda: B.LoopbackGroup.stencil(P, dim, nx, ny, nz, cf, block=blk)
    method = {"classic": 1, "pipecg": 2, "csr_pipecg": 2}.get(case, 0)
    auto = case == "stencil_auto"
    rr = 0 if (method or auto) else 4
    xs = problems.x_star(A.n, 0)
    b = orc.spmv(A, xs)
    out = []
    for transport in (0, 1):
        G = make()
        G.set_option("method", method)
        G.set_option("rr_auto", int(auto))
        G.set_option("bench", 1)
        G.set_option("transport", transport)
        if case == "stencil_split":
            G.set_option("schedule", 2)
        bs = G.apply(G.split(torch.from_numpy(xs).cuda()))
        for rep in range(2):  # the epoch counter carries over between solves
            res = G.solve(bs, tol=0.0, maxit=60, rr_period=rr, gap=True)
        out.append(res)
        G.close()
    kw = dict(tol=0.0, maxit=60, bench=True)
    if method == 1:
        ref = orc.bicgstab(A, b, **kw)
    elif method == 2:
        ref = orc.pipecg(A, b, **kw)
    else:
        ref = orc.pbicgstab(A, b, rr_period=rr, auto_rr=auto, block=4 if case == "stencil_bj" else 1,
                            **kw)
    for res in out:
        _parity(res, ref, xs, bitwise=False)
    assert np.array_equal(out[0].rnorm, out[1].rnorm)
    assert np.array_equal(out[0].x.cpu().numpy(), out[1].x.cpu().numpy())
    assert np.array_equal(out[0].gap, out[1].gap)


@pytest.mark.parametrize("P", [1, 2, 3])
@pytest.mark.parametrize("overlap", [1, 0])
def test_split_stencil_schedule(B, orc, P, overlap):
    """option schedule=2 on a stencil: the paper's 4-phase pipeline (stand-alone
    SpMVs the reductions hide behind) gives the fused schedule's results bitwise,
    with periodic replacement, on 1 and P emulated ranks, overlap on and off."""
    dim, nx, ny, nz = 3, 20, 11, 12
    coef = problems.cfg34_coef()
    A = orc.stencil_csr(dim, nx, ny, nz, coef)
    xs = problems.x_star(A.n, 0)
    b = orc.spmv(A, xs)
    ref = orc.pbicgstab(A, b, tol=1e-11, maxit=150, rr_period=6)
    if P == 1:
        S = B.Solver.stencil(dim, nx, ny, nz, coef)
        S.set_option("schedule", 2)
        b_d = S.apply(torch.from_numpy(xs).cuda())
        res = S.solve(b_d, tol=1e-11, maxit=150, rr_period=6, gap=True)
    else:
        S = B.LoopbackGroup.stencil(P, dim, nx, ny, nz, coef)
        S.set_option("schedule", 2)
        S.set_option("overlap", overlap)
        bs = S.apply(S.split(torch.from_numpy(xs).cuda()))
        res = S.solve(bs, tol=1e-11, maxit=150, rr_period=6, gap=True)
    _parity(res, ref, xs)
    S.close()


@pytest.mark.parametrize("shape,P", [((3, 24, 13, 14), 2), ((3, 24, 13, 14), 3),
                                     ((3, 1100, 3, 3), 3),   # x-segmented tiles, 1 plane/rank
                                     ((2, 40, 30, 1), 4)])
@pytest.mark.parametrize("overlap", [1, 0])
def test_peer_halo_fused_into_sweeps(B, orc, shape, P, overlap):
    """transport 1, fused schedule: sweep A stores its boundary planes of z_i and sweep C
    of w_{i+1} straight into the neighbours' ghost planes (peer memory; loopback members
    share the address space), so the iteration enqueues no z / w halo exchange -- only
    replacement iterations (w replaced after the sweep) and the gap still exchange.
    Iterates bitwise equal to transport 0 and to the oracle above the noise floor."""
    dim, nx, ny, nz = shape
    coef = problems.cfg34_coef() if dim == 3 else problems.cfg2_coef()
    A = orc.stencil_csr(dim, nx, ny, nz, coef)
    xs = problems.x_star(A.n, 0)
    b = orc.spmv(A, xs)
    maxit, rr = 60, 7
    out, halos = [], []
    for transport in (0, 1):
        G = B.LoopbackGroup.stencil(P, dim, nx, ny, nz, coef)
        G.set_option("bench", 1)
        G.set_option("overlap", overlap)
        G.set_option("transport", transport)
        bs = G.apply(G.split(torch.from_numpy(xs).cuda()))
        G.ranks[0].kernel_time("halo", reset=True)
        res = G.solve(bs, tol=0.0, maxit=maxit, rr_period=rr, gap=False)
        halos.append(G.ranks[0].kernel_time("halo")[0])
        out.append(res)
        G.close()
    assert np.array_equal(out[0].rnorm, out[1].rnorm)
    assert np.array_equal(out[0].x.cpu().numpy(), out[1].x.cpu().numpy())
    ref = orc.pbicgstab(A, b, tol=0.0, maxit=maxit, rr_period=rr, bench=True, gap=False)
    _parity(out[1], ref, xs, bitwise=False)
    k = np.nonzero(ref.rnorm < 1e-16 * ref.rnorm[0])[0]
    k = int(k[0]) if k.size else maxit + 1
    assert np.array_equal(out[1].rnorm[:k], ref.rnorm[:k])
    # two exchanges per iteration fewer, except the w halo of replacement iterations
    n_rr = maxit // rr
    assert halos[0] - halos[1] == 2 * maxit - n_rr, halos

