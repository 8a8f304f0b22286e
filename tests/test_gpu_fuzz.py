"""Seeded randomised parity sweep (GPU vs oracle) over the option space: random
grid shapes (2D/3D, odd and even nx, tiny extents), random diagonally dominant
coefficient sets, random solver / replacement / graph / tile / loopback-rank
choices and random CSR band matrices with Jacobi or block Jacobi.  Every case
must meet the north-star bars, and -- above the noise floor -- be bitwise equal.
"""
import os

import numpy as np
import pytest

from paper_1809_01948_b200 import problems

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from test_gpu_parity import check_parity, noise_floor_parity  # noqa: E402

# PBICG_FUZZ_SCALE=k runs k times the cases (a wider sweep than the default suite)
SCALE = int(os.environ.get("PBICG_FUZZ_SCALE", "1"))
# PBICG_FUZZ_OFFSET=j shifts every seed by j * 100000 (independent wide sweeps)
OFFSET = 100000 * int(os.environ.get("PBICG_FUZZ_OFFSET", "0"))
N_CASES = 24 * SCALE


def rand_coef(rng, dim, spd):
    off = -rng.uniform(0.2, 2.0, 6)
    if dim == 2:
        off[4:] = 0.0
    if spd:  # symmetric: -x = +x, -y = +y, -z = +z
        off[1], off[3], off[5] = off[0], off[2], off[4]
    c0 = np.abs(off).sum() * rng.uniform(1.0, 1.5)
    return [float(c0)] + [float(o) for o in off]


def _rank0(S):
    """The handle whose scalar trace a (loopback) solve left: rank 0's."""
    return S.ranks[0] if hasattr(S, "ranks") else S


@pytest.mark.parametrize("seed", range(N_CASES))
def test_fuzz_stencil(orc, seed):
    from paper_1809_01948_b200 import Solver
    from paper_1809_01948_b200.binding import LoopbackGroup
    rng = np.random.default_rng(1000 + seed + OFFSET)
    dim = int(rng.choice([2, 3]))
    nx = int(rng.integers(1, 70))
    ny = int(rng.integers(1, 40))
    nz = int(rng.integers(1, 25)) if dim == 3 else 1
    method = int(rng.choice([0, 0, 1, 2]))
    coef = rand_coef(rng, dim, spd=(method == 2))
    A = orc.stencil_csr(dim, nx, ny, nz, coef)
    xs = problems.x_star(A.n, seed)
    b = orc.spmv(A, xs)
    auto = method == 0 and bool(rng.integers(0, 2))
    rr = int(rng.choice([0, 2, 5, 9])) if method == 0 and not auto else 0
    maxit = int(rng.integers(5, 80))
    tol = float(rng.choice([0.0, 1e-8, 1e-11]))
    outer = nz if dim == 3 else ny
    P = int(rng.choice([1, 1, 2, 3])) if outer >= 3 else 1
    if P == 1:
        S = Solver.stencil(dim, nx, ny, nz, coef)
        S.set_option("graphs", int(rng.integers(0, 2)))
        if not auto and method == 0:
            tile = int(rng.integers(0, 2))
            S.set_option("tile", tile)
            if tile and rng.integers(0, 3) == 0:  # the paper's split schedule
                S.set_option("schedule", 2)
        S.set_option("pdl", int(rng.integers(0, 2)))
        S.set_option("method", method)
        S.set_option("rr_auto", int(auto))
        S.set_option("bench", int(tol == 0.0))
        b_d = S.apply(torch.from_numpy(xs).cuda())
        assert np.array_equal(b_d.cpu().numpy(), b)
        if rng.integers(0, 2):  # a nonzero initial guess
            x0 = rng.uniform(-1, 1, A.n)
            x0_kw = dict(x0=x0)
            res = S.solve(b_d, x0=torch.from_numpy(x0).cuda(), tol=tol, maxit=maxit,
                          rr_period=rr, gap=True)
        else:
            x0_kw = {}
            res = S.solve(b_d, tol=tol, maxit=maxit, rr_period=rr, gap=True)
    else:
        S = LoopbackGroup.stencil(P, dim, nx, ny, nz, coef)
        S.set_option("transport", int(rng.integers(0, 2)))
        S.set_option("method", method)
        S.set_option("rr_auto", int(auto))
        S.set_option("bench", int(tol == 0.0))
        bs = S.apply(S.split(torch.from_numpy(xs).cuda()))
        res = S.solve(bs, tol=tol, maxit=maxit, rr_period=rr, gap=True)
        x0_kw = {}
    kw = dict(tol=tol, maxit=maxit, bench=tol == 0.0, **x0_kw)
    if method == 0:
        ref = orc.pbicgstab(A, b, rr_period=rr, auto_rr=auto, want_scalars=True, **kw)
    elif method == 1:
        ref = orc.bicgstab(A, b, **kw)
    else:
        ref = orc.pipecg(A, b, **kw)
    assert res.outcome == ref.outcome, (res.outcome, ref.outcome)
    rerun = lambda m: orc.pbicgstab(A, b, rr_period=rr, auto_rr=auto, want_trace=True,
                                    **dict(kw, maxit=m))
    noise_floor_parity(_rank0(S) if method == 0 else None, res, ref, xs, tag=f" stencil[{seed}]",
                       rerun=rerun)
    S.close()


@pytest.mark.parametrize("seed", range(12 * SCALE))
def test_fuzz_csr(orc, seed):
    from paper_1809_01948_b200 import Solver
    rng = np.random.default_rng(2000 + seed + OFFSET)
    block = int(rng.choice([1, 1, 2, 4, 8, 16, 32]))
    n = int(rng.integers(64, 400)) * 32
    bw = int(rng.choice([8, 100, 1000, 5000]))
    nnz = int(rng.integers(3, 28))
    M = problems.csr_band(n, nnz_row=min(nnz, bw + 1), band=bw, seed=seed)  # edge rows: bw candidates
    A = orc.csr(M.row_ptr, M.col, M.val)
    S = Solver.csr(n, M.row_ptr, M.col, M.val, block=block)
    S.set_option("csr_tma", int(rng.integers(0, 2)))
    method = int(rng.choice([0, 0, 1]))
    S.set_option("method", method)
    auto = method == 0 and bool(rng.integers(0, 2))
    S.set_option("rr_auto", int(auto))
    rr = int(rng.choice([0, 2, 5])) if method == 0 and not auto else 0
    xs = problems.x_star(n, seed)
    b_d = S.apply(torch.from_numpy(xs).cuda())
    b = orc.spmv(A, xs)
    assert np.array_equal(b_d.cpu().numpy(), b)
    res = S.solve(b_d, tol=1e-12, maxit=60, rr_period=rr, gap=True)
    if method == 0:
        ref = orc.pbicgstab(A, b, tol=1e-12, maxit=60, rr_period=rr, auto_rr=auto, block=block,
                            want_scalars=True)
    else:
        ref = orc.bicgstab(A, b, tol=1e-12, maxit=60, block=block)
    assert res.outcome == ref.outcome
    rerun = lambda m: orc.pbicgstab(A, b, tol=1e-12, maxit=m, rr_period=rr, auto_rr=auto,
                                    block=block, want_trace=True)
    noise_floor_parity(S if method == 0 else None, res, ref, xs, tag=f" csr[{seed}]", rerun=rerun)
    S.close()


@pytest.mark.parametrize("seed", range(8 * SCALE))
def test_fuzz_wide_grids(orc, seed):
    """nx > 1024 (x-segmented tiles for even nx, line kernels for odd nx), random
    solver / replacement options, bitwise above the noise floor."""
    from paper_1809_01948_b200 import Solver
    rng = np.random.default_rng(3000 + seed + OFFSET)
    dim = int(rng.choice([2, 3]))
    nx = int(rng.integers(1025, 2400))
    ny = int(rng.integers(1, 12))
    nz = int(rng.integers(1, 6)) if dim == 3 else 1
    method = int(rng.choice([0, 0, 1])) if nx % 2 == 0 else 0
    coef = rand_coef(rng, dim, spd=False)
    A = orc.stencil_csr(dim, nx, ny, nz, coef)
    xs = problems.x_star(A.n, seed)
    b = orc.spmv(A, xs)
    S = Solver.stencil(dim, nx, ny, nz, coef)
    S.set_option("method", method)
    rr = int(rng.choice([0, 3, 6])) if method == 0 else 0
    b_d = S.apply(torch.from_numpy(xs).cuda())
    assert np.array_equal(b_d.cpu().numpy(), b)
    res = S.solve(b_d, tol=1e-11, maxit=60, rr_period=rr, gap=True)
    ref = (orc.pbicgstab(A, b, tol=1e-11, maxit=60, rr_period=rr, want_scalars=True)
           if method == 0 else orc.bicgstab(A, b, tol=1e-11, maxit=60))
    assert res.outcome == ref.outcome
    noise_floor_parity(S if method == 0 else None, res, ref, xs, tag=f" wide[{seed}]")
    S.close()


@pytest.mark.parametrize("seed", range(8 * SCALE))
def test_fuzz_csr_loopback(orc, seed):
    """Random CSR band matrices split over P emulated ranks at random row cuts (each
    rank >= PBICG_CSR_HALO rows, any parity), Jacobi or block Jacobi, random solver,
    transport, TMA sweeps on/off and replacement."""
    from paper_1809_01948_b200.binding import LoopbackGroup
    rng = np.random.default_rng(4000 + seed + OFFSET)
    P = int(rng.choice([2, 3]))
    block = int(rng.choice([1, 1, 2, 4, 8]))
    halo = 4096
    sizes = [int(rng.integers(halo, halo + 3000)) for _ in range(P)]
    sizes = [sz - sz % block for sz in sizes]
    n = sum(sizes)
    bw = int(rng.choice([8, 100, 1001, 4000]))
    M = problems.csr_band(n, nnz_row=min(int(rng.integers(3, 28)), bw + 1), band=bw,
                          seed=seed)
    A = orc.csr(M.row_ptr, M.col, M.val)
    cuts = np.concatenate([[0], np.cumsum(sizes)])
    blocks = [(int(cuts[r]), M.row_ptr[cuts[r]:cuts[r + 1] + 1] - M.row_ptr[cuts[r]],
               M.col[M.row_ptr[cuts[r]]:M.row_ptr[cuts[r + 1]]],
               M.val[M.row_ptr[cuts[r]]:M.row_ptr[cuts[r + 1]]]) for r in range(P)]
    G = LoopbackGroup.csr(blocks, n, block=block)
    method = int(rng.choice([0, 0, 1]))
    G.set_option("method", method)
    G.set_option("transport", int(rng.integers(0, 2)))
    G.set_option("csr_tma", int(rng.integers(0, 2)))
    G.set_option("overlap", int(rng.integers(0, 2)))
    auto = method == 0 and bool(rng.integers(0, 2))
    G.set_option("rr_auto", int(auto))
    rr = int(rng.choice([0, 3, 7])) if method == 0 and not auto else 0
    xs = problems.x_star(n, seed)
    b = orc.spmv(A, xs)
    bs = G.apply(G.split(torch.from_numpy(xs).cuda()))
    res = G.solve(bs, tol=1e-12, maxit=60, rr_period=rr, gap=True)
    if method == 0:
        ref = orc.pbicgstab(A, b, tol=1e-12, maxit=60, rr_period=rr, block=block,
                            auto_rr=auto, want_scalars=True)
    else:
        ref = orc.bicgstab(A, b, tol=1e-12, maxit=60, block=block)
    assert res.outcome == ref.outcome
    rerun = lambda m: orc.pbicgstab(A, b, tol=1e-12, maxit=m, rr_period=rr, block=block,
                                    auto_rr=auto, want_trace=True)
    noise_floor_parity(G.ranks[0] if method == 0 else None, res, ref, xs,
                       tag=f" csr_loopback[{seed}]", rerun=rerun)
    G.close()


@pytest.mark.parametrize("seed", range(8 * SCALE))
def test_fuzz_stencil_block_jacobi(orc, seed):
    """Random stencils with x-aligned block Jacobi b = 2 / 4 / 8 (per-leg form and
    the transform stage), 1 or P emulated ranks, random transport and replacement."""
    from paper_1809_01948_b200 import Solver
    from paper_1809_01948_b200.binding import LoopbackGroup
    rng = np.random.default_rng(5000 + seed + OFFSET)
    block = int(rng.choice([2, 4, 8]))
    dim = int(rng.choice([2, 3]))
    nx = block * int(rng.integers(1, 840 // block if dim == 3 else 1024 // block))
    ny = int(rng.integers(1, 30 if dim == 3 else 60))
    nz = int(rng.integers(1, 12)) if dim == 3 else 1
    coef = rand_coef(rng, dim, spd=False)
    A = orc.stencil_csr(dim, nx, ny, nz, coef)
    if A.n > 400000:
        pytest.skip("oracle size")
    xs = problems.x_star(A.n, seed)
    b = orc.spmv(A, xs)
    outer = nz if dim == 3 else ny
    P = int(rng.choice([1, 2, 3])) if outer >= 3 else 1
    rr = int(rng.choice([0, 4, 9]))
    if P == 1:
        S = Solver.stencil(dim, nx, ny, nz, coef, block=block)
        bs = S.apply(torch.from_numpy(xs).cuda())
    else:
        S = LoopbackGroup.stencil(P, dim, nx, ny, nz, coef, block=block)
        S.set_option("transport", int(rng.integers(0, 2)))
        bs = S.apply(S.split(torch.from_numpy(xs).cuda()))
    res = S.solve(bs, tol=1e-11, maxit=60, rr_period=rr, gap=True)
    ref = orc.pbicgstab(A, b, tol=1e-11, maxit=60, rr_period=rr, block=block, want_scalars=True)
    assert res.outcome == ref.outcome
    noise_floor_parity(_rank0(S), res, ref, xs, tag=f" stencil_bj[{seed}]")
    S.close()



@pytest.mark.parametrize("seed", range(8 * SCALE))
def test_fuzz_stencil_block_jacobi_methods(orc, seed):
    """Classic BiCGStab and p-CG with stencil block Jacobi b = 2 / 4 / 8 (the derived
    operands' transform stage, the lane-shuffled M^-1 of streamed vectors), 1 or P
    emulated ranks, random transport, bench or tolerance mode."""
    from paper_1809_01948_b200 import Solver
    from paper_1809_01948_b200.binding import LoopbackGroup
    rng = np.random.default_rng(7000 + seed + OFFSET)
    block = int(rng.choice([2, 4, 8]))
    method = int(rng.choice([1, 2]))
    dim = int(rng.choice([2, 3]))
    nx = block * int(rng.integers(1, 840 // block if dim == 3 else 1024 // block))
    ny = int(rng.integers(1, 30 if dim == 3 else 60))
    nz = int(rng.integers(1, 12)) if dim == 3 else 1
    coef = rand_coef(rng, dim, spd=(method == 2))
    A = orc.stencil_csr(dim, nx, ny, nz, coef)
    if A.n > 400000:
        pytest.skip("oracle size")
    xs = problems.x_star(A.n, seed)
    b = orc.spmv(A, xs)
    outer = nz if dim == 3 else ny
    P = int(rng.choice([1, 2, 3])) if outer >= 3 else 1
    tol = float(rng.choice([0.0, 1e-11]))
    maxit = int(rng.integers(5, 60))
    if P == 1:
        S = Solver.stencil(dim, nx, ny, nz, coef, block=block)
        S.set_option("graphs", int(rng.integers(0, 2)))
        bs = S.apply(torch.from_numpy(xs).cuda())
    else:
        S = LoopbackGroup.stencil(P, dim, nx, ny, nz, coef, block=block)
        S.set_option("transport", int(rng.integers(0, 2)))
        bs = S.apply(S.split(torch.from_numpy(xs).cuda()))
    S.set_option("method", method)
    S.set_option("bench", int(tol == 0.0))
    res = S.solve(bs, tol=tol, maxit=maxit, rr_period=0, gap=True)
    fn = orc.bicgstab if method == 1 else orc.pipecg
    ref = fn(A, b, tol=tol, maxit=maxit, bench=tol == 0.0, block=block)
    assert res.outcome == ref.outcome
    noise_floor_parity(None, res, ref, xs, tag=f" stencil_bj_m{method}[{seed}]")
    S.close()
