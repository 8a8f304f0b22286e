"""Regression tests for defects found after round 1.

1. Create-time upload race.  build_csr zero-filled
   the ghosted dinv buffer with cudaMemsetAsync on the handle's stream and then
   filled it with a plain cudaMemcpy on the legacy default stream.  With a
   non-blocking handle stream the two are unordered, so the zero-fill could land
   after the copy: M^-1 = 0 in part of the rows, and the solve stalls at maxit
   (fuzz case test_fuzz_csr_loopback[318]: P = 3, Jacobi, band 8).  The tests make
   the race deterministic: the caller's non-blocking stream is kept busy with a
   long queue of work when the handle is created on it, so a zero-fill enqueued
   there runs only after any legacy-stream copy has finished.  Every create-time
   write now goes through the handle's stream (pbicgstab.cu `upload`).
"""
import numpy as np
import pytest

from paper_1809_01948_b200 import problems

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from test_gpu_parity import check_parity  # noqa: E402


def _busy(stream, ms_target=30):
    """Queue roughly ms_target milliseconds of HBM traffic on `stream`."""
    with torch.cuda.stream(stream):
        buf = torch.empty(1 << 27, dtype=torch.float64, device="cuda")  # 1 GiB
        for _ in range(max(1, ms_target // 1)):
            buf.mul_(1.0)
    return buf


def _band_blocks(M, sizes):
    cuts = np.concatenate([[0], np.cumsum(sizes)])
    return [(int(cuts[r]), M.row_ptr[cuts[r]:cuts[r + 1] + 1] - M.row_ptr[cuts[r]],
             M.col[M.row_ptr[cuts[r]]:M.row_ptr[cuts[r + 1]]],
             M.val[M.row_ptr[cuts[r]]:M.row_ptr[cuts[r + 1]]]) for r in range(len(sizes))]


@pytest.mark.parametrize("block", [1, 2, 8])
def test_csr_create_on_busy_stream(orc, block):
    """Single-rank CSR created on a busy non-blocking stream: the Jacobi / block
    inverse uploads must not be overtaken by the workspace zero-fill."""
    from paper_1809_01948_b200 import Solver
    n = 4096 + 96
    M = problems.csr_band(n, nnz_row=9, band=8, seed=7)
    A = orc.csr(M.row_ptr, M.col, M.val)
    xs = problems.x_star(n, 7)
    b = orc.spmv(A, xs)
    ref = orc.pbicgstab(A, b, tol=1e-12, maxit=60, block=block)
    s = torch.cuda.Stream()
    for trial in range(3):
        keep = _busy(s)
        S = Solver.csr(n, M.row_ptr, M.col, M.val, stream=s, block=block)
        S.set_option("csr_tma", trial % 2)
        with torch.cuda.stream(s):
            b_d = torch.from_numpy(b).to("cuda", non_blocking=False)
            s.synchronize()
            res = S.solve(b_d, tol=1e-12, maxit=60, rr_period=0, gap=True)
        del keep
        assert res.outcome == ref.outcome, (trial, res.outcome, ref.outcome)
        check_parity(res, ref, xs, bitwise=True)
        S.close()


@pytest.mark.parametrize("transport", [0, 1])
def test_csr_loopback_create_on_busy_stream(orc, transport):
    """The failing fuzz configuration (P = 3, Jacobi, half bandwidth 8, per-row
    sweeps, overlap on), created on a busy stream, bitwise vs the oracle."""
    from paper_1809_01948_b200.binding import LoopbackGroup
    rng = np.random.default_rng(318)
    sizes = [int(rng.integers(4096, 4096 + 3000)) for _ in range(3)]
    n = sum(sizes)
    M = problems.csr_band(n, nnz_row=9, band=8, seed=318)
    A = orc.csr(M.row_ptr, M.col, M.val)
    xs = problems.x_star(n, 318)
    b = orc.spmv(A, xs)
    ref = orc.pbicgstab(A, b, tol=1e-12, maxit=60, rr_period=3)
    s = torch.cuda.Stream()
    for trial in range(3):
        keep = _busy(s)
        G = LoopbackGroup.csr(_band_blocks(M, sizes), n, stream=s)
        del keep
        G.set_option("transport", transport)
        G.set_option("csr_tma", 0)
        G.set_option("overlap", 1)
        bs = G.split(torch.from_numpy(b).cuda())
        torch.cuda.synchronize()
        res = G.solve(bs, tol=1e-12, maxit=60, rr_period=3, gap=True)
        assert res.outcome == ref.outcome, (trial, res.outcome, ref.outcome)
        check_parity(res, ref, xs, bitwise=True)
        G.close()


def test_csr_loopback_many_handles_back_to_back(orc):
    """Create / solve / destroy the failing configuration many times in one
    process (the fuzz history the defect depended on), bitwise every time."""
    from paper_1809_01948_b200.binding import LoopbackGroup
    for seed in range(40):
        rng = np.random.default_rng(9000 + seed)
        sizes = [int(rng.integers(4096, 4096 + 3000)) for _ in range(3)]
        n = sum(sizes)
        M = problems.csr_band(n, nnz_row=int(rng.integers(3, 10)), band=8, seed=seed)
        A = orc.csr(M.row_ptr, M.col, M.val)
        xs = problems.x_star(n, seed)
        b = orc.spmv(A, xs)
        G = LoopbackGroup.csr(_band_blocks(M, sizes), n)
        G.set_option("transport", seed % 2)
        G.set_option("csr_tma", 0)
        bs = G.apply(G.split(torch.from_numpy(xs).cuda()))
        assert np.array_equal(torch.cat(bs).cpu().numpy(), b)
        res = G.solve(bs, tol=1e-12, maxit=40, rr_period=0, gap=True)
        ref = orc.pbicgstab(A, b, tol=1e-12, maxit=40)
        assert res.outcome == ref.outcome, (seed, res.outcome, ref.outcome)
        check_parity(res, ref, xs, bitwise=True)
        G.close()
