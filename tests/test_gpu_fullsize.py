"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times
(TMA tile sweeps / window SpMV, CUDA graphs, bench mode), against the oracle run
on the same full-size inputs for the first iterations (the GPU box has the RAM
for the 512^3 oracle: ~35 GB for a few iterations).
"""
import numpy as np
import pytest

from paper_1809_01948_b200 import problems

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _compare(res, ref, xs):
    assert res.iters == ref.iters and res.outcome == ref.outcome
    k = min(30, ref.iters)
    rel = np.abs(res.rnorm[:k + 1] - ref.rnorm[:k + 1]) / ref.rnorm[:k + 1]
    assert rel.max() <= 1e-9, rel.max()
    x = res.x.cpu().numpy()
    e = np.linalg.norm(x - xs) / np.linalg.norm(xs)
    e0 = np.linalg.norm(ref.x - xs) / np.linalg.norm(xs)
    assert e <= 10 * e0 + 1e-15
    # design target: bitwise
    assert np.array_equal(res.rnorm, ref.rnorm)
    assert np.array_equal(x, ref.x)
    if res.gap is not None:
        assert np.array_equal(res.gap, ref.gap)


def test_cfg4_full_size_first_iterations(orc):
    from paper_1809_01948_b200 import Solver
    st = problems.configs()["cfg4"].stencil
    S = Solver.stencil(st.dim, st.nx, st.ny, st.nz, st.coef)
    xs = problems.x_star(st.n, 0)
    b_d = S.apply(torch.from_numpy(xs).cuda())
    S.set_option("bench", 1)
    # 4 iterations, replacement at i = 1 and 3 (rr_period 2), gap tracking on
    res = S.solve(b_d, tol=0.0, maxit=4, rr_period=2, gap=True)
    A = orc.stencil_csr(st.dim, st.nx, st.ny, st.nz, st.coef)
    b = orc.spmv(A, xs)
    assert np.array_equal(b_d.cpu().numpy(), b)  # SpMV, 134M rows, bitwise
    del b_d
    ref = orc.pbicgstab(A, b, tol=0.0, maxit=4, rr_period=2, bench=True)
    _compare(res, ref, xs)
    assert res.gap[0] == 0.0 and res.gap[2] == 0.0 and res.gap[4] == 0.0


def test_cfg5_full_size_solve(orc):
    """cfg5 (CSR band N = 2^23, 27 nnz/row): the normal-mode solve to 1e-10
    (converges in ~8 iterations, so the period-100 replacement never fires)."""
    from paper_1809_01948_b200 import Solver
    cfg = problems.configs()["cfg5"]
    M = problems.csr_band(cfg.csr_n, nnz_row=27, band=4096, seed=1)
    S = Solver.csr(M.n, M.row_ptr, M.col, M.val)
    xs = problems.x_star(M.n, 0)
    b_d = S.apply(torch.from_numpy(xs).cuda())
    res = S.solve(b_d, tol=cfg.tol, maxit=cfg.maxit, rr_period=cfg.rr_period, gap=True)
    A = orc.csr(M.row_ptr, M.col, M.val)
    b = orc.spmv(A, xs)
    assert np.array_equal(b_d.cpu().numpy(), b)
    ref = orc.pbicgstab(A, b, tol=cfg.tol, maxit=cfg.maxit, rr_period=cfg.rr_period)
    assert ref.outcome == "converged"
    _compare(res, ref, xs)


def test_cfg5_full_size_block_jacobi_and_gap(orc):
    """cfg5 at full size with block Jacobi b = 2 (the TMA chunk-ring sweeps with
    shuffle-gathered blocks) in bench mode, replacement every 3 iterations and the
    window-SpMV gap kernel: 8 iterations bitwise."""
    from paper_1809_01948_b200 import Solver
    cfg = problems.configs()["cfg5"]
    M = problems.csr_band(cfg.csr_n, nnz_row=27, band=4096, seed=1)
    S = Solver.csr(M.n, M.row_ptr, M.col, M.val, block=2)
    xs = problems.x_star(M.n, 0)
    b_d = S.apply(torch.from_numpy(xs).cuda())
    S.set_option("bench", 1)
    res = S.solve(b_d, tol=0.0, maxit=8, rr_period=3, gap=True)
    A = orc.csr(M.row_ptr, M.col, M.val)
    b = orc.spmv(A, xs)
    ref = orc.pbicgstab(A, b, tol=0.0, maxit=8, rr_period=3, bench=True, block=2)
    _compare(res, ref, xs)


def test_cfg4_full_size_split_schedule(orc):
    """cfg4 at full size on the paper's split schedule (option schedule 2: TMA
    chunk-ring point-wise sweeps, stand-alone SpMV tiles with the 6-slot ring):
    3 iterations with a replacement, bitwise."""
    from paper_1809_01948_b200 import Solver
    st = problems.configs()["cfg4"].stencil
    S = Solver.stencil(st.dim, st.nx, st.ny, st.nz, st.coef)
    xs = problems.x_star(st.n, 0)
    b_d = S.apply(torch.from_numpy(xs).cuda())
    S.set_option("bench", 1)
    S.set_option("schedule", 2)
    res = S.solve(b_d, tol=0.0, maxit=3, rr_period=2, gap=False)
    del b_d
    A = orc.stencil_csr(st.dim, st.nx, st.ny, st.nz, st.coef)
    b = orc.spmv(A, xs)
    ref = orc.pbicgstab(A, b, tol=0.0, maxit=3, rr_period=2, bench=True, gap=False)
    _compare(res, ref, xs)



@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_converged_full_size_vs_golden(name):
    """BASELINE cfg2 (2D 1024^2, tol 1e-10, ~2000 iterations) and cfg3 (3D 256^3,
    tol 1e-10, replacement every 50, ~510 iterations) solved to convergence at full
    size in bench.py's launch configuration (tile sweeps, CUDA graphs), against the
    oracle's converged solve of the same inputs stored in tests/golden/fullsize_*.json
    by scripts/make_golden_fullsize.py (which calls only oracle/).  The north-star
    bars (||r_i|| within 1e-9 over the first 30, iterations +-2, error within 10x) and
    the design target: bitwise ||r_i|| and gap histories over the whole solve and
    bitwise x (sha256 of its bytes)."""
    import hashlib
    import json
    import os
    from paper_1809_01948_b200 import Solver
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", f"fullsize_{name}.json")))
    cfg = problems.configs()[name]
    st = cfg.stencil
    assert g["n"] == st.n and g["tol"] == cfg.tol and g["rr_period"] == cfg.rr_period
    S = Solver.stencil(st.dim, st.nx, st.ny, st.nz, st.coef)
    xs = problems.x_star(st.n, g["x_star_seed"])
    b_d = S.apply(torch.from_numpy(xs).cuda())
    res = S.solve(b_d, tol=cfg.tol, maxit=cfg.maxit, rr_period=cfg.rr_period, gap=True)
    rn = np.array([float.fromhex(h) for h in g["rnorm_hex"]])
    gp = np.array([float.fromhex(h) for h in g["gap_hex"]])
    k = min(30, g["iters"], res.iters)
    assert np.max(np.abs(res.rnorm[:k + 1] / rn[:k + 1] - 1)) <= 1e-9
    assert abs(res.iters - g["iters"]) <= 2 and res.outcome == g["outcome"]
    x = res.x.cpu().numpy()
    err = np.linalg.norm(x - xs) / np.linalg.norm(xs)
    assert err <= 10 * g["err"]
    assert res.iters == g["iters"]
    assert np.array_equal(res.rnorm, rn), "rnorm history not bitwise"
    assert np.array_equal(res.gap, gp), "gap history not bitwise"
    assert hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest() == g["x_sha256"], \
        "x not bitwise"
    S.close()
