"""GPU vs oracle on exact breakdowns (reading A9; systems pinned in rationals by
tests/test_oracle_breakdown.py): the outcome, the iteration count, the history and
the returned iterate must be the oracle's bitwise, for p-BiCGStab and classic
BiCGStab, on one rank, on the one-rank NCCL path, with and without CUDA graphs."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from test_oracle_breakdown import BD_ALPHA0, BD_DEN, dense_csr  # noqa: E402


@pytest.mark.parametrize("case", ["alpha0", "den"])
@pytest.mark.parametrize("method", [0, 1])
@pytest.mark.parametrize("graphs", [0, 1])
@pytest.mark.parametrize("nccl", [0, 1])
def test_exact_breakdown_parity(orc, case, method, graphs, nccl):
    from paper_1809_01948_b200 import Solver
    from paper_1809_01948_b200 import binding as B
    D, xs = {"alpha0": BD_ALPHA0, "den": BD_DEN}[case]
    b = D @ xs
    A = dense_csr(orc, D)
    d = B.make_dist(1, 0, B.nccl_unique_id(), B.nccl_unique_id()) if nccl else None
    S = Solver.csr(A.n, A.rp, A.ci.astype(np.int32), A.va, dist=d)
    S.set_option("method", method)
    S.set_option("graphs", graphs)
    S.set_option("bench", 1)
    res = S.solve(torch.from_numpy(b).cuda(), tol=0.0, maxit=6, gap=True)
    ref = (orc.pbicgstab if method == 0 else orc.bicgstab)(A, b, tol=0.0, maxit=6, bench=True)
    assert ref.outcome == "breakdown"
    assert (res.outcome, res.iters) == (ref.outcome, ref.iters)
    assert np.array_equal(res.rnorm, ref.rnorm)
    assert np.array_equal(res.gap, ref.gap)
    assert np.array_equal(res.x.cpu().numpy(), ref.x)
    S.close()


def test_classic_cfg5_bench_breakdown_vs_golden():
    """bench.py's classic-BiCGStab cfg5 line stops one iteration before an exact
    breakdown in the noise regime of bench mode (tol 0).  The oracle's run of the
    same inputs (tests/golden/fullsize_cfg5_classic_bench.json, written by
    scripts/make_golden_fullsize.py) fixes where: outcome, iteration, the whole
    ||r_i|| history and x bitwise."""
    import hashlib
    import json
    import os
    from paper_1809_01948_b200 import Solver, problems
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                    "fullsize_cfg5_classic_bench.json")))
    M = problems.csr_band(g["n"], nnz_row=27, band=4096, seed=1)
    S = Solver.csr(g["n"], M.row_ptr, M.col, M.val)
    S.set_option("method", 1)
    S.set_option("bench", 1)
    xs = problems.x_star(g["n"], g["x_star_seed"])
    b_d = S.apply(torch.from_numpy(xs).cuda())
    res = S.solve(b_d, tol=0.0, maxit=g["maxit"], gap=False)
    rn = np.array([float.fromhex(h) for h in g["rnorm_hex"]])
    assert (res.outcome, res.iters) == (g["outcome"], g["iters"])
    assert np.array_equal(res.rnorm, rn)
    x = res.x.cpu().numpy()
    assert hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest() == g["x_sha256"]
    S.close()
