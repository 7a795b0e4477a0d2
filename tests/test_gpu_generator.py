"""K7 device generator (configs 3/4 at full size are built this way):
structural invariants of the generated CSR, a deterministic-replay parity
check against the oracle on a generated instance, and async invariants."""

import numpy as np
import pytest

import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems

pytestmark = pytest.mark.gpu


def _host(dp):
    rp = dp.row_ptr.cpu().numpy().astype(np.int64)
    col = dp.col.cpu().numpy().astype(np.int64)
    val = dp.val.cpu().numpy().astype(np.float64)
    y = dp.y.cpu().numpy().astype(np.float64)
    return rp, col, val, y


@pytest.mark.parametrize("k_dense,k_zipf,s,lognormal", [(0, 30, 1.2, False), (13, 22, 1.05, True)])
def test_generated_rows_are_valid(cuda, k_dense, k_zipf, s, lognormal):
    c = problems.device_zipf_problem(20_000, 50_000, k_dense, k_zipf, s, 500, 1e-6, lognormal, seed=3,
                                     hot_max=0)
    dp = c["problem"]
    rp, col, val, y = _host(dp)
    k = k_dense + k_zipf
    assert np.array_equal(rp, np.arange(dp.n + 1) * k)
    rows = col.reshape(dp.n, k)
    assert np.all(np.diff(rows, axis=1) > 0)                      # strictly increasing (data.py:58-61)
    assert np.all(rows[:, :k_dense] == np.arange(k_dense))        # dense columns in every row
    assert rows.min() >= 0 and rows.max() < dp.p
    norms = np.sqrt((val.reshape(dp.n, k) ** 2).sum(axis=1))
    assert np.allclose(norms, 1.0, atol=1e-6)                     # rows l2-normalised
    assert set(np.unique(y)) <= {-1.0, 1.0}
    freq = np.bincount(col, minlength=dp.p) / dp.n
    head = freq[k_dense]                                          # first Zipf column
    assert head > 0.5                                             # the Zipf head is in most rows
    if not lognormal:
        assert np.allclose(val, 1.0 / np.sqrt(k), rtol=1e-6)


def test_generated_problem_deterministic_parity(cuda):
    from oracle import oracle as O

    c = problems.device_zipf_problem(3_000, 20_000, 13, 22, 1.05, 300, 1e-4, True, seed=5, hot_max=0)
    dp = c["problem"]
    rp, col, val, y = _host(dp)
    gamma = pb.resolve_step_size("1/2L", dp.L, dp.n, c["loss"].lambda1)
    seq = pb.worker_rng(1, 0).integers(0, dp.n, size=3 * dp.n)
    dp.replay(seq, gamma)
    P = O.OracleProblem(rp, col, val, y, dp.p, loss="logistic", lambda1=c["loss"].lambda1, penalty="l1",
                        lam2=c["penalty"].lam2)
    assert P.lipschitz() == pytest.approx(dp.L, rel=1e-14)
    x, _, _ = P.run_sequential(gamma, seq)
    rel = np.max(np.abs(dp.x() - x)) / np.max(np.abs(x))
    assert rel <= 1e-9, rel
    assert dp.objective() == pytest.approx(P.objective(x), rel=1e-12)


def test_generated_problem_async_invariants(cuda):
    c = problems.device_zipf_problem(200_000, 300_000, 0, 30, 1.2, 1_000, 1e-6, False, seed=7)
    dp = c["problem"]
    gamma = pb.resolve_step_size("1/2L", dp.L, dp.n, c["loss"].lambda1)
    f = [dp.objective()]
    for _ in range(6):
        dp.run_async(dp.n, gamma, seed=2)
        f.append(dp.objective())
    assert f[-1] < f[0] and np.isfinite(f).all()
    assert all(b <= a + 1e-3 for a, b in zip(f[2:], f[3:]))
    assert int(dp.counter.item()) == dp.n
    live = dp.abar()
    dp.resync_average()
    assert np.max(np.abs(live - dp.abar())) <= 1e-12
