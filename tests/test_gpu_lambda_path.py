"""λ-path (config 5 generator, scaled down) on the GPU: the device solver
in deterministic mode reproduces the oracle per lambda (<= 1e-9), the async
path reaches the deterministic objectives, and sparsity grows along the path."""

import numpy as np
import pytest

import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import lambda_path as lp
from paper_1707_06468_b200 import problems

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cfg5():
    return problems.config5(seed=1, n=4000, p=200_000)


def test_group_lambda_max_zeroes_the_solution(cuda, cfg5):
    d, part, loss = cfg5["data"], cfg5["partition"], cfg5["loss"]
    lam_max = pb.group_lambda_max(d, part)
    solve = lp.device_solver(d, loss, part, epochs=20, mode="deterministic")
    assert solve(1.01 * lam_max)["nnz"] == 0
    assert solve(0.5 * lam_max)["nnz"] > 0


def test_deterministic_path_matches_oracle(cuda, cfg5):
    from oracle import oracle as O

    d, part, loss = cfg5["data"], cfg5["partition"], cfg5["loss"]
    lams = lp.lambda_grid(pb.group_lambda_max(d, part), 4, 1e-2)
    solve = lp.device_solver(d, loss, part, epochs=3, mode="deterministic", keep_x=True)
    res = lp.run_path(lams, solve)
    seq = pb.worker_rng(0, 0).integers(0, d.n_samples, size=3 * d.n_samples)
    for r in res:
        P = O.from_dataset(d, loss, pb.GroupL2Penalty(r["lam"]), part)
        x, _, _ = P.run_sequential(solve.gamma, seq)
        rel = np.max(np.abs(r["x"] - x)) / max(np.max(np.abs(x)), 1e-300)
        assert rel <= 1e-9, (r["lam"], rel)
        assert r["objective"] == pytest.approx(P.objective(x), rel=1e-12)


def test_async_path_reaches_deterministic_objectives(cuda, cfg5):
    d, part, loss = cfg5["data"], cfg5["partition"], cfg5["loss"]
    lams = lp.lambda_grid(pb.group_lambda_max(d, part), 3, 1e-2)
    det = lp.run_path(lams, lp.device_solver(d, loss, part, epochs=200, mode="deterministic"))
    asy = lp.run_path(lams, lp.device_solver(d, loss, part, epochs=200, mode="async", ctas=8, warps_per_cta=4))
    for a, b in zip(asy, det):
        assert abs(a["objective"] - b["objective"]) <= 1e-6 * abs(b["objective"]), (a, b)
    assert det[0]["nnz"] <= det[-1]["nnz"]


def test_forks_are_independent_states(cuda, cfg5):
    """DeviceProblem.fork: forks share the CSR and layout but not the state.
    Deterministic replays of different lambdas run on their own streams at
    the same time reproduce the serial replays bitwise."""
    import torch

    d, part, loss = cfg5["data"], cfg5["partition"], cfg5["loss"]
    lams = lp.lambda_grid(pb.group_lambda_max(d, part), 3, 1e-2)
    solve = lp.device_solver(d, loss, part, epochs=1, mode="async")
    dp, gamma, n = solve.problem, solve.gamma, d.n_samples
    seq = pb.worker_rng(4, 0).integers(0, n, size=2 * n)
    serial = []
    for lam in lams:
        dp.lam2 = lam
        dp.reset_state()
        dp.replay(seq, gamma)
        serial.append(dp.x())
    forks = [dp] + [dp.fork() for _ in range(len(lams) - 1)]
    streams = [torch.cuda.Stream() for _ in forks]
    s_dev = torch.from_numpy(seq).to(dp.device)
    for f, st, lam in zip(forks, streams, lams):
        f.lam2 = lam
        f.reset_state(stream=st)
        f.replay(s_dev, gamma, stream=st)
    torch.cuda.synchronize()
    for f, x in zip(forks, serial):
        assert np.array_equal(f.x(), x)
    assert forks[1].coord.data_ptr() != forks[0].coord.data_ptr()
    assert forks[1].col.data_ptr() == forks[0].col.data_ptr()  # CSR shared


def test_concurrent_path_matches_serial_objectives(cuda, cfg5):
    """The concurrent schedule (forks on streams, lane kernel) and the serial
    one agree within their duality-gap certificates: both objectives are
    >= F* and each is within its own gap of F*, so they differ by at most the
    larger gap."""
    d, part, loss = cfg5["data"], cfg5["partition"], cfg5["loss"]
    lams = lp.lambda_grid(pb.group_lambda_max(d, part), 6, 1e-1)
    serial = lp.run_path(lams, lp.device_solver(d, loss, part, epochs=200, mode="async"))
    conc = lp.run_path(lams, lp.device_solver(d, loss, part, epochs=200, mode="async", concurrent=6))
    for a, b in zip(serial, conc):
        assert a["gap"] >= -1e-12 and b["gap"] >= -1e-12
        tol = max(a["gap"], b["gap"]) + 1e-9 * abs(a["objective"])
        assert abs(a["objective"] - b["objective"]) <= tol, (a["lam"], a["objective"], a["gap"], b["objective"],
                                                             b["gap"])


def test_regularization_path_defaults_to_the_batched_kernel(cuda, cfg5):
    """regularization_path (the public config-5 driver) runs this rank's
    lambdas through the lambda-batched kernel by default; its objectives agree
    with the one-lambda-at-a-time group kernel schedule (batched=0) within each
    other's certified gaps + 1e-6, and sparsity grows along the path."""
    d, part, loss = cfg5["data"], cfg5["partition"], cfg5["loss"]
    auto = lp.regularization_path(d, loss, part, n_lambdas=5, ratio=1e-2, epochs=150, seed=1)
    serial = lp.regularization_path(d, loss, part, n_lambdas=5, ratio=1e-2, epochs=150, seed=1, batched=0)
    assert auto["lambdas"] == serial["lambdas"] and len(auto["results"]) == 5
    assert all(r["seconds"] == auto["results"][0]["seconds"] for r in auto["results"])  # one batched call
    for a, b in zip(auto["results"], serial["results"]):
        tol = 1e-6 * abs(b["objective"]) + max(a["gap"], 0.0) + max(b["gap"], 0.0)
        assert abs(a["objective"] - b["objective"]) <= tol, (a["lam"], a["objective"], b["objective"])
        assert a["gap"] >= -1e-12
    nnz = [r["nnz"] for r in auto["results"]]
    assert nnz[0] <= nnz[-1]
