"""The lambda-batched group-lasso kernel (ps_batch_run, csrc/batch.cu): B
solves of one problem sharing each sampled row.

Tolerances:
  * deterministic replay: every state equals the single-lambda deterministic
    replay of the same sample sequence (which matches the reference's
    iterates, tests/test_gpu_parity.py) to 1e-9 relative, and the reference's
    golden iterates where the golden case's lambda is used;
  * asynchronous: each state's objective within 1e-6 relative of that
    lambda's optimum (a long deterministic replay; 1e-5 below 0.01 lambda_max,
    where the replay itself is not converged and the asynchronous iterate
    fluctuates at the 1e-6 level), abar = A^T alpha / n per state to 1e-12.
"""

import numpy as np
import pytest

import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems
from paper_1707_06468_b200.device import DeviceProblem
from paper_1707_06468_b200.lambda_path import BatchedPath, device_solver
from paper_1707_06468_b200.saga import resolve_step_size, worker_rng

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.mark.parametrize("B", [4, 16])
def test_batched_deterministic_replay_matches_single_lambda(cuda, B, small_cases, golden_small):
    case, g = small_cases["grp_contig"], golden_small
    data, loss, part = case["data"], case["loss"], case["partition"]
    lam0 = case["penalty"].lam2
    lams = [lam0 * f for f in (1.0, 0.5, 0.2, 0.05, 2.0, 0.1, 0.01, 1.5)][:B] + [lam0] * max(0, B - 8)
    bp = BatchedPath(data, loss, part, B=B)
    gamma = resolve_step_size(case["step"], bp.dp.L, bp.dp.n, loss.lambda1)
    seq = worker_rng(case["seed"], 0).integers(0, data.n_samples, size=case["segments"][0])
    bp.reset(lams)
    bp.run(0, gamma, samples=seq)
    for beta, lam in enumerate(lams):
        dp = DeviceProblem(data, loss, pb.GroupL2Penalty(lam), part, drop_dead_blocks=True, hot_max=0)
        dp.replay(seq, gamma)
        x = bp.field(beta).cpu().numpy()
        assert _rel(x, dp.x()) <= 1e-9, (beta, lam)
        assert _rel(bp.field(beta, 1).cpu().numpy(), dp.abar()) <= 1e-9
        a = bp.alpha.view(-1, B)[:, beta].cpu().numpy()
        assert np.max(np.abs(a - dp.alpha.cpu().numpy())) <= 1e-9
        if lam == lam0:  # the reference's own iterate (tests/golden, make_golden.py)
            assert _rel(x, g["grp_contig__x"][0]) <= 1e-9


@pytest.fixture
def tune2():
    """ps_batch_tune2 with the defaults restored afterwards."""
    from paper_1707_06468_b200 import _lib

    def set_(nhot, hstride, hshare, hab):
        _lib.check(_lib.load().ps_batch_tune2(nhot, hstride, hshare, hab))

    yield set_
    set_(-1, 128, 4, -1)


@pytest.mark.parametrize("B,factors,nrep,layout", [
    (8, (0.5, 0.2, 0.1, 0.05, 0.03, 0.02, 0.01, 0.005), 0, None), (2, (0.3, 0.01), 0, None), (16, (0.5, 0.01), 0, None),
    (8, (0.5, 0.2, 0.1, 0.05, 0.03, 0.02, 0.01, 0.005), 4, None), (2, (0.3, 0.01), 8, None),
    (4, (0.5, 0.1, 0.03, 0.01), 0, (-1, 128, 0, 64)), (4, (0.5, 0.1, 0.03, 0.01), 0, (0, 0, 0, 0)),
    (4, (0.5, 0.1, 0.03, 0.01), 0, (-1, 128, 4, 0))],
    ids=["B8", "B2", "B16", "B8rep", "B2rep", "B4noshare", "B4contiguous", "B4packed"])
def test_batched_async_reaches_each_optimum(cuda, tune2, B, factors, nrep, layout):
    """Spread block layout with the scattered hot blocks of the state (the
    default: no replicas), and the opt-in replicated x-delta accumulators of the
    hottest blocks (ps_batch_run_rep, folded after the launch).  Layout variants
    (ps_batch_tune2): every row loading stored block 0 itself (no CTA-shared
    copy), every block in the contiguous record (no scattered hot blocks), and
    hot slots with one packed (x, abar) sector."""
    if layout is not None:
        tune2(*layout)
    rng = np.random.default_rng(11)
    data = problems._zipf_logistic(rng, 8000, 40000, 20, 1.1, 100)
    part = pb.contiguous_partition(data.n_features, 10)
    lam1 = 1.0 / data.n_samples
    loss = pb.Loss("logistic", lam1)
    lmax = pb.group_lambda_max(data, part)
    lams = [f * lmax for f in factors]
    solve = device_solver(data, loss, part, epochs=60, seed=3, batched=B, nrep=nrep, nrb=16 if nrep else 0)
    res = solve.batch(lams)
    bp = solve.batched
    assert bp.dp.perm is not None  # spread layout
    assert bp.nrep == nrep and BatchedPath.AUTO_NREP[B] == 0
    n = data.n_samples
    for beta, (lam, r) in enumerate(zip(lams, res)):
        dp = DeviceProblem(data, loss, pb.GroupL2Penalty(lam), part, drop_dead_blocks=True, hot_max=0)
        gamma = resolve_step_size("1/2L", dp.L, n, lam1)
        dp.replay(worker_rng(99, 0).integers(0, n, size=150 * n), gamma)
        fref = dp.objective()
        # 1e-6 of the optimum; at lambda < 0.01 lambda_max this instance's asynchronous iterate
        # hovers in a +-1e-6..3e-6 band (spikes to 7e-6) around the 150-epoch replay, which is
        # itself not converged there (negative differences occur) -- measured the same for the
        # contiguous, scattered and shared-load layouts (tools/gpu/exp_batch_share_conv.py)
        tol = 1e-6 if lam >= 0.0099 * lmax else 1e-5
        assert abs(r["objective"] - fref) <= tol * abs(fref), (lam / lmax, r["objective"], fref)
        assert r["gap"] >= -1e-12 and r["objective"] >= r["dual"]
        # abar stays the exact average of this state's alpha table
        dp.alpha.copy_(bp.alpha.view(-1, B)[:, beta])
        dp.resync_average()
        assert np.max(np.abs(bp.field(beta, 1).cpu().numpy() - dp.abar())) <= 1e-12


def test_run_async_group_lasso_runs_the_batched_kernel(cuda):
    """run_async (asynchronous.py:131-210) with a group penalty on contiguous
    blocks goes through the lambda-batched kernel with one state: one trace row
    per epoch, the replay optimum within 1e-6, the final x / abar / alpha in the
    problem's records (abar the exact average of alpha); AsyncConfig
    (group_batched=False) keeps the coordinate-record group kernel."""
    rng = np.random.default_rng(11)
    data = problems._zipf_logistic(rng, 8000, 40000, 20, 1.1, 100)
    part = pb.contiguous_partition(data.n_features, 10)
    lam1 = 1.0 / data.n_samples
    loss = pb.Loss("logistic", lam1)
    pen = pb.GroupL2Penalty(0.1 * pb.group_lambda_max(data, part))
    index = pb.build_support_index(data.features, part, drop_dead_blocks=True)
    n, epochs = data.n_samples, 40
    ref = DeviceProblem(data, loss, pen, part, drop_dead_blocks=True, hot_max=0)
    gamma = resolve_step_size("1/2L", ref.L, n, lam1)
    ref.replay(worker_rng(99, 0).integers(0, n, size=150 * n), gamma)
    fref = ref.objective()
    tr = pb.run_async(data, loss, pen, part, pb.AsyncConfig(step_size="1/2L", epochs=epochs, seed=2, threads=2),
                      index=index)
    assert tr.meta["kernel"].startswith("lambda-batched") and tr.meta["warps_in_flight"] >= 16
    assert len(tr.iterations) == epochs + 1 and tr.iterations[-1] == epochs * n
    assert abs(tr.objective[-1] - fref) <= 1e-6 * abs(fref), (tr.objective[-1], fref)
    dp = tr.shared
    assert abs(dp.objective() - tr.objective[-1]) <= 1e-15 * abs(fref)  # the records hold the final state
    assert abs(ref.objective_of(tr.final_x) - tr.objective[-1]) <= 1e-12 * abs(fref)
    live = dp.abar()
    dp.resync_average()
    assert np.max(np.abs(live - dp.abar())) <= 1e-12
    tr2 = pb.run_async(data, loss, pen, part,
                       pb.AsyncConfig(step_size="1/2L", epochs=epochs, seed=2, threads=2, group_batched=False),
                       index=index)
    assert "kernel" not in tr2.meta and len(tr2.iterations) == epochs + 1
    assert abs(tr2.objective[-1] - fref) <= 1e-6 * abs(fref), (tr2.objective[-1], fref)
