"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
vectors (tests/golden/ref_small.npz, produced by the unmodified reference).

Tolerances (written here, per BASELINE.json north_star):
  * deterministic fp64 iterates: max|x_gpu - x_ref| / max|x_ref| <= 1e-9
    (observed ~1e-15: the only differences are summation order of the
    margin / block norms);
  * objective / fixed-point residual / gradient: 1e-12 relative;
  * block counts n_B, weights d_B, delta: exact.
"""

import numpy as np
import pytest

import paper_1707_06468_b200 as pb
from paper_1707_06468_b200.device import DeviceProblem
from paper_1707_06468_b200.saga import resolve_step_size, worker_rng

pytestmark = pytest.mark.gpu

DET_TOL = 1e-9

CASES = ["cfg1", "acc_l1", "grp_random", "l1_blocks", "grp_contig", "grp_g1", "box_sq", "zero_sq",
         "single_block", "l1_ragged", "grp_ragged_contig", "cfg2_small", "cfg5_small"]


def _dp(case):
    return DeviceProblem(case["data"], case["loss"], case["penalty"], case["partition"],
                         drop_dead_blocks=case["drop_dead"])


def _gamma(case, dp):
    mu = case["loss"].lambda1
    return resolve_step_size(case["step"], dp.L, dp.n, mu if mu > 0 else None)


@pytest.mark.parametrize("name", CASES)
def test_deterministic_replay_matches_reference(cuda, name, small_cases, golden_small):
    case, g = small_cases[name], golden_small
    dp = _dp(case)
    gamma = _gamma(case, dp)
    assert gamma == pytest.approx(float(g[f"{name}__gamma"]), rel=1e-14)
    assert dp.delta == pytest.approx(float(g[f"{name}__delta"]), rel=1e-15)
    counts, weights, _ = dp.block_stats()
    assert np.array_equal(counts, g[f"{name}__nB"])
    assert np.array_equal(weights, g[f"{name}__dB"])
    seq = worker_rng(case["seed"], 0).integers(0, dp.n, size=case["steps"])
    done = 0
    for k, s in enumerate(case["segments"]):
        dp.replay(seq[done:s], gamma)
        done = s
        ref = g[f"{name}__x"][k]
        x = dp.x()
        rel = np.max(np.abs(x - ref)) / max(np.max(np.abs(ref)), 1e-300)
        assert rel <= DET_TOL, f"{name} segment {k}: rel {rel:.3e}"
        assert dp.objective() == pytest.approx(float(g[f"{name}__obj"][k]), rel=1e-12)
    alpha = dp.alpha.cpu().numpy()
    assert np.max(np.abs(alpha - g[f"{name}__alpha"])) <= DET_TOL * max(1.0, np.max(np.abs(alpha)))
    assert np.max(np.abs(dp.abar() - g[f"{name}__abar"])) <= DET_TOL
    res = dp.fixed_point_residual(gamma)
    assert res == pytest.approx(float(g[f"{name}__residual"]), rel=1e-8, abs=1e-13)
    assert np.allclose(dp.smooth_gradient_of(dp.x()), g[f"{name}__grad"], rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("name", ["cfg1", "acc_l1", "grp_contig", "grp_g1", "box_sq", "l1_ragged",
                                  "grp_ragged_contig", "cfg2_small", "cfg5_small"])
def test_deterministic_replay_through_hot_layout(cuda, name, small_cases, golden_small):
    """Same parity with the hot-unit layout forced on (columns / whole blocks
    renumbered and strided, rows re-sorted, coordinates padded to whole units)."""
    case, g = small_cases[name], golden_small
    dp = DeviceProblem(case["data"], case["loss"], case["penalty"], case["partition"],
                       drop_dead_blocks=case["drop_dead"], hot_min_rows=0, hot_max=64, hot_stride=4)
    assert dp.perm is not None and dp.H > 0
    gamma = _gamma(case, dp)
    counts, weights, _ = dp.block_stats()
    assert np.array_equal(counts, g[f"{name}__nB"])
    assert np.array_equal(weights, g[f"{name}__dB"])
    seq = worker_rng(case["seed"], 0).integers(0, dp.n, size=case["steps"])
    done = 0
    for k, s in enumerate(case["segments"]):
        dp.replay(seq[done:s], gamma)
        done = s
        ref = g[f"{name}__x"][k]
        rel = np.max(np.abs(dp.x() - ref)) / max(np.max(np.abs(ref)), 1e-300)
        assert rel <= DET_TOL, f"{name} segment {k}: rel {rel:.3e}"
        assert dp.objective() == pytest.approx(float(g[f"{name}__obj"][k]), rel=1e-12)
    assert np.max(np.abs(dp.abar() - g[f"{name}__abar"])) <= DET_TOL
    assert dp.fixed_point_residual(gamma) == pytest.approx(float(g[f"{name}__residual"]), rel=1e-8, abs=1e-13)
    assert np.allclose(dp.smooth_gradient_of(dp.x()), g[f"{name}__grad"], rtol=1e-12, atol=1e-15)


def test_run_sequential_api_matches_reference_trace(cuda, small_cases, golden_small):
    """saga.py:217-259 contract on the acceptance instance (3 epochs, seed 2)."""
    case = small_cases["acc_l1"]
    pen = pb.L1Penalty(float(golden_small["acc__lam2"]))
    tr = pb.run_sequential(case["data"], case["loss"], pen, case["partition"], pb.SolverConfig(epochs=3, seed=2))
    assert tr.iterations == list(golden_small["acc__seq3_it"])
    ref = golden_small["acc__seq3_x"]
    assert np.max(np.abs(tr.final_x - ref)) / np.max(np.abs(ref)) <= DET_TOL
    assert np.allclose(tr.objective, golden_small["acc__seq3_obj"], rtol=1e-12)


def test_sequential_precision_criterion_4(cuda, small_cases, golden_small):
    """test_acceptance.py:67-73: suboptimality <= 1e-10 after 150 epochs."""
    case = small_cases["acc_l1"]
    pen = pb.L1Penalty(float(golden_small["acc__lam2"]))
    tr = pb.run_sequential(case["data"], case["loss"], pen, case["partition"],
                           pb.SolverConfig(step_size="1/5L", epochs=150, seed=0))
    assert tr.objective[-1] - float(golden_small["acc__fstar"]) <= 1e-10
    assert np.allclose(tr.objective, golden_small["acc__seq150_obj"], rtol=1e-11)


def test_single_warp_async_equals_sequential_bitwise(cuda, small_cases, golden_small):
    """test_async.py:105-112: one worker replays the sequential solver exactly."""
    case = small_cases["acc_l1"]
    pen = pb.L1Penalty(float(golden_small["acc__lam2"]))
    seq = pb.run_sequential(case["data"], case["loss"], pen, case["partition"], pb.SolverConfig(epochs=3, seed=2))
    par = pb.run_async(case["data"], case["loss"], pen, case["partition"],
                       pb.AsyncConfig(epochs=3, seed=2, threads=1))
    assert np.array_equal(seq.final_x, par.final_x)
    assert par.iterations[-1] == 3 * case["data"].n_samples


@pytest.mark.parametrize("warps", [2, 64, None])
def test_async_converges_to_reference_optimum(cuda, small_cases, golden_small, warps):
    """test_async.py:122-126 / test_acceptance.py:76-98 (C5): many warps, <= 1e-8."""
    case = small_cases["acc_l1"]
    pen = pb.L1Penalty(float(golden_small["acc__lam2"]))
    fstar = float(golden_small["acc__fstar"])
    worst = 0.0
    for seed in range(3):
        tr = pb.run_async(case["data"], case["loss"], pen, case["partition"],
                          pb.AsyncConfig(step_size="1/5L", epochs=120, seed=seed, threads=2, warps=warps))
        worst = max(worst, tr.objective[-1] - fstar)
        assert tr.iterations[-1] == 120 * case["data"].n_samples
    assert worst <= 1e-8, worst


def test_async_average_stays_consistent(cuda, small_cases, golden_small):
    """test_async.py:129-136: abar == A^T alpha / n after a many-warp run (<1e-12)."""
    case = small_cases["acc_l1"]
    pen = pb.L1Penalty(float(golden_small["acc__lam2"]))
    tr = pb.run_async(case["data"], case["loss"], pen, case["partition"],
                      pb.AsyncConfig(epochs=10, seed=0, threads=4))
    dp = tr.device_problem
    live = dp.abar()
    dp.resync_average()
    exact = dp.abar()
    assert np.max(np.abs(live - exact)) < 1e-12


@pytest.mark.parametrize("name", ["grp_random", "grp_contig", "cfg5_small", "box_sq", "l1_ragged"])
def test_async_other_penalties_converge(cuda, name, small_cases, golden_small):
    """Many-warp async on group / box / long-row layouts approaches the
    deterministic solution (objective within 1e-6 relative of a long
    deterministic device run)."""
    case = small_cases[name]
    dp = _dp(case)
    gamma = _gamma(case, dp)
    n = dp.n
    epochs = max(300, 60000 // n)
    seq = worker_rng(99, 0).integers(0, n, size=epochs * n)
    dp.replay(seq, gamma)
    fref = dp.objective()
    dp.reset_state()
    dp.run_async(epochs * n, gamma, seed=5, batch=8, ctas=2, warps_per_cta=2)
    f = dp.objective()
    assert abs(f - fref) <= 1e-6 * abs(fref), (f, fref)


def test_device_prox_known_answers(cuda, golden_small):
    """test_penalties.py:28-48 golden prox values on the device prox."""
    g = golden_small
    assert np.allclose(pb.L1Penalty(1.0).prox(g["ka__l1_in"], 1.0), g["ka__l1_out"], atol=0)
    assert np.allclose(pb.GroupL2Penalty(1.0).prox_block(g["ka__grp_in"], 1.0), g["ka__grp_out1"], rtol=1e-15)
    assert np.array_equal(pb.GroupL2Penalty(1.0).prox_block(g["ka__grp_in"], 6.0), g["ka__grp_out6"])
    assert np.array_equal(pb.BoxPenalty(-1.0, 2.0).prox(g["ka__box_in"], 0.7), g["ka__box_out"])
    assert np.array_equal(pb.L1Penalty(0.7).prox(g["ka__sep_v"], g["ka__sep_eff"]), g["ka__sep_l1"])
    assert np.array_equal(pb.BoxPenalty(-0.5, 1.5).prox(g["ka__sep_v"], g["ka__sep_eff"]), g["ka__sep_box"])
    assert np.allclose(pb.GroupL2Penalty(0.7).prox_block(g["ka__grp_v"], 2.3), g["ka__grp_v_out"], rtol=1e-14)
    v = np.array([1.0, -2.0])
    out = pb.ZeroPenalty().prox(v, 3.0)
    assert np.array_equal(out, v) and out is not v


def test_support_index_known_answer(cuda, golden_small):
    """test_data.py:151-161 through the device column-statistics kernel."""
    m = pb.CsrMatrix(3, 3, np.array([0, 2, 3, 6]), np.array([0, 2, 1, 0, 1, 2]),
                     np.array([0.5, -2.0, 1.5, 1.0, 2.0, 3.0]))
    idx = pb.build_support_index(m, pb.singleton_partition(3))
    assert np.array_equal(idx.n_B, golden_small["ka__small_nB"])
    assert np.allclose(idx.d_B, golden_small["ka__small_dB"])
    assert idx.delta == pytest.approx(float(golden_small["ka__small_delta"]))
    assert np.allclose(idx.coord_weights(), 1.5)


def test_dead_blocks_raise_unless_dropped(cuda):
    """data.py:255-257."""
    m = pb.CsrMatrix(2, 4, np.array([0, 1, 2]), np.array([0, 2]), np.array([1.0, 2.0]))
    with pytest.raises(pb.DeadBlockError) as e:
        pb.build_support_index(m, pb.singleton_partition(4))
    assert e.value.block_ids == [1, 3]
    idx = pb.build_support_index(m, pb.singleton_partition(4), drop_dead_blocks=True)
    assert list(idx.dropped_blocks) == [1, 3] and idx.d_B[1] == 0.0


def test_one_dimensional_analytic_fixed_point(cuda):
    """test_saga.py:106-128 on the device."""
    feats = pb.CsrMatrix(1, 1, np.array([0, 1]), np.array([0]), np.array([1.0]))
    data = pb.Dataset(features=feats, labels=np.array([2.0]))
    loss, pen = pb.Loss("squared", 0.0), pb.L1Penalty(0.6)
    tr = pb.run_sequential(data, loss, pen, pb.singleton_partition(1), pb.SolverConfig(epochs=400, seed=0))
    assert tr.final_x[0] == pytest.approx(1.4, abs=1e-10)
    idx = pb.build_support_index(feats, pb.singleton_partition(1))
    assert pb.fixed_point_residual(np.array([1.4]), data, loss, pen, idx, 0.3) < 1e-14
    assert pb.fixed_point_residual(np.array([0.0]), data, loss, pen, idx, 0.3) > 0.1


def test_checkpoint_cadence_and_tolerance(cuda, small_cases, tmp_path):
    """test_saga.py:131-151."""
    case = small_cases["acc_l1"]
    d = case["data"]
    tr = pb.run_sequential(d, case["loss"], case["penalty"], case["partition"],
                           pb.SolverConfig(epochs=2, seed=0, checkpoint_every=100))
    assert tr.iterations == list(range(0, 2 * d.n_samples + 1, 100))
    tr.to_csv(tmp_path / "t.csv")
    assert (tmp_path / "t.csv").read_text().splitlines()[0] == "iterations,epochs,objective,wall_seconds"
    tr.write_sidecar(tmp_path / "t.json")
    assert "sparse-saga" in (tmp_path / "t.json").read_text()
    tr2 = pb.run_sequential(d, case["loss"], case["penalty"], case["partition"],
                            pb.SolverConfig(epochs=200, seed=0, tolerance=1e-6))
    assert tr2.iterations[-1] < 200 * d.n_samples


def test_lambda_max_matches_reference_formula(cuda, small_cases):
    """problems.py:94-97: max |A^T(-b/2)| / n."""
    d = small_cases["acc_l1"]["data"]
    A = d.features.toarray()
    expect = np.max(np.abs(A.T @ (-0.5 * d.labels))) / d.n_samples
    assert pb.lambda_max(d) == pytest.approx(expect, rel=1e-13)


@pytest.mark.parametrize("flags", [0, 128, 128 | 262144, 32],
                         ids=["warp_per_block", "lane_per_block", "lane_store_zeros", "delta_zero"])
@pytest.mark.parametrize("name", ["grp_contig", "cfg5_small"])
def test_async_group_kernels_converge(cuda, name, flags, small_cases, golden_small):
    """The group-lasso async kernels (the warp-cooperative default, the
    lane-per-block one with and without PS_FLAG_GROUP_STORE_ZEROS, and the
    reference's literal delta commit of zeroed blocks) reach the deterministic solution within 1e-6 relative (grp_contig
    has a ragged last block: p = 103, G = 10)."""
    case = small_cases[name]
    dp = _dp(case)
    gamma = _gamma(case, dp)
    n = dp.n
    epochs = max(300, 60000 // n)
    seq = worker_rng(99, 0).integers(0, n, size=epochs * n)
    dp.replay(seq, gamma)
    fref = dp.objective()
    dp.reset_state()
    dp.run_async(epochs * n, gamma, seed=5, flags=flags)
    f = dp.objective()
    assert abs(f - fref) <= 1e-6 * abs(fref), (f, fref)


@pytest.mark.parametrize("name", ["cfg1", "acc_l1", "grp_random", "grp_contig", "box_sq", "zero_sq", "single_block",
                                  "l1_ragged", "cfg2_small", "cfg5_small"])
def test_dual_objective_matches_oracle(cuda, name, small_cases, golden_small):
    """ps_dual_objective (device) == the oracle's numpy restatement at the
    same x (the deterministic iterate after its replay), <= 1e-10 relative;
    weak duality holds (gap >= 0)."""
    from oracle import oracle as O

    case = small_cases[name]
    dp = _dp(case)
    gamma = _gamma(case, dp)
    n = dp.n
    dp.replay(worker_rng(3, 0).integers(0, n, size=5 * n), gamma)
    x = dp.x()
    P = O.from_dataset(case["data"], case["loss"], case["penalty"], case["partition"])
    d_ref = P.dual_objective(x)
    prim, dual, gap = dp.duality_gap()
    assert dual == pytest.approx(d_ref, rel=1e-10, abs=1e-13), (dual, d_ref)
    assert gap >= -1e-12 * max(1.0, abs(prim))
