"""Pin the C oracle (oracle/sps_oracle.c) to the reference's own outputs.

Golden vectors come from the unmodified reference (tests/golden/make_golden.py);
known answers are the reference tests' own (test_penalties.py:28-48,
test_data.py:151-161, test_saga.py:106-128, test_async.py:63-72,105-112).
CPU only.
"""

import numpy as np
import pytest

from oracle import oracle as O


def _oracle_for(case):
    data, loss, pen, part = case["data"], case["loss"], case["penalty"], case["partition"]
    return O.from_dataset(data, loss, pen, part)


def _gamma(case, P):
    from paper_1707_06468_b200.saga import resolve_step_size

    mu = case["loss"].lambda1
    return resolve_step_size(case["step"], P.lipschitz(), P.n, mu if mu > 0 else None)


CASES = ["cfg1", "acc_l1", "grp_random", "l1_blocks", "grp_contig", "grp_g1", "box_sq", "zero_sq",
         "single_block", "l1_ragged", "grp_ragged_contig", "cfg2_small", "cfg5_small"]


@pytest.mark.parametrize("name", CASES)
def test_oracle_replays_reference(name, small_cases, golden_small):
    case = small_cases[name]
    P = _oracle_for(case)
    g = golden_small
    gamma = _gamma(case, P)
    assert gamma == pytest.approx(float(g[f"{name}__gamma"]), rel=1e-15)
    assert P.delta == pytest.approx(float(g[f"{name}__delta"]), rel=1e-15)
    assert np.array_equal(P.counts, g[f"{name}__nB"])
    assert np.array_equal(P.d_B, g[f"{name}__dB"])
    seq = O.sample_sequence(case["seed"], P.n, case["steps"])
    x = np.zeros(P.p)
    alpha = np.zeros(P.n)
    abar = np.zeros(P.p)
    done = 0
    for k, s in enumerate(case["segments"]):
        x, alpha, abar = P.run_sequential(gamma, seq[done:s], x, alpha, abar)
        done = s
        ref = g[f"{name}__x"][k]
        scale = max(np.max(np.abs(ref)), 1e-300)
        assert np.max(np.abs(x - ref)) / scale <= 1e-12, f"segment {k}"
        assert P.objective(x) == pytest.approx(float(g[f"{name}__obj"][k]), rel=1e-12)
    assert np.max(np.abs(alpha - g[f"{name}__alpha"])) <= 1e-12 * max(1.0, np.max(np.abs(alpha)))
    assert np.max(np.abs(abar - g[f"{name}__abar"])) <= 1e-12
    assert P.fixed_point_residual(x, gamma) == pytest.approx(float(g[f"{name}__residual"]), rel=1e-8, abs=1e-14)
    assert np.allclose(P.smooth_gradient(x), g[f"{name}__grad"], rtol=1e-12, atol=1e-15)


def test_support_index_known_answer(golden_small):
    """test_data.py:151-161: n_B=[2,2,2], d=1.5, delta=2/3."""
    P = O.OracleProblem([0, 2, 3, 6], [0, 2, 1, 0, 1, 2], [0.5, -2.0, 1.5, 1.0, 2.0, 3.0], [1, -1, 1], 3)
    assert np.array_equal(P.counts, golden_small["ka__small_nB"])
    assert np.allclose(P.d_B, golden_small["ka__small_dB"])
    assert P.delta == pytest.approx(float(golden_small["ka__small_delta"]))


def test_one_dimensional_fixed_point():
    """test_saga.py:106-116: squared loss, one feature, x -> 2 - 0.6."""
    P = O.OracleProblem([0, 1], [0], [1.0], [2.0], 1, loss="squared", penalty="l1", lam2=0.6)
    gamma = 1.0 / 5.0  # 1/5L with L = 1
    x, _, _ = P.run_sequential(gamma, O.sample_sequence(0, 1, 400))
    assert x[0] == pytest.approx(1.4, abs=1e-10)
    assert P.fixed_point_residual(np.array([1.4]), 0.3) < 1e-14
    assert P.fixed_point_residual(np.array([0.0]), 0.3) > 0.1


def test_async_single_worker_equals_sequential(small_cases):
    """test_async.py:105-112 on the oracle: one worker == sequential, bitwise."""
    case = small_cases["acc_l1"]
    P = _oracle_for(case)
    gamma = _gamma(case, P)
    seq = O.sample_sequence(2, P.n, 3 * P.n)
    xs, _, _ = P.run_sequential(gamma, seq)
    xa, _, _, cnt = P.run_async(gamma, [seq])
    assert np.array_equal(xs, xa)
    assert cnt == 3 * P.n


def test_async_multi_worker_converges(small_cases, golden_small):
    """test_async.py:122-126 analogue on the oracle's pthread Hogwild port."""
    case = small_cases["acc_l1"]
    P = O.from_dataset(case["data"], case["loss"], __import__("paper_1707_06468_b200").L1Penalty(
        float(golden_small["acc__lam2"])), case["partition"])
    gamma = 1.0 / (5.0 * P.lipschitz())
    total = 60 * P.n
    counts = O.split_iterations(total, 4)
    seqs = [O.sample_sequence(1, P.n, c, worker_id=w) for w, c in enumerate(counts)]
    x, alpha, abar, cnt = P.run_async(gamma, seqs)
    assert cnt == total
    assert P.objective(x) - float(golden_small["acc__fstar"]) < 1e-6


def test_oracle_atomic_exactness():
    """verify.py:368-381: 8 threads x 1e5 CAS adds of 1.0 are exact."""
    cell = np.zeros(1)
    O.add_repeat_threads(cell, 1.0, 100_000, 8)
    assert cell[0] == 800_000.0


def test_acceptance_optimum_pins(small_cases, golden_small):
    """The oracle evaluates the reference optimum's objective identically."""
    import paper_1707_06468_b200 as pb

    case = small_cases["acc_l1"]
    P = O.from_dataset(case["data"], case["loss"], pb.L1Penalty(float(golden_small["acc__lam2"])),
                       case["partition"])
    assert P.objective(golden_small["acc__xstar"]) == pytest.approx(float(golden_small["acc__fstar"]), rel=1e-13)
    gamma = 1.0 / (5.0 * P.lipschitz())
    assert P.fixed_point_residual(golden_small["acc__xstar"], gamma) <= 1e-8
