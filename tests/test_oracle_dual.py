"""Duality gap, oracle side (CPU): the numpy restatement of the Fenchel dual
that ps_dual_objective evaluates on the device.  The reference has no dual
(parity unpinned), so it is pinned by the two properties that define it:
weak duality P(x) >= D(theta(x)) at any x, and a vanishing gap at the optimum
(strong duality; theta(x*) is the dual optimum)."""

import numpy as np
import pytest

import paper_1707_06468_b200 as pb
from oracle import oracle as O

CASES = ["cfg1", "acc_l1", "grp_random", "grp_contig", "box_sq", "zero_sq", "single_block", "l1_ragged"]


@pytest.mark.parametrize("name", CASES)
def test_weak_duality_at_random_points(name, small_cases):
    case = small_cases[name]
    P = O.from_dataset(case["data"], case["loss"], case["penalty"], case["partition"])
    rng = np.random.default_rng(3)
    for scale in (0.0, 0.01, 0.3):
        x = scale * rng.standard_normal(P.p)
        if P.penalty == "box":
            x = np.clip(x, P.lo, P.hi)
        prim, dual = P.objective(x), P.dual_objective(x)
        assert dual <= prim + 1e-12 * max(1.0, abs(prim)), (scale, prim, dual)


@pytest.mark.parametrize("name", ["acc_l1", "grp_contig", "box_sq", "zero_sq", "cfg1"])
def test_gap_vanishes_at_the_optimum(name, small_cases):
    case = small_cases[name]
    P = O.from_dataset(case["data"], case["loss"], case["penalty"], case["partition"])
    L = P.lipschitz()
    gamma = 1.0 / (3.0 * L)
    x, _, _ = P.run_sequential(gamma, O.sample_sequence(1, P.n, 3000 * P.n))
    prim, dual = P.objective(x), P.dual_objective(x)
    assert prim - dual >= -1e-12
    assert prim - dual <= 1e-8 * max(1.0, abs(prim)), (prim, dual, prim - dual)


def test_logistic_conjugate_fenchel_young():
    """l(z) + l*(l'(z)) = l'(z) z for the logistic loss (the identity the dual uses)."""
    P = O.OracleProblem([0, 1], [0], [1.0], [1.0], 1, loss="logistic", lambda1=1.0, penalty="zero")
    for z in (-3.0, -0.2, 0.0, 0.7, 5.0):
        prim = P.objective(np.array([z]))            # l(z) + z^2 / 2
        dual = P.dual_objective(np.array([z]))       # -l*(s) - v^2 / 2, v = -s
        t = 1.0 / (1.0 + np.exp(z))                  # s = -t
        assert np.isclose(prim - dual, np.log1p(np.exp(-z)) + 0.5 * z * z + (t * np.log(t) + (1 - t) * np.log1p(-t))
                          + 0.5 * t * t)
