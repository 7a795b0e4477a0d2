"""Device FISTA (paper_1707_06468_b200/fista.py) against
the unmodified reference's run_fista (tests/golden/ref_fista.npz, made by
tests/golden/make_fista.py): the objective trace and the final iterate;
and the cross-solver agreement the reference tests (test_acceptance.py
C9): FISTA's optimum is the SAGA solvers' optimum."""

from pathlib import Path

import numpy as np
import pytest

import paper_1707_06468_b200 as pb

pytestmark = pytest.mark.gpu

GOLD = np.load(Path(__file__).parent / "golden" / "ref_fista.npz")


@pytest.mark.parametrize("name", ["acc_l1", "grp_contig", "box_sq", "cfg1", "grp_random"])
def test_fista_matches_reference(cuda, name, small_cases):
    case = small_cases[name]
    iters = int(GOLD[f"{name}__iters"])
    tr = pb.run_fista(case["data"], case["loss"], case["penalty"], case["partition"], max_iters=iters)
    ref = GOLD[f"{name}__obj"]
    assert len(tr.objective) == len(ref)
    # identical algorithm and deterministic; only the order of the A^T s sums differs (~1e-16)
    np.testing.assert_allclose(tr.objective, ref, rtol=1e-10, atol=1e-14)
    x, xr = tr.final_x, GOLD[f"{name}__x"]
    assert np.max(np.abs(x - xr)) <= 1e-8 * max(1.0, np.max(np.abs(xr)))


def test_fista_and_saga_agree(cuda, small_cases):
    """test_acceptance.py:128-139: the optimum FISTA converges to is the one
    the asynchronous SAGA solver reaches."""
    case = small_cases["acc_l1"]
    d, loss, pen, part = case["data"], case["loss"], case["penalty"], case["partition"]
    tf = pb.run_fista(d, loss, pen, part, max_iters=3000, checkpoint_every=100)
    ts = pb.run_async(d, loss, pen, part, pb.AsyncConfig(epochs=400, seed=0, threads=4))
    assert abs(tf.objective[-1] - ts.objective[-1]) <= 1e-8 * abs(tf.objective[-1])
