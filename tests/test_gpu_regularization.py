"""gen_regularization (problems.py:100-128) with device solves: the lambda2
bisection on solution density, restated from the reference's
tests/test_problems.py:84-104, plus the CLI's ``--lambda2 auto-nnz=F``
(cli.py:91-108) end to end.

Tolerance: the density of the returned solution is within +-20% of the target
(the reference's rel_window).
"""

import numpy as np
import pytest

import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import cli

pytestmark = pytest.mark.gpu


def test_trivial_targets(cuda):
    data = pb.gen_sparse_glm(60, 15, 0.4, 4)
    lam1, lam2 = pb.gen_regularization(data, 1.0, solve=None)
    assert lam1 == pytest.approx(1.0 / 60)
    assert lam2 == 0.0


@pytest.mark.parametrize("solver", ["fista", "sps"])
def test_bisection_hits_target_density(cuda, solver):
    data = pb.gen_sparse_glm(100, 30, 0.3, 12)
    part = pb.singleton_partition(30)

    def solve(l1, l2):
        loss = pb.Loss("logistic", l1)
        if solver == "fista":
            return pb.run_fista(data, loss, pb.L1Penalty(l2), part, max_iters=150).final_x
        cfg = pb.SolverConfig(step_size="1/5L", epochs=100, seed=0)
        return pb.run_sequential(data, loss, pb.L1Penalty(l2), part, cfg).final_x

    target = 0.2
    lam1, lam2 = pb.gen_regularization(data, target, solve)
    frac = np.count_nonzero(solve(lam1, lam2)) / 30
    assert abs(frac - target) <= 0.2 * target + 1e-12
    assert 0 < lam2 < pb.lambda_max(data)


def test_cli_auto_nnz(cuda, tmp_path, capsys):
    """sparsesaga solve --lambda2 auto-nnz=0.2: the bisection's 100-epoch probes
    and the final solve all run on the device; the reported solution has the
    target density."""
    argv = ["solve", "--synthetic", "100,30,0.3,12", "--penalty", "l1", "--lambda2", "auto-nnz=0.2",
            "--epochs", "100", "--step", "1/5L", "--trace-out", str(tmp_path / "t.csv")]
    assert cli.main(argv) == cli.EXIT_OK
    out = capsys.readouterr().out
    assert "final objective" in out
    import json

    meta = json.loads((tmp_path / "t.json").read_text())
    lam2 = float(meta["penalty"].split("lam2=")[1].rstrip(")"))
    data = pb.gen_sparse_glm(100, 30, 0.3, 12)
    tr = pb.run_sequential(data, pb.Loss("logistic", 1.0 / 100), pb.L1Penalty(lam2), pb.singleton_partition(30),
                           pb.SolverConfig(step_size="1/5L", epochs=100, seed=0))
    frac = np.count_nonzero(tr.final_x) / 30
    assert abs(frac - 0.2) <= 0.2 * 0.2 + 1e-12
