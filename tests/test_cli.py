"""The command-line routing (paper_1707_06468_b200/cli.py), modelled on the
reference's test_cli.py: exit-code contract (cli.py:36-39), usage errors,
generate -> parse round trip, and solve / speedup end to end on the device
(gpu-marked).  Without a GPU, solve must fail loudly with the solver-error
exit code (no CPU fallback)."""

import json

import numpy as np
import pytest

import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import cli


def _has_gpu():
    import torch

    return torch.cuda.is_available()


@pytest.mark.parametrize("argv", [
    [],
    ["solve"],  # neither --data nor --synthetic
    ["solve", "--synthetic", "10,5,0.5"],
    ["solve", "--synthetic", "10,5,x,0"],
    ["solve", "--synthetic", "10,5,0.5,0", "--data", "f.svm"],
    ["solve", "--synthetic", "10,5,0.5,0", "--lambda1", "-1"],
    ["solve", "--synthetic", "10,5,0.5,0", "--lambda1", "abc"],
    ["solve", "--synthetic", "10,5,0.5,0", "--lambda2", "-2"],
    ["solve", "--synthetic", "10,5,0.5,0", "--lambda2", "auto-nnz=0"],
    ["solve", "--synthetic", "10,5,0.5,0", "--lambda2", "auto-nnz=x"],
    ["solve", "--synthetic", "10,5,0.5,0", "--blocks", "file:/nonexistent/partition.txt"],
    ["solve", "--synthetic", "10,5,0.5,0", "--solver", "dense"],
    ["solve", "--synthetic", "10,5,0.5,0", "--penalty", "elastic"],
    ["speedup", "--synthetic", "10,5,0.5,0", "--cores", "1,x"],
])
def test_usage_errors_exit_2(argv, capsys):
    assert cli.main(argv) == cli.EXIT_USAGE


def test_generate_round_trip(tmp_path, capsys):
    out = tmp_path / "d.svm"
    assert cli.main(["generate", "--synthetic", "60,30,0.2,4", "--out", str(out)]) == cli.EXIT_OK
    assert "wrote 60 x 30 dataset" in capsys.readouterr().out
    ref = pb.gen_sparse_glm(60, 30, 0.2, 4)
    back = pb.parse_libsvm(str(out), n_cols=30, device=None)
    assert np.array_equal(back.features.row_offsets, ref.features.row_offsets)
    assert np.array_equal(back.features.col_indices, ref.features.col_indices)
    assert np.allclose(back.features.values, ref.features.values, rtol=1e-15)
    out2 = tmp_path / "disjoint.svm"
    assert cli.main(["generate", "--kind", "disjoint", "--synthetic", "40,20,0,1", "--out", str(out2)]) == 0
    assert pb.parse_libsvm(str(out2), device=None).n_samples == 40


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU behaviour")
def test_solve_without_gpu_is_a_solver_error(capsys):
    rc = cli.main(["solve", "--synthetic", "50,20,0.2,0", "--epochs", "2"])
    assert rc == cli.EXIT_SOLVER_ERROR
    assert "solver error" in capsys.readouterr().err


@pytest.mark.gpu
@pytest.mark.parametrize("threads", [1, 4])
def test_solve_routes_to_device_solver(cuda, tmp_path, capsys, threads):
    trace_path = tmp_path / "trace.csv"
    argv = ["solve", "--synthetic", "400,60,0.1,3", "--penalty", "l1", "--lambda2", "1e-3", "--epochs", "20",
            "--step", "1/2L", "--threads", str(threads), "--trace-out", str(trace_path)]
    assert cli.main(argv) == cli.EXIT_OK
    out = capsys.readouterr().out
    assert out.startswith("algorithm=")
    data = pb.gen_sparse_glm(400, 60, 0.1, 3)
    loss, pen = pb.Loss("logistic", 1.0 / 400), pb.L1Penalty(1e-3)
    part = pb.singleton_partition(60)
    if threads == 1:  # the deterministic replay: identical to the API call
        tr = pb.run_sequential(data, loss, pen, part, pb.SolverConfig(step_size="1/2L", epochs=20, seed=0))
        assert f"final objective {tr.objective[-1]:.12e}" in out
    rows = trace_path.read_text().splitlines()
    assert rows[0].startswith("iterations,epochs,objective,wall_seconds")
    assert len(rows) >= 3
    meta = json.loads((tmp_path / "trace.json").read_text())
    assert meta["problem_hash"] and meta["n_samples"] == 400
    assert meta["algorithm"] == ("sparse-saga" if threads == 1 else "async-saga")


@pytest.mark.gpu
def test_solve_fista_and_speedup(cuda, tmp_path, capsys):
    argv = ["solve", "--synthetic", "300,40,0.1,5", "--solver", "fista", "--lambda2", "1e-3", "--epochs", "50"]
    assert cli.main(argv) == cli.EXIT_OK
    assert "final objective" in capsys.readouterr().out
    out = tmp_path / "speedup.csv"
    argv = ["speedup", "--synthetic", "600,50,0.1,2", "--lambda2", "1e-3", "--cores", "1,4", "--epochs", "150",
            "--step", "1/2L", "--target", "1e-6", "--cache-dir", str(tmp_path / "cache"), "--out", str(out)]
    assert cli.main(argv) == cli.EXIT_OK
    text = capsys.readouterr().out
    assert "cores,wall_speedup,theoretical_speedup,reached" in text
    lines = out.read_text().splitlines()
    assert lines[0] == "cores,wall_speedup,theoretical_speedup,reached"
    assert lines[1].startswith("1,1.0,1.0,true")
    assert len(list((tmp_path / "cache").glob("optimum-*.npz"))) == 1


@pytest.mark.gpu
def test_solve_from_libsvm_file(cuda, tmp_path, capsys):
    """generate -> solve --data: the file goes through the device LibSVM parser
    and the same solve as the in-memory dataset (deterministic replay)."""
    path = tmp_path / "d.svm"
    assert cli.main(["generate", "--synthetic", "300,40,0.1,9", "--out", str(path)]) == cli.EXIT_OK
    capsys.readouterr()
    assert cli.main(["solve", "--data", str(path), "--lambda2", "1e-3", "--epochs", "10", "--step", "1/2L"]) == 0
    out = capsys.readouterr().out
    data = pb.parse_libsvm(str(path), device=None)
    tr = pb.run_sequential(data, pb.Loss("logistic", 1.0 / 300), pb.L1Penalty(1e-3),
                           pb.singleton_partition(data.n_features), pb.SolverConfig(step_size="1/2L", epochs=10))
    assert f"final objective {tr.objective[-1]:.12e}" in out
