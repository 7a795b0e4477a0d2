"""Host-side logic (CPU): descriptors, validation, configs, traces, generators.
Mirrors the reference tests test_data.py / test_saga.py / test_async.py /
test_penalties.py / test_problems.py where they do not need the device."""

import gzip
import io

import numpy as np
import pytest

import paper_1707_06468_b200 as pb
from paper_1707_06468_b200.data import partition_structure

SAMPLE = "1 1:0.5 3:-2.0\n-1 2:1.5\n1 1:1.0 2:2.0 3:3.0\n"


def small_matrix():
    return pb.CsrMatrix(3, 3, np.array([0, 2, 3, 6]), np.array([0, 2, 1, 0, 1, 2]),
                        np.array([0.5, -2.0, 1.5, 1.0, 2.0, 3.0]))


def test_csr_validation():
    """test_data.py:113-121."""
    with pytest.raises(ValueError):
        pb.CsrMatrix(2, 2, np.array([0, 1]), np.array([0]), np.array([1.0]))
    with pytest.raises(ValueError, match="strictly increasing"):
        pb.CsrMatrix(1, 2, np.array([0, 2]), np.array([1, 0]), np.array([1.0, 2.0]))
    with pytest.raises(ValueError):
        pb.CsrMatrix(1, 2, np.array([0, 1]), np.array([5]), np.array([1.0]))
    with pytest.raises(ValueError):
        pb.CsrMatrix(1, 1, np.array([0, 1]), np.array([0]), np.array([np.inf]))
    with pytest.raises(ValueError, match="row 1"):
        pb.CsrMatrix(2, 4, np.array([0, 2, 4]), np.array([0, 3, 2, 2]), np.ones(4))
    # a decrease across a row boundary is fine
    pb.CsrMatrix(3, 4, np.array([0, 2, 2, 4]), np.array([2, 3, 0, 1]), np.ones(4))


def test_csr_keeps_fp32_values():
    m = pb.CsrMatrix(1, 2, np.array([0, 2]), np.array([0, 1]), np.array([1.0, 2.0], dtype=np.float32))
    assert m.values.dtype == np.float32
    m2 = pb.CsrMatrix(1, 2, np.array([0, 2]), np.array([0, 1]), [1, 2])
    assert m2.values.dtype == np.float64


def test_dataset_label_length_checked():
    with pytest.raises(ValueError):
        pb.Dataset(features=small_matrix(), labels=np.array([1.0]))


def test_partition_validation_and_structure():
    """test_data.py:133-143 plus the device layout detection."""
    with pytest.raises(ValueError):
        pb.BlockPartition(np.array([0, 0]), [np.array([0, 1]), np.array([1])])
    with pytest.raises(ValueError):
        pb.BlockPartition(np.array([0, 0]), [np.array([0])])
    with pytest.raises(ValueError):
        pb.BlockPartition(np.array([0]), [np.array([0]), np.array([], dtype=int)])
    part = pb.singleton_partition(4)
    assert part.is_singleton and part.n_blocks == 4 and len(part.blocks[2]) == 1
    whole = pb.single_block_partition(4)
    assert whole.n_blocks == 1 and len(whole.blocks[0]) == 4
    assert partition_structure(part) == ("singleton", 1)
    assert partition_structure(pb.contiguous_partition(25, 10)) == ("contiguous", 10)
    c = pb.contiguous_partition(25, 10)
    assert c.n_blocks == 3 and list(c.blocks[2]) == [20, 21, 22, 23, 24]
    explicit = pb.BlockPartition(np.arange(6) // 3, [np.arange(3), np.arange(3, 6)])
    assert partition_structure(explicit) == ("contiguous", 3)
    assert partition_structure(whole) in (("contiguous", 4), ("general", 0))
    rnd = pb.BlockPartition(np.array([1, 0, 1, 0]), [np.array([1, 3]), np.array([0, 2])])
    assert partition_structure(rnd) == ("general", 0)


def test_load_partition_file(tmp_path):
    path = tmp_path / "blocks.txt"
    path.write_text("0 2\n1\n\n3\n")
    part = pb.load_partition_file(path, 4)
    assert part.n_blocks == 3 and list(part.blocks[0]) == [0, 2]


def test_libsvm_parse_and_round_trip(tmp_path):
    """test_data.py:38-92."""
    data = pb.parse_libsvm(io.StringIO(SAMPLE))
    assert data.n_samples == 3 and data.n_features == 3
    assert list(data.labels) == [1.0, -1.0, 1.0]
    cols, vals = data.features.row(0)
    assert list(cols) == [0, 2] and list(vals) == [0.5, -2.0]
    with pytest.raises(pb.ParseError) as exc:
        pb.parse_libsvm(io.StringIO("1 1:0.5\nbad 1:2\n"))
    assert exc.value.line == 2
    for bad in ("1 2:1.0 2:2.0\n", "1 0:1.0\n", ""):
        with pytest.raises(pb.ParseError):
            pb.parse_libsvm(io.StringIO(bad))
    assert pb.parse_libsvm(io.StringIO("1 2:1.0\n"), n_cols=5).n_features == 5
    path = tmp_path / "out.svm.gz"
    pb.to_libsvm(data, path)
    with gzip.open(path, "rt") as fh:
        assert fh.readline().startswith("1.0 ")
    again = pb.parse_libsvm(path)
    assert np.array_equal(again.features.values, data.features.values)


def test_resolve_step_size_rules():
    """test_saga.py:24-35."""
    r = pb.resolve_step_size
    assert r("1/5L", 2.0) == pytest.approx(0.1)
    assert r("1/2L", 2.0) == pytest.approx(0.25)
    assert r("1/36L", 1.0) == pytest.approx(1 / 36)
    assert r("1/36nmu", 1.0, n=10, mu=0.5) == pytest.approx(1 / 180)
    assert r(0.07, 1.0) == 0.07
    for bad in (("1/3L", 1.0), ("1/36nmu", 1.0, 10, 0.0), (-1.0, 1.0)):
        with pytest.raises(ValueError):
            r(*bad)


def test_worker_streams():
    """test_saga.py:38-43 / test_async.py:99-102."""
    a = pb.worker_rng(3, 0).integers(0, 100, size=10)
    assert np.array_equal(a, pb.worker_rng(3, 0).integers(0, 100, size=10))
    assert not np.array_equal(a, pb.worker_rng(3, 1).integers(0, 100, size=10))
    assert np.array_equal(pb.worker_rng(7, 0).integers(0, 50, size=100), pb.worker_sample_sequence(7, 0, 100, 50))
    assert pb.split_iterations(10, 3) == [4, 3, 3]
    assert sum(pb.split_iterations(1001, 4)) == 1001


def test_config_validation():
    with pytest.raises(ValueError):
        pb.SolverConfig(epochs=0)
    with pytest.raises(ValueError):
        pb.SolverConfig(step_size=-0.1)
    with pytest.raises(ValueError):
        pb.SolverConfig(checkpoint_every=0)
    with pytest.raises(ValueError):
        pb.AsyncConfig(threads=0)
    with pytest.raises(ValueError):
        pb.AsyncConfig(counter_batch=0)
    with pytest.raises(ValueError):
        pb.AsyncConfig(warps=0)


def test_thread_cap_checked_before_any_device_work():
    d = pb.gen_sparse_glm(10, 5, 0.4, 0)
    with pytest.raises(ValueError):
        pb.run_async(d, pb.Loss("logistic", 0.1), pb.L1Penalty(0.01), pb.singleton_partition(5),
                     pb.AsyncConfig(epochs=1, threads=128))


def test_trace_csv_and_sidecar(tmp_path):
    tr = pb.Trace(meta={"algorithm": "async-saga"})
    for it, obj in [(0, 1.0), (100, 0.5)]:
        tr.append(it, 100, obj, 0.01 * it, threads=2)
    tr.to_csv(tmp_path / "t.csv")
    lines = (tmp_path / "t.csv").read_text().splitlines()
    assert lines[0] == "iterations,epochs,objective,wall_seconds,threads,counter_iterations"
    assert len(lines) == 3
    tr.write_sidecar(tmp_path / "t.json")
    assert "async-saga" in (tmp_path / "t.json").read_text()


def test_iterations_to_target_interpolates():
    """test_async.py:139-147."""
    tr = pb.Trace()
    for it, obj in [(0, 1.0), (100, 1e-2), (200, 1e-6)]:
        tr.append(it, 100, obj, it * 0.001)
    iters, wall = pb.iterations_to_target(tr, 0.0, 1e-4)
    assert 100 < iters < 200 and 0.1 < wall < 0.2
    assert pb.iterations_to_target(tr, 0.0, 1e-12) is None


def test_measure_speedup_validates_cores():
    d = pb.gen_sparse_glm(10, 5, 0.4, 0)
    cfg = pb.AsyncConfig(epochs=1)
    for cores in ([2, 4], [1, 4, 2]):
        with pytest.raises(ValueError):
            pb.measure_speedup(d, pb.Loss("logistic"), pb.L1Penalty(0.1), pb.singleton_partition(5), cfg, cores,
                               1e-6, 0.0)


def test_penalty_descriptors():
    """test_penalties.py:91-151 (non-device parts)."""
    assert isinstance(pb.make_penalty("none"), pb.ZeroPenalty)
    assert isinstance(pb.make_penalty("l1", lam2=0.1), pb.L1Penalty)
    assert isinstance(pb.make_penalty("group-l1", lam2=0.1), pb.GroupL2Penalty)
    box = pb.make_penalty("box", lo=-2, hi=2)
    assert isinstance(box, pb.BoxPenalty) and box.hi == 2.0
    for bad in (lambda: pb.make_penalty("elastic"), lambda: pb.L1Penalty(-1.0), lambda: pb.BoxPenalty(1.0, 0.0),
                lambda: pb.ProxStep(gamma=0.0), lambda: pb.ProxStep(gamma=1.0, scale=0.5)):
        with pytest.raises(ValueError):
            bad()
    assert pb.ProxStep(gamma=0.5, scale=3.0).effective == pytest.approx(1.5)
    assert pb.L1Penalty(1.0).value(np.array([3.0, -0.5, 0.0, -4.0])) == pytest.approx(7.5)
    assert pb.BoxPenalty(-1.0, 2.0).value(np.array([0.0, 2.0])) == 0.0
    assert pb.BoxPenalty(-1.0, 2.0).value(np.array([2.1])) == np.inf
    part = pb.contiguous_partition(4, 2)
    assert pb.GroupL2Penalty(2.0).value(np.array([3.0, 4.0, 0.0, 1.0]), part) == pytest.approx(12.0)
    with pytest.raises(ValueError):
        pb.prox_block(pb.L1Penalty(1.0), np.array([np.nan]), pb.ProxStep(1.0))
    with pytest.raises(ValueError):
        pb.GroupL2Penalty(1.0).prox(np.ones(2), np.ones(2))


def test_generators_reproduce_reference_instances(golden_small):
    """gen_sparse_glm is a restatement of problems.py:13-50: same seed, same
    instance (data hash recorded from the reference)."""
    from tests.golden.make_golden import data_hash

    d = pb.gen_sparse_glm(200, 50, 0.1, 42)
    assert data_hash(d.features, d.labels) == str(golden_small["acc__hash"])


def test_baseline_config2_statistics():
    """SURVEY.md §0/§8d probe numbers for config 2 (k=20 distinct Zipf(1.1) columns)."""
    from paper_1707_06468_b200 import problems

    c = problems.config2(seed=0)
    f = c["data"].features
    assert f.values.dtype == np.float32 and f.nnz == 2_000_000
    counts = np.bincount(f.col_indices, minlength=f.n_cols)
    assert counts.max() / f.n_rows == pytest.approx(0.963, abs=0.002)      # delta
    assert int(np.sum(counts == 0)) == pytest.approx(1142, abs=60)          # dead columns
    assert np.all(np.diff(f.col_indices.reshape(-1, 20), axis=1) > 0)


def test_diagnostics_host_logic(tmp_path):
    """diagnostics.py:25-62 restated: suboptimality clamps within the slack
    and raises below it; the rate factor; envelope records."""
    from paper_1707_06468_b200 import diagnostics as dg

    assert dg.suboptimality([1.0, 0.5 + 1e-13, 0.75], 0.5) == [0.5, 1e-13 + 0.5 - 0.5, 0.25]
    with pytest.raises(dg.StaleOptimumError):
        dg.suboptimality([0.4], 0.5)
    assert dg.theorem_rate_factor(200, 50.0) == pytest.approx(0.2 / 200)
    assert dg.theorem_rate_factor(10, 50.0) == pytest.approx(0.2 / 50)
    recs = dg.rate_envelope_check({0: 1.0, 10: 0.5, 20: 0.9}, 0.05, 1.0, 1.0)
    assert [r["passed"] for r in recs] == [True, True, False]
    assert recs[1]["bound"] == pytest.approx(0.95 ** 10)
    with pytest.raises(ValueError):
        dg.rate_envelope_check({0: 1.0}, 1.5, 1.0, 1.0)
    d = pb.gen_sparse_glm(30, 10, 0.3, 1)
    h1 = dg.problem_hash(d, pb.Loss("logistic", 0.1), pb.L1Penalty(0.2), pb.singleton_partition(10))
    h2 = dg.problem_hash(d, pb.Loss("logistic", 0.1), pb.L1Penalty(0.3), pb.singleton_partition(10))
    assert h1 != h2 and len(h1) == 64
    assert dg.default_cache_dir().name


def test_bench_first_crossing_interpolation():
    """bench._first_crossing: log-linear interpolation of the first checkpoint
    under the target (asynchronous.py:213-230 on the relative gap)."""
    import math

    import bench

    its = [100, 200, 300]
    walls = [1.0, 2.0, 3.0]
    rel = [1e-4, 1e-6 * 0.1, 1e-9]
    sec, ep = bench._first_crossing(its, walls, rel, 100, 1e-6)
    frac = math.log(1e-4 / 1e-6) / math.log(1e-4 / 1e-7)
    assert sec == pytest.approx(1.0 + frac) and ep == pytest.approx((100 + frac * 100) / 100)
    assert bench._first_crossing(its, walls, [1e-3, 1e-4, 1e-5], 100, 1e-6) is None
    # already under the target at the first checkpoint: interpolated from (0, rel 1)
    sec, ep = bench._first_crossing([50], [0.5], [1e-8], 100, 1e-6)
    assert 0 < sec < 0.5 and 0 < ep < 0.5


def test_async_grid_launches_exactly_the_requested_warps():
    """measure_speedup's c warps: ctas * warps_per_cta == c (c=12 ran 8 warps)."""
    from types import SimpleNamespace

    from paper_1707_06468_b200.asynchronous import _grid

    for c in (1, 2, 3, 4, 8, 12, 20, 24, 32, 48, 100, 148, 4736):
        ctas, wpc = _grid(None, SimpleNamespace(warps=c, warps_per_cta=0))
        assert ctas * wpc == c, (c, ctas, wpc)
        assert 1 <= wpc <= 32
    assert _grid(None, SimpleNamespace(warps=None, warps_per_cta=0)) == (0, 0)
    assert _grid(None, SimpleNamespace(warps=64, warps_per_cta=16)) == (4, 16)


def test_bench_line_splits_long_numeric_arrays():
    import importlib.util
    from pathlib import Path

    spec = importlib.util.spec_from_file_location("bench", Path(__file__).resolve().parents[1] / "bench.py")
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    detail = {}
    line = {"a": list(range(20)), "b": [1, 2], "c": [{"x": list(range(9)), "y": 1}], "d": {"e": [0.5] * 30}}
    out = bench._split_arrays(line, "", detail)
    assert out["b"] == [1, 2] and out["c"][0]["y"] == 1
    assert set(detail) == {"a", "c[0].x", "d.e"}
    assert detail["a"] == list(range(20)) and isinstance(out["a"], str)
