"""The reference's step-level entry points on the device:
``sps_step`` (saga.py:169-185), ``worker_iteration`` (asynchronous.py:80-117),
``sparse_gradient_estimate`` (saga.py:150-166), ``prox_phi`` /
``prox_extended_slice`` (penalties.py:153-186), ``loss_scalar``
(losses.py:73-86).

Tolerances:
  * a host loop of ``pb.sps_step`` over the reference's sample stream matches
    the reference's golden iterates to 1e-9 relative (the deterministic bar);
  * a one-caller ``pb.worker_iteration`` loop equals the ``pb.sps_step`` loop
    bitwise (the reference's 1-thread async == sequential, test_async.py:105-112);
  * unbiasedness of v: max |E_i v_i - grad f(x)| <= 1e-12 (verify.py:229-250);
  * zero penalty: sps_step == the no-prox update built from
    sparse_gradient_estimate, to 1e-14 (verify.py:304-329);
  * write sparsity: bit-exact shadow copy (verify.py:384-404).
"""

import numpy as np
import pytest

import paper_1707_06468_b200 as pb
from paper_1707_06468_b200.saga import resolve_step_size, worker_rng

pytestmark = pytest.mark.gpu


def _index(case):
    return pb.build_support_index(case["data"].features, case["partition"], drop_dead_blocks=case["drop_dead"])


def _gamma(case):
    mu = case["loss"].lambda1
    L = pb.lipschitz_constant(case["data"], case["loss"]).L
    return resolve_step_size(case["step"], L, case["data"].n_samples, mu if mu > 0 else None)


@pytest.mark.parametrize("name", ["cfg1", "acc_l1", "grp_random", "grp_contig", "box_sq", "l1_ragged"])
def test_sps_step_loop_matches_reference_golden(cuda, name, small_cases, golden_small):
    case, g = small_cases[name], golden_small
    data = case["data"]
    n, p = data.n_samples, data.n_features
    index = _index(case)
    gamma = _gamma(case)
    seq = worker_rng(case["seed"], 0).integers(0, n, size=case["segments"][0])
    x = np.zeros(p)
    mem = pb.GradientMemory.zeros(n, p)
    for i in seq:
        pb.sps_step(x, mem, int(i), gamma, case["penalty"], index, case["loss"], data)
    ref = g[f"{name}__x"][0]
    rel = np.max(np.abs(x - ref)) / max(np.max(np.abs(ref)), 1e-300)
    assert rel <= 1e-9, f"{name}: rel {rel:.3e}"
    assert pb.full_objective(data, case["loss"], case["penalty"], x, case["partition"]) == pytest.approx(
        float(g[f"{name}__obj"][0]), rel=1e-12)


@pytest.mark.parametrize("name", ["acc_l1", "grp_random", "l1_blocks"])
def test_worker_iteration_equals_sps_step_bitwise(cuda, name, small_cases):
    case = small_cases[name]
    data = case["data"]
    n, p = data.n_samples, data.n_features
    index = _index(case)
    gamma = _gamma(case)
    seq = worker_rng(7, 0).integers(0, n, size=2 * n)
    x = np.zeros(p)
    mem = pb.GradientMemory.zeros(n, p)
    shared = pb.SharedState(n, p)
    for i in seq:
        before = shared.x.copy()
        dx = pb.worker_iteration(shared, int(i), gamma, case["penalty"], index, case["loss"], data)
        pb.sps_step(x, mem, int(i), gamma, case["penalty"], index, case["loss"], data)
        ecols = index.ext_slice(int(i))[0]
        assert len(dx) == len(ecols)
        assert np.array_equal(shared.x[ecols], before[ecols] + dx)  # x moved by exactly the returned delta
    assert np.array_equal(shared.x, x)
    assert np.array_equal(shared.avg, mem.avg)
    assert np.array_equal(shared.scalars, mem.scalars)


def test_gradient_estimate_is_unbiased(cuda):
    rng = np.random.default_rng(40)
    worst = 0.0
    for _ in range(4):
        n, p = int(rng.integers(20, 41)), int(rng.integers(5, 16))
        data = pb.gen_sparse_glm(n, p, float(rng.uniform(0.3, 0.8)), int(rng.integers(1e6)))
        nb = int(rng.integers(2, p + 1))
        perm = rng.permutation(p)
        blocks = [np.sort(b) for b in np.array_split(perm, nb)]
        bo = np.empty(p, dtype=np.int64)
        for b, c in enumerate(blocks):
            bo[c] = b
        part = pb.BlockPartition(bo, blocks)
        index = pb.build_support_index(data.features, part, drop_dead_blocks=True)
        loss = pb.Loss("logistic", float(rng.uniform(0.0, 0.1)))
        x = rng.standard_normal(p)
        mem = pb.GradientMemory(scalars=rng.standard_normal(n), avg=np.zeros(p))
        pb.resync_average(mem, data)
        mean = np.zeros(p)
        for i in range(n):
            ecols, v, _ = pb.sparse_gradient_estimate(i, x, mem, index, loss, data)
            mean[ecols] += v
        worst = max(worst, float(np.max(np.abs(mean / n - pb.smooth_gradient(data, loss, x)))))
    assert worst <= 1e-12


def test_zero_penalty_step_equals_plain_gradient_step(cuda, small_cases):
    case = small_cases["acc_l1"]
    data, loss = case["data"], case["loss"]
    n, p = data.n_samples, data.n_features
    index = _index(case)
    gamma = _gamma(case)
    pen = pb.ZeroPenalty()
    x, xr = np.zeros(p), np.zeros(p)
    mem, memr = pb.GradientMemory.zeros(n, p), pb.GradientMemory.zeros(n, p)
    worst = 0.0
    for i in worker_rng(0, 0).integers(0, n, size=n):
        i = int(i)
        pb.sps_step(x, mem, i, gamma, pen, index, loss, data)
        cols, vals = data.features.row(i)
        ecols, v, new = pb.sparse_gradient_estimate(i, xr, memr, index, loss, data)
        xe = xr[ecols]
        z = xe - gamma * v
        xr[ecols] = xe + (z - xe)
        memr.avg[cols] += ((new - memr.scalars[i]) / memr.n) * vals
        memr.scalars[i] = new
        worst = max(worst, float(np.max(np.abs(x - xr))))
    assert worst <= 1e-14


def test_sps_step_writes_only_the_extended_support(cuda, small_cases):
    case = small_cases["grp_random"]
    data = case["data"]
    n, p = data.n_samples, data.n_features
    index = _index(case)
    gamma = _gamma(case)
    x = np.zeros(p)
    shadow = x.copy()
    mem = pb.GradientMemory.zeros(n, p)
    for i in worker_rng(3, 0).integers(0, n, size=2 * n):
        i = int(i)
        pb.sps_step(x, mem, i, gamma, case["penalty"], index, case["loss"], data)
        ecols = index.ext_slice(i)[0]
        shadow[ecols] = x[ecols]
        assert np.array_equal(x, shadow)


def test_prox_phi_matches_slice_form_and_block_weights(cuda, small_cases):
    """penalties.py:153-186; reference tests test_penalties.py:110-137."""
    case = small_cases["grp_random"]
    data = case["data"]
    index = _index(case)
    rng = np.random.default_rng(5)
    for pen in (pb.GroupL2Penalty(0.3), pb.L1Penalty(0.2)):
        for i in range(6):
            v = rng.standard_normal(data.n_features)
            full = pb.prox_phi(pen, index, i, 0.1, v)
            coords = index.ext_slice(i)[0]
            sliced = pb.prox_extended_slice(pen, index, i, 0.1, v[coords])
            assert np.array_equal(full[coords], sliced)
            rest = np.setdiff1d(np.arange(data.n_features), coords)
            assert np.array_equal(full[rest], v[rest])
            # block weights: each block of T_i gets step 0.1 * d_B
            bo = index.partition.block_of
            for b in np.unique(bo[coords]):
                bc = index.partition.blocks[b]
                want = pen.prox_block(v[bc], 0.1 * index.d_B[b]) if not pen.separable else \
                    pen.prox(v[bc], 0.1 * index.d_B[b] * np.ones(len(bc)))
                assert np.array_equal(full[bc], want)


def test_loss_scalar_known_answers(cuda):
    """losses.py:73-86: squared (3, 1) -> (2, 2); logistic (0, 1) -> (log 2, -1/2)
    (test_losses.py:55-58); value/derivative consistent with a
    central difference."""
    assert pb.loss_scalar("squared", 3.0, 1.0) == (2.0, 2.0)
    v, d = pb.loss_scalar("logistic", 0.0, 1.0)
    assert v == pytest.approx(np.log(2.0), rel=1e-15) and d == -0.5
    for z, b in ((0.7, 1.0), (-3.0, -1.0), (40.0, 1.0), (-40.0, 1.0)):
        eps = 1e-6
        fp, _ = pb.loss_scalar("logistic", z + eps, b)
        fm, _ = pb.loss_scalar("logistic", z - eps, b)
        _, d = pb.loss_scalar("logistic", z, b)
        assert (fp - fm) / (2 * eps) == pytest.approx(d, rel=1e-6, abs=1e-12)
    with pytest.raises(ValueError):
        pb.loss_scalar("hinge", 0.0, 1.0)
