"""λ-path sharding (config 5's multi-GPU workload) on CPU: world_size-2 gloo
processes, each solving its share of the lambdas with the C oracle (the
checker; on the GPU box the same run_path drives DeviceProblem solves), must
reproduce the single-process path exactly (independent solves, no data-path
collective, one all_gather of the summaries)."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import lambda_path as lp


def test_lambda_grid_and_assignment():
    lams = lp.lambda_grid(2.0, 16, 1e-3)
    assert len(lams) == 16 and lams[0] == 2.0 and lams[-1] == pytest.approx(2e-3)
    assert all(a > b for a, b in zip(lams, lams[1:]))
    shards = lp.assign(lams, 4)
    assert sorted(k for s in shards for k in s) == list(range(16))
    assert [len(s) for s in shards] == [4, 4, 4, 4]
    # longest work (smallest lambda) first: rank 0 gets the smallest lambda
    assert shards[0][0] == 15 and shards[1][0] == 14
    assert lp.assign(lams, 1) == [sorted(range(16), key=lambda k: lams[k])]


def _problem():
    data = pb.gen_sparse_glm(120, 40, 0.15, 3)
    part = pb.contiguous_partition(40, 5)
    loss = pb.Loss("logistic", 1.0 / 120)
    return data, loss, part


def _oracle_solver(data, loss, part):
    from oracle import oracle as O

    def solve(lam):
        P = O.from_dataset(data, loss, pb.GroupL2Penalty(lam), part)
        gamma = 1.0 / (2.0 * P.lipschitz())
        x, _, _ = P.run_sequential(gamma, O.sample_sequence(0, P.n, 20 * P.n))
        return {"objective": P.objective(x), "nnz": int(np.count_nonzero(x)), "updates": 20 * P.n}

    return solve


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        data, loss, part = _problem()
        lams = lp.lambda_grid(0.05, 6, 1e-2)
        res = lp.run_path(lams, _oracle_solver(data, loss, part))
        out[rank] = [(r["index"], r["rank"], r["objective"], r["nnz"]) for r in res]
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_path_sharded_over_two_gloo_ranks_matches_single_process():
    data, loss, part = _problem()
    lams = lp.lambda_grid(0.05, 6, 1e-2)
    single = lp.run_path(lams, _oracle_solver(data, loss, part), rank=0, world=1)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert out[0] == out[1]  # every rank holds the gathered path
    got = out[0]
    assert [g[0] for g in got] == list(range(6))
    assert sorted({g[1] for g in got}) == [0, 1]  # both ranks solved something
    for g, s in zip(got, single):
        assert g[2] == s["objective"] and g[3] == s["nnz"]  # independent solves: bitwise
    # the path is monotone in sparsity: larger lambda -> fewer nonzeros
    nnz = [g[3] for g in got]
    assert nnz[0] <= nnz[-1]


def test_run_path_uses_batch_solver_when_present():
    """A solver exposing ``batch`` (concurrent solves per rank) gets this
    rank's lambdas in one call, in assignment order."""
    calls = []

    def solve(lam):  # pragma: no cover - must not be called
        raise AssertionError("per-lambda path used")

    def batch(lams):
        calls.append(list(lams))
        return [{"objective": lam * 2.0} for lam in lams]

    solve.batch = batch
    lams = lp.lambda_grid(1.0, 6, 1e-2)
    res = lp.run_path(lams, solve, rank=0, world=1)
    assert len(calls) == 1 and calls[0] == [lams[k] for k in lp.assign(lams, 1)[0]]
    assert [r["index"] for r in res] == list(range(6))
    assert all(r["objective"] == r["lam"] * 2.0 for r in res)
