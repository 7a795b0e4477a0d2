"""Seeded parity cases shared by make_golden.py (reference side) and the tests.

Each case: data / loss / penalty / partition (this package's host
descriptors; numpy only), the step rule, the sample-stream seed, the number of
sequential steps and the step counts at which x is snapshotted.
"""

from __future__ import annotations

import numpy as np

import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems


def _random_partition(rng, p, n_blocks):
    perm = rng.permutation(p)
    cuts = np.sort(rng.choice(np.arange(1, p), size=n_blocks - 1, replace=False))
    pieces = np.split(perm, cuts)
    blocks = [np.sort(b) for b in pieces]
    bo = np.empty(p, dtype=np.int64)
    for b, c in enumerate(blocks):
        bo[c] = b
    return pb.BlockPartition(bo, blocks)


def _ragged(seed, n, p, kmax, empty_every=7):
    rng = np.random.default_rng(seed)
    ks = rng.integers(0, kmax + 1, size=n)
    ks[::empty_every] = 0
    ks[1] = kmax  # at least one long row
    offs = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(ks, out=offs[1:])
    cols = np.concatenate([np.sort(rng.choice(p, size=k, replace=False)) for k in ks])
    vals = rng.standard_normal(len(cols))
    f = pb.CsrMatrix(n, p, offs, cols, vals)
    y = np.where(rng.standard_normal(n) > 0, 1.0, -1.0)
    return pb.Dataset(f, y)


def _case(data, loss, penalty, partition, step, seed, epochs, seg_epochs=None, drop_dead=False):
    n = data.n_samples
    steps = epochs * n
    segs = [e * n for e in (seg_epochs or range(1, epochs + 1))]
    return dict(data=data, loss=loss, penalty=penalty, partition=partition, step=step, seed=seed,
                steps=steps, segments=segs, drop_dead=drop_dead)


def small_cases():
    c = {}
    cfg1 = problems.config1(seed=0)
    c["cfg1"] = _case(cfg1["data"], cfg1["loss"], cfg1["penalty"], cfg1["partition"], 1.0 / 3.0, 0, 20)
    d = pb.gen_sparse_glm(200, 50, 0.1, 42)
    c["acc_l1"] = _case(d, pb.Loss("logistic", 1 / 200), pb.L1Penalty(0.01), pb.singleton_partition(50),
                        "1/5L", 2, 3)
    d = pb.gen_sparse_glm(60, 40, 0.3, 7)
    rng = np.random.default_rng(11)
    c["grp_random"] = _case(d, pb.Loss("logistic", 0.01), pb.GroupL2Penalty(0.05), _random_partition(rng, 40, 9),
                            "1/5L", 1, 4)
    c["l1_blocks"] = _case(d, pb.Loss("logistic", 0.01), pb.L1Penalty(0.03), _random_partition(rng, 40, 13),
                           "1/2L", 3, 3)
    d = pb.gen_sparse_glm(70, 103, 0.08, 9)
    c["grp_contig"] = _case(d, pb.Loss("logistic", 0.02), pb.GroupL2Penalty(0.02), pb.contiguous_partition(103, 10),
                            "1/5L", 4, 4)
    c["grp_g1"] = _case(d, pb.Loss("logistic", 0.02), pb.GroupL2Penalty(0.02), pb.singleton_partition(103),
                        "1/5L", 5, 2)
    d = pb.gen_sparse_glm(80, 30, 0.2, 5, loss_kind="squared")
    c["box_sq"] = _case(d, pb.Loss("squared", 0.05), pb.BoxPenalty(-0.2, 0.3), pb.singleton_partition(30),
                        "1/5L", 6, 3)
    c["zero_sq"] = _case(d, pb.Loss("squared", 0.1), pb.ZeroPenalty(), pb.singleton_partition(30), 0.05, 7, 3)
    c["single_block"] = _case(d, pb.Loss("squared", 0.05), pb.GroupL2Penalty(0.1), pb.single_block_partition(30),
                              "1/5L", 8, 3)
    d = _ragged(13, 50, 300, 150)
    c["l1_ragged"] = _case(d, pb.Loss("logistic", 0.02), pb.L1Penalty(0.01), pb.singleton_partition(300),
                           "1/2L", 9, 6, drop_dead=True)
    c["grp_ragged_contig"] = _case(d, pb.Loss("logistic", 0.02), pb.GroupL2Penalty(0.01),
                                   pb.contiguous_partition(300, 7), "1/2L", 10, 4, drop_dead=True)
    cfg2s = problems.config2(seed=3, n=2000, p=5000)
    c["cfg2_small"] = _case(cfg2s["data"], cfg2s["loss"], cfg2s["penalty"], cfg2s["partition"], "1/2L", 0, 5,
                            drop_dead=True)
    cfg5s = problems.config5(seed=4, n=3000, p=100_000)
    c["cfg5_small"] = _case(cfg5s["data"], cfg5s["loss"], pb.GroupL2Penalty(2e-4), cfg5s["partition"], "1/2L", 0,
                            3, drop_dead=True)
    return c


def large_cases():
    cfg2 = problems.config2(seed=0)
    return {"cfg2": _case(cfg2["data"], cfg2["loss"], cfg2["penalty"], cfg2["partition"], "1/2L", 0, 30,
                          seg_epochs=[1, 5, 30], drop_dead=True)}
