"""Seeded synthetic problems.

* ``gen_sparse_glm`` / ``gen_disjoint_glm`` restate the reference's desk-scale
  generators (problems.py:13-91) with the same numpy call sequence, so the
  same seed gives the same instance (pinned in tests against golden data).
* ``baseline_config(k)`` builds BASELINE.json configs 1-5:
  the paper's LibSVM datasets are absent, so seeded synthetic inputs with the
  configs' shapes, sparsity laws and value distributions stand in for them.
* ``lambda_max`` / ``group_lambda_max`` use the device gradient at x = 0.
"""

from __future__ import annotations

import numpy as np

from .data import CsrMatrix, Dataset, contiguous_partition, singleton_partition
from .losses import LOGISTIC, SQUARED, Loss
from .penalties import GroupL2Penalty, L1Penalty

LABEL_NOISE = 0.05


def _labels_from_planted(rng, features_vals, cols, offsets, n, p, planted, loss_kind):
    margins = np.add.reduceat(features_vals * planted[cols], offsets[:-1]) if len(cols) else np.zeros(n)
    margins[np.diff(offsets) == 0] = 0.0
    return margins


def gen_sparse_glm(n, p, density, seed, loss_kind=LOGISTIC):
    """problems.py:13-50 — exact per-row density, planted 10% model, 5% noise."""
    if n < 1 or p < 1:
        raise ValueError("n and p must be >= 1")
    if not 0 < density <= 1:
        raise ValueError("density must be in (0, 1]")
    rng = np.random.default_rng(int(seed))
    k = max(1, round(density * p))
    offsets = np.arange(n + 1, dtype=np.int64) * k
    cols = np.empty(n * k, dtype=np.int64)
    vals = rng.standard_normal(n * k)
    for i in range(n):
        cols[i * k:(i + 1) * k] = np.sort(rng.choice(p, size=k, replace=False))
    feats = CsrMatrix(n_rows=n, n_cols=p, row_offsets=offsets, col_indices=cols, values=vals)
    planted = np.zeros(p)
    support = rng.choice(p, size=max(1, p // 10), replace=False)
    planted[support] = rng.standard_normal(len(support))
    margins = feats.to_scipy() @ planted
    if loss_kind == LOGISTIC:
        labels = np.where(margins >= 0, 1.0, -1.0)
        flips = rng.random(n) < LABEL_NOISE
        labels[flips] *= -1.0
    elif loss_kind == SQUARED:
        scale = float(np.std(margins)) or 1.0
        labels = margins + LABEL_NOISE * scale * rng.standard_normal(n)
    else:
        raise ValueError(f"unknown loss kind {loss_kind!r}")
    return Dataset(features=feats, labels=labels)


def gen_disjoint_glm(n, p, seed, coords_per_row=2, loss_kind=LOGISTIC):
    """problems.py:53-91 — near-disjoint row windows, unit-norm rows."""
    if n < 1 or p < 1 or coords_per_row < 1:
        raise ValueError("n, p and coords_per_row must be >= 1")
    if n * coords_per_row < p:
        raise ValueError("need n * coords_per_row >= p to cover every coordinate")
    rng = np.random.default_rng(int(seed))
    k = coords_per_row
    offsets = np.arange(n + 1, dtype=np.int64) * k
    vals = rng.standard_normal(n * k)
    win = (np.arange(k, dtype=np.int64)[None, :] + k * np.arange(n, dtype=np.int64)[:, None]) % p
    win.sort(axis=1)
    cols = win.reshape(-1)
    for i in range(n):  # per-row norm, same reduction as the reference
        seg = vals[i * k:(i + 1) * k]
        vals[i * k:(i + 1) * k] = seg / np.linalg.norm(seg)
    feats = CsrMatrix(n_rows=n, n_cols=p, row_offsets=offsets, col_indices=cols, values=vals)
    planted = np.zeros(p)
    support = rng.choice(p, size=max(1, p // 10), replace=False)
    planted[support] = rng.standard_normal(len(support))
    margins = feats.to_scipy() @ planted
    if loss_kind == LOGISTIC:
        labels = np.where(margins >= 0, 1.0, -1.0)
        flips = rng.random(n) < LABEL_NOISE
        labels[flips] *= -1.0
    else:
        scale = float(np.std(margins)) or 1.0
        labels = margins + LABEL_NOISE * scale * rng.standard_normal(n)
    return Dataset(features=feats, labels=labels)


def lambda_max(data, device=None):
    """Smallest l1 weight with x = 0 optimal, logistic (problems.py:94-97)."""
    from .losses import smooth_gradient

    g = smooth_gradient(data, Loss(LOGISTIC, 0.0), np.zeros(data.n_features), device=device)
    return float(np.max(np.abs(g)))


def group_lambda_max(data, partition, device=None):
    """Group analogue (no reference counterpart): max_B ||grad_B f(0)||_2."""
    from .losses import smooth_gradient

    g = smooth_gradient(data, Loss(LOGISTIC, 0.0), np.zeros(data.n_features), device=device)
    sq = np.bincount(partition.block_of, weights=g * g, minlength=partition.n_blocks)
    return float(np.sqrt(sq.max()))


def gen_regularization(data, target_nnz_fraction, solve, max_steps=40, rel_window=0.2, device=None):
    """lambda2 bisection on solution density (problems.py:100-128)."""
    if data.n_samples == 0:
        raise ValueError("dataset is empty")
    lam1 = 1.0 / data.n_samples
    if target_nnz_fraction >= 1.0:
        return lam1, 0.0
    lo, hi = 0.0, lambda_max(data, device=device)
    lo_frac = _nnz_fraction(solve(lam1, lo))
    if lo_frac <= target_nnz_fraction * (1 + rel_window):
        return lam1, lo
    for _ in range(max_steps):
        mid = 0.5 * (lo + hi)
        frac = _nnz_fraction(solve(lam1, mid))
        if abs(frac - target_nnz_fraction) <= rel_window * target_nnz_fraction:
            return lam1, mid
        if frac > target_nnz_fraction:
            lo = mid
        else:
            hi = mid
    raise RuntimeError(f"bisection did not converge in {max_steps} steps (bracket [{lo}, {hi}])")


def _nnz_fraction(x):
    x = np.asarray(x)
    return float(np.count_nonzero(np.abs(x) > 0)) / len(x)


# ---------------------------------------------------------------------------
# BASELINE.json configs

def zipf_rows(rng, n, p, k, s, col_offset=0, chunk=1 << 20):
    """n rows of k DISTINCT sorted columns drawn from P(j) ∝ (j+1)^-s on [0, p).

    Resample-until-distinct per row, vectorised: sort each
    row, redraw duplicated slots only, repeat."""
    w = np.arange(1, p + 1, dtype=np.float64) ** (-s)
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    out = np.empty((n, k), dtype=np.int64)
    for r0 in range(0, n, chunk):
        r1 = min(n, r0 + chunk)
        blk = np.searchsorted(cdf, rng.random((r1 - r0, k)), side="right").clip(max=p - 1)
        blk.sort(axis=1)
        while True:
            dup = np.zeros_like(blk, dtype=bool)
            dup[:, 1:] = blk[:, 1:] == blk[:, :-1]
            cnt = int(dup.sum())
            if cnt == 0:
                break
            blk[dup] = np.searchsorted(cdf, rng.random(cnt), side="right").clip(max=p - 1)
            blk.sort(axis=1)
        out[r0:r1] = blk
    return out + col_offset


def _logistic_labels(rng, feats, n_planted, noise=0.1):
    p = feats.n_cols
    w = np.zeros(p)
    sup = rng.choice(p, size=min(n_planted, p), replace=False)
    w[sup] = rng.standard_normal(len(sup))
    m = feats.to_scipy() @ w + noise * rng.standard_normal(feats.n_rows)
    return np.where(m >= 0, 1.0, -1.0)


def config1(seed=0):
    """Lasso, fp64, 2000 x 500, Bernoulli(0.05), N(0,1), unit rows, lambda=1e-3, gamma=1/3."""
    rng = np.random.default_rng(seed)
    n, p = 2000, 500
    mask = rng.random((n, p)) < 0.05
    vals = rng.standard_normal((n, p))
    rows, cols = np.nonzero(mask)
    v = vals[rows, cols]
    norms = np.sqrt(np.bincount(rows, weights=v * v, minlength=n))
    v = v / np.where(norms[rows] > 0, norms[rows], 1.0)
    offsets = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=offsets[1:])
    feats = CsrMatrix(n, p, offsets, cols, v)
    w = np.zeros(p)
    sup = rng.choice(p, size=25, replace=False)
    w[sup] = rng.standard_normal(25)
    b = feats.to_scipy() @ w + 0.01 * rng.standard_normal(n)
    data = Dataset(feats, b)
    return dict(data=data, loss=Loss(SQUARED, 0.0), penalty=L1Penalty(1e-3), partition=singleton_partition(p),
                step=1.0 / 3.0, epochs=20, name="cfg1-lasso-2000x500")


def _zipf_logistic(rng, n, p, k, s, n_planted, binary=True, dtype=np.float32):
    cols = zipf_rows(rng, n, p, k, s)
    offsets = np.arange(n + 1, dtype=np.int64) * k
    vals = np.full(n * k, np.float32(1.0 / np.sqrt(k)) if dtype == np.float32 else 1.0 / np.sqrt(k),
                   dtype=dtype)
    feats = CsrMatrix(n, p, offsets, cols.reshape(-1), vals)
    y = _logistic_labels(rng, feats, n_planted)
    return Dataset(feats, y)


def config2(seed=0, n=100_000, p=50_000):
    """l1-logistic, fp32 values / int32 idx, 1e5 x 5e4, k=20 Zipf(1.1), lambda=1/n, 30 epochs."""
    rng = np.random.default_rng(seed)
    data = _zipf_logistic(rng, n, p, 20, 1.1, 500)
    lam = 1.0 / n
    return dict(data=data, loss=Loss(LOGISTIC, lam), penalty=L1Penalty(lam), partition=singleton_partition(p),
                step="1/2L", epochs=30, name=f"cfg2-l1logistic-{n}x{p}-zipf1.1")


def config5(seed=0, n=100_000, p=10_000_000, group=10):
    """group-lasso logistic path instance: config 2's generator, p=1e7, G=10."""
    rng = np.random.default_rng(seed)
    data = _zipf_logistic(rng, n, p, 20, 1.1, 500)
    lam1 = 1.0 / n
    part = contiguous_partition(p, group)
    return dict(data=data, loss=Loss(LOGISTIC, lam1), penalty=GroupL2Penalty(0.0), partition=part,
                step="1/2L", epochs=30, name=f"cfg5-grouplogistic-{n}x{p}-G{group}")


def baseline_config(k, seed=0, **kw):
    return {1: config1, 2: config2, 5: config5}[k](seed=seed, **kw)


# ---------------------------------------------------------------------------
# Configs 3 and 4 at full size: generated on the device (K7, csrc/gen.cu)

def _zipf_cdf(m, s):
    w = np.arange(1, m + 1, dtype=np.float64) ** (-s)
    c = np.cumsum(w)
    c /= c[-1]
    return c


def device_zipf_problem(n, p, k_dense, k_zipf, s, n_planted, lam2, lognormal, seed=0, device=None, noise=0.1,
                        **problem_kw):
    """Generate a logistic l1 problem on the device and wrap it in a
    DeviceProblem (lambda1 = 1/n, gamma rule 1/2L as configs 2-5)."""
    import torch

    from . import _lib
    from .device import DeviceProblem

    _lib.require_device()
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else int(device))
    k = k_dense + k_zipf
    nnz = n * k
    m = p - k_dense
    cdf = torch.from_numpy(_zipf_cdf(m, s)).to(dev)
    row_ptr = torch.empty(n + 1, dtype=torch.int64, device=dev)
    col = torch.empty(nnz, dtype=torch.int32, device=dev)
    val = torch.empty(nnz, dtype=torch.float32, device=dev)
    L = _lib.load()
    _lib.check(L.ps_gen_zipf_csr(n, k_dense, k_zipf, cdf.data_ptr(), m, seed, int(lognormal), row_ptr.data_ptr(),
                                 col.data_ptr(), val.data_ptr(), _lib.stream_ptr()))
    del cdf
    rng = np.random.default_rng(seed)
    w = np.zeros(p)
    sup = rng.choice(p, size=min(n_planted, p), replace=False)
    w[sup] = rng.standard_normal(len(sup))
    wt = torch.from_numpy(w).to(dev)
    y = torch.empty(n, dtype=torch.float32, device=dev)
    _lib.check(L.ps_gen_labels(n, k, col.data_ptr(), val.data_ptr(), wt.data_ptr(), noise, seed + 1, y.data_ptr(),
                               _lib.stream_ptr()))
    del wt
    if nnz < 2 ** 31 - 1:
        row_ptr = row_ptr.to(torch.int32)
    loss = Loss(LOGISTIC, 1.0 / n)
    pen = L1Penalty(lam2)
    dp = DeviceProblem.from_device_csr(row_ptr, col, val, y, p, loss, pen, None, device=dev, **problem_kw)
    return dict(problem=dp, loss=loss, penalty=pen, step="1/2L", k=k)


def config3(seed=0, n=20_000_000, p=30_000_000, **kw):
    """l1-logistic, n=2e7 x p=3e7, 30 distinct Zipf(1.2) columns per row, binary
    values row-normalised, planted w* with 10k nonzeros, lambda=1e-7, 10 epochs."""
    d = device_zipf_problem(n, p, 0, 30, 1.2, 10_000, 1e-7, False, seed=seed, **kw)
    d.update(epochs=10, name=f"cfg3-l1logistic-{n}x{p}-zipf1.2")
    return d


def config4(seed=0, n=45_000_000, p=1_000_000, **kw):
    """l1-logistic, n=4.5e7 x p=1e6, 13 dense columns + 22 Zipf(1.05) per row,
    lognormal(0,1) values row-normalised, planted w* with 2k nonzeros,
    lambda=1e-6, 5 epochs."""
    d = device_zipf_problem(n, p, 13, 22, 1.05, 2_000, 1e-6, True, seed=seed, **kw)
    d.update(epochs=5, name=f"cfg4-l1logistic-{n}x{p}-dense13+zipf1.05")
    return d
