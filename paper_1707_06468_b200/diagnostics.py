"""Suboptimality bookkeeping and the certified optimum F* (diagnostics.py of
the reference, the parts the solver path and the CLI consume).

``reference_optimum`` follows diagnostics.py:153-200: solve with a growing
epoch budget until the weighted fixed-point residual (saga.py:299-317) drops
below the target, cache x*, F(x*) and the residual on disk keyed by the
problem hash.  The solves run on the device (run_sequential: the
deterministic replay of the reference's own sample stream); the reference's
``solver="dense"`` choice (dense SAGA, out of this repo's scope) is accepted
and served by the same sparse solver -- both certify the same optimum to the
residual target.
"""

from __future__ import annotations

import hashlib
import os
from pathlib import Path

import numpy as np

from .losses import full_objective
from .saga import SolverConfig, resolve_step_size, run_sequential


class StaleOptimumError(RuntimeError):
    """A trace objective dropped below the cached optimum (diagnostics.py:21-22)."""


def suboptimality(trace_objectives, xstar_objective, slack=1e-12):
    """Per-checkpoint absolute gaps clamped at zero within ``slack``
    (diagnostics.py:25-34)."""
    out = []
    for obj in trace_objectives:
        gap = obj - xstar_objective
        if gap < -slack:
            raise StaleOptimumError(f"objective {obj} is {-gap:.3e} below the cached optimum")
        out.append(max(gap, 0.0))
    return out


def default_cache_dir():
    """$SPARSESAGA_CACHE_DIR, else ~/.cache/sparsesaga (diagnostics.py:135-139)."""
    env = os.environ.get("SPARSESAGA_CACHE_DIR")
    return Path(env) if env else Path.home() / ".cache" / "sparsesaga"


def problem_hash(data, loss, penalty, partition, extra=""):
    """SHA-256 over the dataset bytes and the problem description
    (diagnostics.py:142-150)."""
    h = hashlib.sha256()
    f = data.features
    block_of = partition.block_of if partition is not None else np.arange(data.n_features, dtype=np.int64)
    for arr in (f.row_offsets, f.col_indices, f.values, data.labels, block_of):
        h.update(np.ascontiguousarray(arr).tobytes())
    h.update(f"{loss.kind}|{loss.lambda1!r}|{penalty!r}|{extra}".encode())
    return h.hexdigest()


def reference_optimum(data, loss, penalty, partition, cache_dir=None, solver="dense", step="1/5L",
                      max_epochs=5000, residual_target=1e-9, check_every=25, device=None):
    """Certified high-precision solution, cached by problem hash
    (diagnostics.py:153-200).  Returns {"x", "objective", "residual", "cached"}."""
    if solver not in ("dense", "sparse"):
        raise ValueError(f"unknown solver {solver!r}")
    cache_dir = Path(cache_dir) if cache_dir is not None else default_cache_dir()
    key = problem_hash(data, loss, penalty, partition,
                       extra=f"opt|{solver}|{step}|{max_epochs}|{residual_target}|b200")
    path = cache_dir / f"optimum-{key}.npz"
    if path.exists():
        blob = np.load(path, allow_pickle=False)
        return {"x": blob["x"], "objective": float(blob["objective"]), "residual": float(blob["residual"]),
                "cached": True}
    best_x, best_res, done, seed = None, np.inf, 0, 9999
    while done < max_epochs:
        chunk = min(check_every, max_epochs - done)
        cfg = SolverConfig(step_size=step, epochs=done + chunk, seed=seed,
                           checkpoint_every=data.n_samples * (done + chunk))
        # re-run from scratch with a growing budget, as the reference does
        trace = run_sequential(data, loss, penalty, partition, cfg, device=device)
        dp = trace.device_problem
        gamma = resolve_step_size(step, dp.L, data.n_samples, loss.lambda1 if loss.lambda1 > 0 else None)
        done += chunk
        res = dp.fixed_point_residual(gamma)  # of the final iterate, on the solve's own partition
        if res < best_res:
            best_res, best_x = res, trace.final_x
        if best_res <= residual_target:
            break
        check_every *= 2
    objective = full_objective(data, loss, penalty, best_x, partition)
    cache_dir.mkdir(parents=True, exist_ok=True)
    np.savez(path, x=best_x, objective=objective, residual=best_res)
    return {"x": best_x, "objective": float(objective), "residual": float(best_res), "cached": False}


def theorem_rate_factor(n, kappa, a=1.0):
    """Geometric rate factor of the sequential solver at step a/(5L)
    (diagnostics.py:60-62; PAPER Theorem 1)."""
    return 0.2 * min(1.0 / n, a / kappa)


def theorem_constant(data, loss, xstar, L):
    """Envelope constant ||x0 - x*||^2 + sum_i ||grad f_i(x*)||^2 / (5 L^2)
    with x0 = 0 and zero-initialised memory (diagnostics.py:65-81).  The
    per-sample gradients at x* are formed from the device margins; the sum
    over i of ||l'_i a_i + lambda1 x*||^2 expands to
    l'_i^2 ||a_i||^2 + 2 lambda1 l'_i (a_i.x*) + lambda1^2 ||x*||^2."""
    import torch

    from . import _lib

    _lib.require_device()
    f = data.features
    ro = np.asarray(f.row_offsets, dtype=np.int64)
    cols = np.asarray(f.col_indices, dtype=np.int64)
    vals = np.asarray(f.values, dtype=np.float64)
    xs = np.asarray(xstar, dtype=np.float64)
    lens = np.diff(ro)
    starts = np.minimum(ro[:-1], max(len(vals) - 1, 0))
    z = np.where(lens > 0, np.add.reduceat(vals * xs[cols], starts), 0.0) if len(vals) else np.zeros(len(lens))
    sq = np.where(lens > 0, np.add.reduceat(vals * vals, starts), 0.0) if len(vals) else np.zeros(len(lens))
    # l'(z_i, b_i) by the library's loss code (ps_loss_deriv, the deterministic kernels' arithmetic)
    zd = torch.from_numpy(np.ascontiguousarray(z)).cuda()
    bd = torch.from_numpy(np.ascontiguousarray(data.labels, dtype=np.float64)).cuda()
    out = torch.empty_like(zd)
    _lib.check(_lib.load().ps_loss_deriv(_lib.LOSS[loss.kind], 0, zd.data_ptr(), bd.data_ptr(), zd.numel(),
                                         out.data_ptr(), _lib.stream_ptr()))
    deriv = out.cpu().numpy()
    lam = loss.lambda1
    acc = float(np.sum(deriv ** 2 * sq + 2.0 * lam * deriv * z) + data.n_samples * lam * lam * float(xs @ xs))
    return float(xs @ xs) + acc / (5.0 * L ** 2)


def rate_envelope_check(distance_checkpoints, rho, C0, slack):
    """Median squared distances against (1 - rho)^t C0 slack
    (diagnostics.py:37-57): one record per checkpoint."""
    if not 0 < rho < 1:
        raise ValueError("rho must be in (0, 1)")
    records = []
    for t, dist in sorted(distance_checkpoints.items()):
        bound = (1.0 - rho) ** t * C0 * slack
        records.append({"iteration": int(t), "distance": float(dist), "bound": float(bound),
                        "passed": bool(dist <= bound), "margin": float(bound - dist)})
    return records
