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
