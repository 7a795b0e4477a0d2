"""Sequential Sparse Proximal SAGA on the device (mirrors saga.py:1-337).

``run_sequential`` keeps the reference's signature, sample stream and trace
contract (saga.py:217-259): x0 = 0, zero memory, the whole sample sequence
``default_rng([seed, 0]).integers(0, n, epochs*n)`` drawn up front, an
objective checkpoint at iteration 0 and every ``checkpoint_every`` updates,
optional ``tolerance`` early stop.  The updates themselves are replayed on
one warp by ps_run in deterministic mode, fp64, in sps_step's arithmetic
order, so iterates agree with the reference to rounding.
"""

from __future__ import annotations

import json
import time
from dataclasses import dataclass, field

import numpy as np

STEP_RULES = ("1/5L", "1/2L", "1/36L", "1/36nmu")


def resolve_step_size(step, L, n=None, mu=None):
    """Rule string or explicit float -> step size (saga.py:25-42)."""
    if isinstance(step, (int, float)):
        if step <= 0:
            raise ValueError("step size must be positive")
        return float(step)
    rule = step.replace(" ", "")
    if rule == "1/5L":
        return 1.0 / (5.0 * L)
    if rule == "1/2L":
        return 1.0 / (2.0 * L)
    if rule == "1/36L":
        return 1.0 / (36.0 * L)
    if rule == "1/36nmu":
        if n is None or mu is None or mu <= 0:
            raise ValueError("rule 1/36nmu needs n and mu > 0")
        return 1.0 / (36.0 * n * mu)
    raise ValueError(f"unknown step rule {step!r}; known: {STEP_RULES}")


def worker_rng(seed, worker_id=0):
    """Stream (seed, worker_id) — identical to saga.py:45-51."""
    return np.random.default_rng([int(seed), int(worker_id)])


@dataclass
class GradientMemory:
    """Host view of the scalar memory + running average (saga.py:54-72)."""

    scalars: np.ndarray
    avg: np.ndarray

    @classmethod
    def zeros(cls, n, p):
        return cls(scalars=np.zeros(n), avg=np.zeros(p))

    @property
    def n(self):
        return len(self.scalars)


@dataclass
class SolverConfig:
    step_size: object = "1/5L"
    epochs: int = 100
    seed: int = 0
    checkpoint_every: int = None
    tolerance: float = 0.0

    def __post_init__(self):
        if self.epochs < 1:
            raise ValueError("epochs must be >= 1")
        if isinstance(self.step_size, (int, float)) and self.step_size <= 0:
            raise ValueError("step size must be positive")
        if self.checkpoint_every is not None and self.checkpoint_every < 1:
            raise ValueError("checkpoint_every must be >= 1")


@dataclass
class Trace:
    """Checkpoint rows + final iterate (saga.py:98-139), same CSV/JSON output."""

    iterations: list = field(default_factory=list)
    epochs: list = field(default_factory=list)
    objective: list = field(default_factory=list)
    wall_seconds: list = field(default_factory=list)
    threads: list = None
    distances: list = None
    final_x: np.ndarray = None
    meta: dict = field(default_factory=dict)

    def append(self, iteration, n, objective, wall, distance=None, threads=None):
        self.iterations.append(int(iteration))
        self.epochs.append(iteration / n)
        self.objective.append(float(objective))
        self.wall_seconds.append(float(wall))
        if distance is not None:
            if self.distances is None:
                self.distances = []
            self.distances.append(float(distance))
        if threads is not None:
            if self.threads is None:
                self.threads = []
            self.threads.append(int(threads))

    def to_csv(self, path):
        header = ["iterations", "epochs", "objective", "wall_seconds"]
        columns = [self.iterations, self.epochs, self.objective, self.wall_seconds]
        if self.threads is not None:
            header += ["threads", "counter_iterations"]
            columns += [self.threads, self.iterations]
        with open(path, "w") as fh:
            fh.write(",".join(header) + "\n")
            for row in zip(*columns):
                fh.write(",".join(repr(v) if isinstance(v, float) else str(v) for v in row) + "\n")

    def write_sidecar(self, path):
        with open(path, "w") as fh:
            json.dump(self.meta, fh, indent=2, default=_json_default)
            fh.write("\n")


def _json_default(obj):
    if isinstance(obj, np.ndarray):
        return obj.tolist()
    if isinstance(obj, (np.integer, np.floating)):
        return obj.item()
    return str(obj)


def _problem(data, loss, penalty, partition, index, device):
    from .device import DeviceProblem

    drop = bool(index is not None and len(getattr(index, "dropped_blocks", [])) > 0)
    return DeviceProblem(data, loss, penalty, partition, device=device, drop_dead_blocks=drop)


def _prepare(dp, loss, config, n):
    mu = loss.lambda1
    gamma = resolve_step_size(config.step_size, dp.L, n, mu if mu > 0 else None)
    return gamma


def _run_meta(dp, data, loss, penalty, config, gamma, threads, algorithm="sparse-saga"):
    mu = loss.lambda1
    return {
        "algorithm": algorithm,
        "n_samples": data.n_samples,
        "n_features": data.n_features,
        "loss": loss.kind,
        "lambda1": loss.lambda1,
        "penalty": repr(penalty),
        "step_size": gamma,
        "step_rule": config.step_size if isinstance(config.step_size, str) else None,
        "epochs": config.epochs,
        "seed": config.seed,
        "threads": threads,
        "L": dp.L,
        "kappa": dp.L / mu if mu > 0 else None,
        "delta": dp.delta,
        "device": str(dp.device),
        "value_dtype": "float32" if dp.value_type == 0 else "float64",
        "partition": dp.part_kind,
    }


def run_sequential(data, loss, penalty, partition, config, index=None, track_distance_to=None,
                   device=None):
    """Deterministic SPS from x0 = 0 (saga.py:217-259) on the device.

    The sample sequence is the reference's; segments between checkpoints are
    replayed by one ps_run call each; the objective is evaluated on the device.
    """
    dp = _problem(data, loss, penalty, partition, index, device)
    n = data.n_samples
    gamma = _prepare(dp, loss, config, n)
    every = config.checkpoint_every or n
    total = config.epochs * n
    samples_np = worker_rng(config.seed, 0).integers(0, n, size=total)
    samples = dp.torch.from_numpy(samples_np).to(dp.device)
    trace = Trace(meta=_run_meta(dp, data, loss, penalty, config, gamma, threads=1))
    track = track_distance_to is not None
    start = time.perf_counter()

    def checkpoint(t):
        obj = dp.objective()
        dist = float(np.sum((dp.x() - track_distance_to) ** 2)) if track else None
        trace.append(t, n, obj, time.perf_counter() - start, distance=dist)

    checkpoint(0)
    last_epoch_obj = trace.objective[0]
    done = 0
    while done < total:
        # one replay per checkpoint segment; the tolerance test runs where the
        # reference's does: at checkpoints that are also epoch ends (saga.py:248-256)
        nxt = min(total, (done // every + 1) * every)
        dp.replay(samples[done:nxt], gamma)
        done = nxt
        checkpoint(done)
        if config.tolerance > 0 and done % n == 0:
            if abs(trace.objective[-1] - last_epoch_obj) < config.tolerance:
                break
            last_epoch_obj = trace.objective[-1]
    trace.final_x = dp.x()
    trace.meta["iterations_run"] = trace.iterations[-1]
    trace.device_problem = dp
    return trace


def sps_steps(dp, samples, gamma):
    """Replay explicit steps on an existing DeviceProblem (sps_step, saga.py:169-185)."""
    dp.replay(samples, gamma)


def fixed_point_residual(x, data, loss, penalty, index, gamma, device=None):
    """||x - prox_{gamma D phi}(x - gamma D grad f(x))|| on the device (saga.py:299-317)."""
    if gamma <= 0:
        raise ValueError("gamma must be positive")
    from . import _cache

    partition = index.partition if index is not None else None
    dp = _cache.problem_for(data, loss, penalty, partition, device=device)
    dp.set_x(x)
    return dp.fixed_point_residual(gamma)


def resync_average(memory, data, device=None):
    """avg = A^T scalars / n on the device (saga.py:75-78)."""
    from . import _cache
    from .losses import Loss

    dp = _cache.problem_for(data, Loss("squared"), None, None, device=device)
    dp.alpha.copy_(dp.torch.from_numpy(np.asarray(memory.scalars, dtype=np.float64)))
    dp.resync_average()
    memory.avg[:] = dp.abar()
    return memory
