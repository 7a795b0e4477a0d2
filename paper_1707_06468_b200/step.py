"""The reference's step-level entry points, executed by the device kernel.

``sps_step`` (saga.py:169-185), ``sparse_gradient_estimate`` (saga.py:150-166)
and ``worker_iteration`` (asynchronous.py:80-117) keep their signatures and
their in-place semantics on the caller's host arrays.  Each call moves only
the extended support T_i of the sampled row: x^ and abar^ on T_i and
alpha_i go up into a cached device problem (``_cache.problem_for``, no hot
layout so coordinates keep their ids), ONE deterministic step runs through
``ps_run`` (the same kernel code as ``run_sequential``'s replay), and the
updated coordinates -- plus the step's gradient estimate v and applied delta
z - x^, written by the kernel through ``ps_sched_t.trace_v / trace_dx`` --
come back.  A loop of these calls therefore reproduces the device replay
(and the reference's iterates to ~1e-15); it is the API for reference-style
drivers and checks (verify.py:283-329, 384-404), not a fast path.
"""

from __future__ import annotations

import numpy as np

from . import _cache


def _ext_coords(index, features, i):
    """Sorted coordinates of T_i (the blocks touching row i's support)."""
    cols = np.asarray(features.row(i)[0], dtype=np.int64)
    part = index.partition
    bo = np.asarray(part.block_of)
    if len(cols) == 0:
        return np.empty(0, dtype=np.int64), cols
    if len(bo) == features.n_cols and part.n_blocks == features.n_cols and np.array_equal(bo[cols], cols):
        return cols, cols  # singleton blocks: T_i = S_i
    blocks = np.unique(bo[cols])
    coords = np.sort(np.concatenate([np.asarray(part.blocks[b], dtype=np.int64) for b in blocks]))
    return coords, cols


class _Bufs:
    """Per-problem device buffers of the step traces."""

    def __init__(self, dp):
        torch = dp.torch
        self.v = torch.zeros(dp.p_dev, dtype=torch.float64, device=dp.device)
        self.dx = torch.zeros(dp.p_dev, dtype=torch.float64, device=dp.device)


def _device_step(x, avg, scalars, i, gamma, penalty, index, loss, data):
    """One device step on sample i from (x, avg, scalars); returns
    (ecols, cols, x_new[ecols], avg_new[ecols], new_scalar, v, dx)."""
    dp = _cache.problem_for(data, loss, penalty, index.partition, hot_max=0)
    torch = dp.torch
    i = int(i)
    if not 0 <= i < dp.n:
        raise IndexError("sample index out of range")
    ecols, cols = _ext_coords(index, data.features, i)
    bufs = getattr(dp, "_step_bufs", None)
    if bufs is None:
        bufs = dp._step_bufs = _Bufs(dp)
    with torch.cuda.device(dp.device):
        ec = torch.from_numpy(ecols).to(dp.device)
        if len(ecols):
            state = np.stack([np.asarray(x, dtype=np.float64)[ecols], np.asarray(avg, dtype=np.float64)[ecols]], 1)
            dp.coord[ec, 0:2] = torch.from_numpy(state).to(dp.device)
        dp.alpha[i] = float(scalars[i])
        dp.replay(np.array([i], dtype=np.int64), float(gamma), trace=(bufs.v.data_ptr(), bufs.dx.data_ptr()))
        out = torch.stack([dp.coord[ec, 0], dp.coord[ec, 1], bufs.v[ec], bufs.dx[ec]]).cpu().numpy()
        new = float(dp.alpha[i].item())
    return ecols, cols, out[0], out[1], new, out[2], out[3]


def sps_step(x, memory, i, gamma, penalty, index, loss, data):
    """One sparse proximal step in place on x / memory (saga.py:169-185)."""
    if not gamma > 0:
        raise ValueError("gamma must be positive")
    ecols, cols, xn, an, new, _, _ = _device_step(x, memory.avg, memory.scalars, i, gamma, penalty, index,
                                                  loss, data)
    x[ecols] = xn
    memory.avg[ecols] = an  # only S_i moved; T_i \\ S_i comes back unchanged
    memory.scalars[int(i)] = new


def sparse_gradient_estimate(i, x, memory, index, loss, data):
    """(coords, v, new_scalar) of sample i at (x, memory) (saga.py:150-166);
    the caller's arrays are not modified."""
    ecols, _, _, _, new, v, _ = _device_step(x, memory.avg, memory.scalars, i, 1.0, None, index, loss, data)
    return ecols, v, new


class SharedState:
    """Host mirror of the shared solver state (asynchronous.py:44-72): x and
    avg per coordinate, the scalar memory per sample, the iteration counter.
    The asynchronous solve itself keeps this state on the device
    (DeviceProblem.coord / alpha / counter); ``from_device`` snapshots it."""

    def __init__(self, n, p):
        self.x = np.zeros(p)
        self.avg = np.zeros(p)
        self.scalars = np.zeros(n)
        self.counter = np.zeros(1, dtype=np.int64)
        self._all_coords = np.arange(p, dtype=np.int64)

    @classmethod
    def from_device(cls, dp, iterations=0):
        s = cls(dp.n, dp.p)
        s.x[:] = dp.x()
        s.avg[:] = dp.abar()
        s.scalars[:] = dp.alpha.cpu().numpy()
        s.counter[0] = int(iterations)
        return s

    def read_coords(self, coords, out=None):
        coords = np.asarray(coords, dtype=np.int64)
        if len(coords) and (coords.min() < 0 or coords.max() >= len(self.x)):
            raise IndexError("coordinate index out of range")
        if out is None:
            out = np.empty(len(coords))
        out[:] = self.x[coords]
        return out

    def snapshot_x(self):
        return self.read_coords(self._all_coords)

    def counter_value(self):
        return int(self.counter[0])

    def bump_counter(self, k):
        self.counter[0] += int(k)


def worker_iteration(shared, i, gamma, penalty, index, loss, data):
    """One lock-free iteration on sample i (asynchronous.py:80-117); returns
    the applied x delta on T_i.  Runs the device step: with one caller it is
    the sequential step, as the reference's one-thread run is."""
    if not gamma > 0:
        raise ValueError("gamma must be positive")
    ecols, cols, xn, an, new, _, dx = _device_step(shared.x, shared.avg, shared.scalars, i, gamma, penalty, index,
                                                   loss, data)
    shared.x[ecols] = xn
    shared.avg[ecols] = an
    shared.scalars[int(i)] = new
    return dx
