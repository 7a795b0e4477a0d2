"""Loss descriptors and device-evaluated smooth terms (mirrors losses.py:1-136).

``Loss`` is the reference's frozen descriptor.  The objective, smooth value,
gradient and Lipschitz constant are computed by the CUDA library
(ps_objective / ps_smooth_gradient / ps_prepare); there is no host
implementation of the math.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

LOGISTIC = "logistic"
SQUARED = "squared"

# losses.py:19 — upper bounds on the scalar second derivative.
_CURVATURE = {LOGISTIC: 0.25, SQUARED: 1.0}


@dataclass(frozen=True)
class Loss:
    kind: str
    lambda1: float = 0.0

    def __post_init__(self):
        if self.kind not in _CURVATURE:
            raise ValueError(f"unknown loss kind {self.kind!r}")
        if self.lambda1 < 0:
            raise ValueError("lambda1 must be nonnegative")

    @property
    def curvature(self):
        return _CURVATURE[self.kind]


@dataclass(frozen=True)
class SmoothnessInfo:
    """L = c * max_i ||a_i||^2 + lambda1 (losses.py:89-105)."""

    L: float
    max_row_sqnorm: float

    @property
    def max_L(self):
        return self.L


def lipschitz_constant(data, loss, device=None):
    """Device max row norm -> L (losses.py:99-105)."""
    if data.n_samples == 0:
        raise ValueError("dataset is empty")
    from . import _cache

    dp = _cache.problem_for(data, loss, None, None, device=device)
    msq = float(dp.stats.max_row_sqnorm)
    return SmoothnessInfo(L=_CURVATURE[loss.kind] * msq + loss.lambda1, max_row_sqnorm=msq)


def loss_scalar(kind, z, b):
    """(value, derivative) of the scalar loss at margin z with label b
    (losses.py:73-86), evaluated by the device's loss code (ps_loss_eval)."""
    import torch

    from . import _lib

    if kind not in _CURVATURE:
        raise ValueError(f"unknown loss kind {kind!r}")
    _lib.require_device()
    dev = torch.device("cuda", torch.cuda.current_device())
    t = torch.tensor([float(z), float(b), 0.0, 0.0], dtype=torch.float64, device=dev)
    _lib.check(_lib.load().ps_loss_eval(_lib.LOSS[kind], t.data_ptr(), t.data_ptr() + 8, 1, t.data_ptr() + 16,
                                        t.data_ptr() + 24, _lib.stream_ptr()))
    out = t[2:].cpu().numpy()
    return float(out[0]), float(out[1])


def _problem(data, loss, penalty, partition, device):
    from . import _cache
    from .penalties import ZeroPenalty

    return _cache.problem_for(data, loss, penalty if penalty is not None else ZeroPenalty(), partition,
                              device=device)


def full_objective(data, loss, penalty, x, partition=None, device=None):
    """F(x) = mean loss + (lambda1/2)||x||^2 + h(x), on the device (losses.py:134-136).

    Without a partition a group penalty is the whole-vector norm
    (penalties.py:99-100), as in the reference."""
    from .data import single_block_partition

    if partition is None and type(penalty).__name__ == "GroupL2Penalty":
        partition = single_block_partition(data.n_features)
    dp = _problem(data, loss, penalty, partition, device)
    return dp.objective_of(np.asarray(x, dtype=np.float64))


def smooth_value(data, loss, x, device=None):
    dp = _problem(data, loss, None, None, device)
    parts = dp.objective_parts_of(np.asarray(x, dtype=np.float64))
    return parts[0] + parts[1]


def smooth_gradient(data, loss, x, device=None):
    """A^T l'(Ax)/n + lambda1 x on the device (losses.py:118-122)."""
    dp = _problem(data, loss, None, None, device)
    return dp.smooth_gradient_of(np.asarray(x, dtype=np.float64))
