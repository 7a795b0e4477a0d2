"""Reuse of uploaded problems across the reference-style helper calls.

The reference's helpers (``lipschitz_constant``, ``full_objective``,
``smooth_gradient``, ``fixed_point_residual``, ``resync_average`` and the
step-level entry points ``sps_step`` / ``worker_iteration`` /
``sparse_gradient_estimate``) take the dataset on every call.  Building a
``DeviceProblem`` per call re-uploads the CSR and re-runs ps_prepare (and the
hot layout), which dominates loops such as the lambda_max bisection of
``gen_regularization`` or a step-by-step replay.  ``problem_for`` keeps the
last few uploads, keyed by the identity of the feature matrix, labels and
partition objects (held through weak references, so a freed dataset never
matches a new one that reuses its address), and re-targets the cached
problem to the call's loss and penalty (plain parameters of the launches).
Arrays mutated in place after an upload are not detected: pass a new object.
"""

from __future__ import annotations

import collections
import weakref

from . import _lib

_MAX_ENTRIES = 8
_entries: "collections.OrderedDict[tuple, tuple]" = collections.OrderedDict()


def _ref(obj):
    if obj is None:
        return lambda: None
    try:
        return weakref.ref(obj)
    except TypeError:  # not weak-referenceable: keep it alive with the entry
        return lambda o=obj: o


def configure(dp, loss, penalty):
    """Point a DeviceProblem at another loss / penalty of the same structure."""
    from .penalties import penalty_code

    dp.loss_kind = loss.kind if loss is not None else "squared"
    dp.lambda1 = float(loss.lambda1) if loss is not None else 0.0
    if penalty is None:
        dp.pen_code, dp.lam2, dp.lo, dp.hi = _lib.PEN_ZERO, 0.0, -1.0, 1.0
    else:
        dp.pen_code, dp.lam2, dp.lo, dp.hi = penalty_code(penalty)
    dp.L = (0.25 if dp.loss_kind == "logistic" else 1.0) * float(dp.stats.max_row_sqnorm) + dp.lambda1
    return dp


def problem_for(data, loss, penalty, partition, device=None, hot_max=None):
    """A DeviceProblem for (data, partition), reused across calls, configured
    for ``loss`` / ``penalty``.  Dead blocks are allowed (d_B = 0), as in a
    support index built with drop_dead_blocks."""
    import torch

    from .device import DeviceProblem
    from .penalties import penalty_code

    _lib.require_device()
    features = data.features if hasattr(data, "features") else data
    labels = getattr(data, "labels", None)
    dev = torch.cuda.current_device() if device is None else (
        device.index if isinstance(device, torch.device) else int(device))
    group = penalty is not None and penalty_code(penalty)[0] == _lib.PEN_GROUP
    key = (id(features), id(labels), id(partition), group, dev, hot_max)
    hit = _entries.get(key)
    if hit is not None:
        refs, dp = hit
        if refs[0]() is features and refs[1]() is labels and refs[2]() is partition:
            _entries.move_to_end(key)
            return configure(dp, loss, penalty)
        del _entries[key]
    dp = DeviceProblem(data, loss, penalty, partition, device=dev, drop_dead_blocks=True, hot_max=hot_max)
    _entries[key] = ((_ref(features), _ref(labels), _ref(partition)), dp)
    while len(_entries) > _MAX_ENTRIES:
        _entries.popitem(last=False)
    return dp


def clear():
    _entries.clear()
