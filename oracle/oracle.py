"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes front end of ``liboracle.so`` (the plain-C fp64 restatement of the
reference's Sparse Proximal SAGA path, see ``sps_oracle.c``) plus the numpy
glue that lays a problem out for it.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline legs import this
module; the product package (``paper_1707_06468_b200``) never does.

Reference anchors (``/root/reference/pkg/src/sparsesaga``):
  * ``run_sequential``  -> saga.py:217-259 (hot loop :248-256, step :169-185)
  * ``run_async``       -> asynchronous.py:131-210 (worker :80-117)
  * ``block_weights``   -> data.py:236-262
  * ``objective``       -> losses.py:134-136
  * ``fixed_point_residual`` -> saga.py:299-317
  * ``sample_sequence`` -> saga.py:45-51, 233-235; asynchronous.py:120-128
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "liboracle.so"

LOSSES = {"logistic": 0, "squared": 1}
PENALTIES = {"zero": 0, "l1": 1, "group": 2, "box": 3}

_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)


class _Problem(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64), ("p", ctypes.c_int64),
        ("row_ptr", _i64p), ("col", _i64p), ("val", _f64p), ("y", _f64p),
        ("n_blocks", ctypes.c_int64), ("block_of", _i64p), ("blk_ptr", _i64p),
        ("blk_coords", _i64p), ("d_B", _f64p),
        ("loss", ctypes.c_int), ("lambda1", ctypes.c_double),
        ("pen", ctypes.c_int), ("lam2", ctypes.c_double), ("lo", ctypes.c_double),
        ("hi", ctypes.c_double), ("singleton", ctypes.c_int),
    ]


_lib = None


def build():
    subprocess.run(["make", "-s", "-C", str(HERE), "all"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(LIB_PATH))
        L.oracle_block_weights.restype = ctypes.c_int64
        L.oracle_block_weights.argtypes = [ctypes.c_int64, _i64p, _i64p, ctypes.c_int64, _i64p,
                                           _i64p, _f64p, _f64p]
        L.oracle_run_sequential.restype = ctypes.c_int
        L.oracle_run_sequential.argtypes = [ctypes.POINTER(_Problem), ctypes.c_double, _i64p,
                                            ctypes.c_int64, _f64p, _f64p, _f64p]
        L.oracle_run_async.restype = ctypes.c_int
        L.oracle_run_async.argtypes = [ctypes.POINTER(_Problem), ctypes.c_double, ctypes.c_int,
                                       _i64p, _i64p, _f64p, _f64p, _f64p, _i64p, ctypes.c_int64]
        L.oracle_objective.restype = ctypes.c_double
        L.oracle_objective.argtypes = [ctypes.POINTER(_Problem), _f64p]
        L.oracle_smooth_gradient.restype = None
        L.oracle_smooth_gradient.argtypes = [ctypes.POINTER(_Problem), _f64p, _f64p]
        L.oracle_fixed_point_residual.restype = ctypes.c_double
        L.oracle_fixed_point_residual.argtypes = [ctypes.POINTER(_Problem), _f64p, ctypes.c_double]
        L.oracle_add_repeat_threads.restype = None
        L.oracle_add_repeat_threads.argtypes = [_f64p, ctypes.c_double, ctypes.c_int64, ctypes.c_int]
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t)


class OracleProblem:
    """A problem laid out for the C oracle (int64 CSR, fp64 values).

    ``block_of`` defaults to the singleton partition.  ``d_B`` is computed as
    data.py:259-261 does (``drop_dead_blocks=True`` semantics: dead -> 0).
    """

    def __init__(self, row_ptr, col, val, y, p, loss="logistic", lambda1=0.0,
                 penalty="l1", lam2=0.0, lo=-1.0, hi=1.0, block_of=None):
        self.row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
        self.col = np.ascontiguousarray(col, dtype=np.int64)
        self.val = np.ascontiguousarray(val, dtype=np.float64)
        self.y = np.ascontiguousarray(y, dtype=np.float64)
        self.n = len(self.row_ptr) - 1
        self.p = int(p)
        singleton = block_of is None
        if block_of is None:
            block_of = np.arange(self.p, dtype=np.int64)
        self.block_of = np.ascontiguousarray(block_of, dtype=np.int64)
        self.n_blocks = int(self.block_of.max()) + 1 if self.p else 0
        order = np.argsort(self.block_of, kind="stable")
        self.blk_coords = np.ascontiguousarray(order, dtype=np.int64)
        self.blk_ptr = np.zeros(self.n_blocks + 1, dtype=np.int64)
        np.cumsum(np.bincount(self.block_of, minlength=self.n_blocks), out=self.blk_ptr[1:])
        self.counts = np.zeros(self.n_blocks, dtype=np.int64)
        self.d_B = np.zeros(self.n_blocks)
        delta = ctypes.c_double(0.0)
        self.n_dead = int(lib().oracle_block_weights(
            self.n, _p(self.row_ptr, _i64p), _p(self.col, _i64p), self.n_blocks,
            _p(self.block_of, _i64p), _p(self.counts, _i64p), _p(self.d_B, _f64p),
            ctypes.byref(delta)))
        self.delta = delta.value
        self.loss, self.lambda1 = loss, float(lambda1)
        self.penalty, self.lam2, self.lo, self.hi = penalty, float(lam2), float(lo), float(hi)
        self._s = _Problem(self.n, self.p, _p(self.row_ptr, _i64p), _p(self.col, _i64p),
                           _p(self.val, _f64p), _p(self.y, _f64p), self.n_blocks,
                           _p(self.block_of, _i64p), _p(self.blk_ptr, _i64p),
                           _p(self.blk_coords, _i64p), _p(self.d_B, _f64p),
                           LOSSES[loss], self.lambda1, PENALTIES[penalty], self.lam2,
                           self.lo, self.hi, int(singleton))

    # -- reference: losses.py:99-105 ------------------------------------
    def lipschitz(self):
        c = 0.25 if self.loss == "logistic" else 1.0
        sq = np.zeros(self.n)
        nz = np.flatnonzero(np.diff(self.row_ptr) > 0)
        if len(nz):
            sq[nz] = np.add.reduceat(self.val ** 2, self.row_ptr[nz])
        return float((c * sq + self.lambda1).max())

    def run_sequential(self, gamma, samples, x=None, alpha=None, abar=None):
        samples = np.ascontiguousarray(samples, dtype=np.int64)
        x = np.zeros(self.p) if x is None else np.array(x, dtype=np.float64)
        alpha = np.zeros(self.n) if alpha is None else np.array(alpha, dtype=np.float64)
        abar = np.zeros(self.p) if abar is None else np.array(abar, dtype=np.float64)
        lib().oracle_run_sequential(ctypes.byref(self._s), float(gamma), _p(samples, _i64p),
                                    len(samples), _p(x, _f64p), _p(alpha, _f64p), _p(abar, _f64p))
        return x, alpha, abar

    def run_async(self, gamma, per_worker_samples, batch=100, state=None):
        """Hogwild workers from x0 = 0, or continuing ``state`` = (x, alpha, abar)
        arrays in place (checkpointed runs)."""
        seqs = [np.ascontiguousarray(s, dtype=np.int64) for s in per_worker_samples]
        flat = np.ascontiguousarray(np.concatenate(seqs)) if seqs else np.zeros(0, np.int64)
        counts = np.array([len(s) for s in seqs], dtype=np.int64)
        if state is None:
            x, alpha, abar = np.zeros(self.p), np.zeros(self.n), np.zeros(self.p)
        else:
            x, alpha, abar = state
        counter = np.zeros(1, dtype=np.int64)
        lib().oracle_run_async(ctypes.byref(self._s), float(gamma), len(seqs), _p(flat, _i64p),
                               _p(counts, _i64p), _p(x, _f64p), _p(alpha, _f64p), _p(abar, _f64p),
                               _p(counter, _i64p), int(batch))
        return x, alpha, abar, int(counter[0])

    def objective(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        return float(lib().oracle_objective(ctypes.byref(self._s), _p(x, _f64p)))

    def smooth_gradient(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        g = np.zeros(self.p)
        lib().oracle_smooth_gradient(ctypes.byref(self._s), _p(x, _f64p), _p(g, _f64p))
        return g

    def dual_objective(self, x):
        """Fenchel dual value at theta_i = -l'(a_i.x) (numpy restatement of the
        formulas ps_dual_objective evaluates; the reference has no dual, so
        this is pinned only by weak duality and by its zero gap at the optimum)."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        rows = np.repeat(np.arange(self.n), np.diff(self.row_ptr))
        z = np.bincount(rows, weights=self.val * x[self.col], minlength=self.n)
        b = self.y
        if self.loss == "logistic":
            t = -b * z
            with np.errstate(over="ignore"):
                sig = np.where(t > 0, 1.0 / (1.0 + np.exp(-t)), np.exp(t) / (1.0 + np.exp(t)))
            s = -b * sig
        else:
            s = z - b

        def conj(sv):
            if self.loss == "logistic":
                t = -b * sv
                r = np.zeros_like(t)
                pos, lt1 = t > 0, t < 1
                r[pos] += t[pos] * np.log(t[pos])
                r[lt1] += (1 - t[lt1]) * np.log1p(-t[lt1])
                return r
            return 0.5 * sv * sv + sv * b

        w = np.bincount(self.col, weights=self.val * s[rows], minlength=self.p)
        v = -w / self.n
        l1, lam2 = self.lambda1, self.lam2
        if self.penalty == "group":
            norms = np.array([np.linalg.norm(v[self.blk_coords[self.blk_ptr[k]:self.blk_ptr[k + 1]]])
                              for k in range(self.n_blocks)])
            vmax = norms.max() if len(norms) else 0.0
            gstar = np.sum(np.maximum(norms - lam2, 0.0) ** 2) / (2 * l1) if l1 > 0 else 0.0
        else:
            vmax = np.abs(v).max() if len(v) else 0.0
            if self.penalty == "l1":
                gstar = np.sum(np.maximum(np.abs(v) - lam2, 0.0) ** 2) / (2 * l1) if l1 > 0 else 0.0
            elif self.penalty == "box":
                if l1 > 0:
                    c = np.clip(v / l1, self.lo, self.hi)
                    gstar = np.sum(v * c - 0.5 * l1 * c * c)
                else:
                    gstar = np.sum(np.maximum(v * self.lo, v * self.hi))
            else:
                if l1 > 0:
                    gstar = np.sum(v * v) / (2 * l1)
                else:
                    return -np.inf if vmax > 0 else -np.sum(conj(s)) / self.n
        if l1 <= 0 and self.penalty in ("l1", "group") and vmax > lam2:
            s = s * (lam2 / vmax)
        return float(-np.sum(conj(s)) / self.n - gstar)

    def fixed_point_residual(self, x, gamma):
        x = np.ascontiguousarray(x, dtype=np.float64)
        return float(lib().oracle_fixed_point_residual(ctypes.byref(self._s), _p(x, _f64p), float(gamma)))


def from_dataset(data, loss, penalty, partition=None):
    """Lay out a (duck-typed) reference/product Dataset + Loss + Penalty."""
    f = data.features
    kind = type(penalty).__name__
    pen = {"ZeroPenalty": "zero", "L1Penalty": "l1", "GroupL2Penalty": "group",
           "BoxPenalty": "box"}[kind]
    block_of = None
    if partition is not None and not (partition.n_blocks == partition.n_coords
                                      and np.array_equal(partition.block_of, np.arange(partition.n_coords))):
        block_of = partition.block_of
    return OracleProblem(f.row_offsets, f.col_indices, f.values, data.labels, f.n_cols,
                         loss=loss.kind, lambda1=loss.lambda1, penalty=pen,
                         lam2=getattr(penalty, "lam2", 0.0), lo=getattr(penalty, "lo", -1.0),
                         hi=getattr(penalty, "hi", 1.0), block_of=block_of)


def sample_sequence(seed, n, count, worker_id=0):
    """saga.py:45-51 + :233-235 — numpy PCG64 seeded with [seed, worker]."""
    return np.random.default_rng([int(seed), int(worker_id)]).integers(0, n, size=count)


def split_iterations(total, threads):
    """asynchronous.py:125-128."""
    base = total // threads
    return [base + (1 if w < total % threads else 0) for w in range(threads)]


def add_repeat_threads(cell, delta, count, threads):
    lib().oracle_add_repeat_threads(_p(cell, _f64p), float(delta), int(count), int(threads))
