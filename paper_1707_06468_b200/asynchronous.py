"""ProxASAGA on the device (mirrors asynchronous.py:1-298).

``run_async`` keeps the reference's signature and trace contract
(asynchronous.py:131-210).  The reference's Python worker threads become
resident warps of one persistent kernel (ps_run, async mode): the call's
sample slots are split statically over the warps (the reference's
split_iterations, :125-128), each warp draws its rows from an on-device
counter-based sampler, reads x / abar inconsistently and commits with REDs /
atomic exchanges (hot columns through per-CTA staging).  The monitor
(:187-198) is the live one: ONE launch for the whole solve, a progress
counter bumped every 16 updates of a warp, and at each checkpoint mark a
copy-engine snapshot of the running solve (ps_run_monitored) -- for very
large problems an x-only device snapshot copied by a few CTAs beside the
solve; the stop-the-world schedule (one launch per segment) remains for
snapshots that fit neither and for distance tracking.

``config.threads == 1`` replays worker 0's reference sample stream on a single
warp, so a 1-thread run equals ``run_sequential`` bit for bit, as in the
reference (test_async.py:105-112).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np

from .saga import SolverConfig, Trace, _prepare, _problem, _run_meta, worker_rng


@dataclass
class AsyncConfig(SolverConfig):
    threads: int = 1
    counter_batch: int = 100
    warps: int = None           # resident warps (None: library default grid) when threads > 1
    warps_per_cta: int = 0      # 0: library default
    contention: float = 4.0     # c of gamma_j = gamma * min(1, c * D_j / tau); 0 = plain gamma
    group_batched: bool = True  # group lasso on contiguous blocks: the lambda-batched kernel with one state

    def __post_init__(self):
        super().__post_init__()
        if self.threads < 1:
            raise ValueError("threads must be >= 1")
        if self.counter_batch < 1:
            raise ValueError("counter_batch must be >= 1")
        if self.warps is not None and self.warps < 1:
            raise ValueError("warps must be >= 1")


def worker_sample_sequence(seed, worker_id, count, n):
    """asynchronous.py:120-122."""
    return worker_rng(seed, worker_id).integers(0, n, size=count)


def split_iterations(total, threads):
    """asynchronous.py:125-128."""
    base = total // threads
    return [base + (1 if w < total % threads else 0) for w in range(threads)]


def _grid(dp, config):
    """(ctas, warps_per_cta) launching exactly config.warps warps: warps per CTA
    = the largest divisor of the count up to 8 (one CTA of all of them up to
    32), unless warps_per_cta is given (then ctas * wpc may round down)."""
    if config.warps is None:
        return 0, config.warps_per_cta
    w = int(config.warps)
    if config.warps_per_cta:
        wpc = int(config.warps_per_cta)
    elif w <= 32:
        wpc = w
    else:
        wpc = max(d for d in range(1, 9) if w % d == 0)
    return max(1, w // wpc), wpc


def run_async(data, loss, penalty, partition, config, index=None, track_distance_to=None, max_threads=64,
              device=None):
    """Lock-free ProxASAGA (asynchronous.py:131-210) on the device."""
    if config.threads > max_threads:
        raise ValueError(f"threads={config.threads} exceeds the cap of {max_threads}")
    dp = _problem(data, loss, penalty, partition, index, device)
    n = data.n_samples
    gamma = _prepare(dp, loss, config, n)
    every = config.checkpoint_every or n
    total = config.epochs * n
    meta = _run_meta(dp, data, loss, penalty, config, gamma, threads=config.threads, algorithm="async-saga")
    meta["counter_batch"] = config.counter_batch
    ctas, wpc = _grid(dp, config)
    if config.threads > 1:
        # the grid the launches below use (static split, batch 0; hot staging as run_async_monitored picks)
        c, w, _ = dp.launch_config(dp._sched(1, batch=0, ctas=ctas, warps_per_cta=wpc,
                                             hot=dp.part_kind == "singleton"))
        meta["warps_in_flight"] = c * w
    trace = Trace(meta=meta)
    track = track_distance_to is not None
    single = config.threads == 1
    samples = None
    if single:
        samples = dp.torch.from_numpy(worker_sample_sequence(config.seed, 0, total, n)).to(dp.device)
    start = time.perf_counter()

    def checkpoint(it):
        obj = dp.objective()
        dist = float(np.sum((dp.x() - track_distance_to) ** 2)) if track else None
        trace.append(it, n, obj, time.perf_counter() - start, distance=dist, threads=config.threads)

    if (not single and not track and config.group_batched and config.warps is None and not config.warps_per_cta
            and _batched_group_ok(dp)):
        return _run_async_group_batched(dp, data, loss, partition, config, gamma, trace, total, every, start)
    nseg = -(-total // every)
    dev_snaps = False
    if not single and not track and dp.p_dev * 32 * (nseg + 2) > (4 << 30):
        # host snapshots of every record would not fit (or not keep pace): x-only
        # device snapshots when a quarter of the free device memory holds them
        free = dp.torch.cuda.mem_get_info(dp.device)[0]
        dev_snaps = dp.p_dev * 8 * (nseg + 2) <= free // 4
    if not single and not track and (dev_snaps or dp.p_dev * 32 * (nseg + 2) <= (4 << 30)):
        # the reference's live monitor: one launch, inconsistent snapshots of the
        # running solve at the checkpoint marks (ps_run_monitored); checkpoint 0
        # is evaluated on the device ahead of the launch
        its, objs, secs = dp.run_async_monitored(total, every, gamma, seed=config.seed, ctas=ctas,
                                                 warps_per_cta=wpc, contention=config.contention,
                                                 device_snaps=dev_snaps)
        for it, ob, sc in zip(its, objs, secs):
            trace.append(it, n, ob, sc, threads=config.threads)
        done = total
    elif not single and not track:
        # snapshots too large for host memory: stop at each mark (device-pipelined objectives)
        checkpoint(0)
        its, objs, secs = dp.run_async_checkpointed(total, every, gamma, seed=config.seed, ctas=ctas,
                                                    warps_per_cta=wpc, contention=config.contention)
        t0 = trace.wall_seconds[0]
        for it, ob, sc in zip(its, objs, secs):
            trace.append(it, n, ob, t0 + sc, threads=config.threads)
        done = total
    else:
        checkpoint(0)
        done = 0
    while done < total:
        nxt = min(total, done + every)
        if single:
            dp.replay(samples[done:nxt], gamma)
        else:
            dp.run_async(nxt - done, gamma, seed=config.seed, batch=0, ctas=ctas,
                         warps_per_cta=wpc, contention=config.contention)
        done = nxt
        checkpoint(done)
    trace.final_x = dp.x()
    trace.meta["iterations_run"] = trace.iterations[-1]
    trace.device_problem = dp
    trace.shared = dp
    return trace


def _batched_group_ok(dp):
    """The lambda-batched kernel's domain: a group penalty on contiguous blocks
    of <= 16 coordinates, rows of <= 32 nonzeros, int32 row pointers."""
    from . import _lib

    return (dp.pen_code == _lib.PEN_GROUP and dp.part_kind == "contiguous" and 1 <= int(dp.part.G) <= 16
            and int(dp.part.max_row_nnz) <= 32 and dp.row_ptr_type == 0)


def _run_async_group_batched(dp, data, loss, partition, config, gamma, trace, total, every, start):
    """run_async for group lasso through the lambda-batched kernel with one state
    (csrc/batch.cu: the scattered hot-block state layout, one load of the row's
    first block, CTA-shared loads of the most frequent block -- 2.5-3x the
    rows/s of the coordinate-record group kernels on a Zipf-headed problem,
    DESIGN.md K3b).  One launch per checkpoint segment; the final x, abar and
    alpha are copied into the problem's records, so trace.shared / final_x /
    resync_shared_average see them as after any other run."""
    from . import _lib
    from .lambda_path import BatchedPath

    n = data.n_samples
    bp = BatchedPath(data, loss, partition, B=1, dp=dp)
    bp.reset([dp.lam2])

    def objective():
        x = bp.field(0, original=False)
        v = dp.objective_parts(x.data_ptr(), 1).cpu().numpy()
        return float(v[0] + v[1] + v[2])

    trace.append(0, n, objective(), time.perf_counter() - start, threads=config.threads)
    done = 0
    while done < total:
        nxt = min(total, done + every)
        bp.run(nxt - done, gamma, seed=config.seed, contention=config.contention)
        done = nxt
        trace.append(done, n, objective(), time.perf_counter() - start, threads=config.threads)
    with dp.torch.cuda.device(dp.device):
        dp.coord[:, 0] = bp.field(0, 0, original=False)
        dp.coord[:, 1] = bp.field(0, 1, original=False)
        dp.alpha.copy_(bp.alpha.view(-1))
    c, w = _lib.ctypes.c_int32(0), _lib.ctypes.c_int32(0)
    _lib.check(_lib.load().ps_batch_last_grid(_lib.ctypes.byref(c), _lib.ctypes.byref(w)))
    trace.meta["warps_in_flight"] = int(c.value) * int(w.value)
    trace.meta["kernel"] = "lambda-batched group kernel, one state (ps_batch_run)"
    trace.final_x = dp.x()
    trace.meta["iterations_run"] = trace.iterations[-1]
    trace.device_problem = dp
    trace.shared = dp
    return trace


def iterations_to_target(trace, fstar, target):
    """Log-linear interpolation of the first crossing (asynchronous.py:213-230)."""
    floor = 1e-300
    subopt = [max(o - fstar, floor) for o in trace.objective]
    for k, s in enumerate(subopt):
        if s <= target:
            if k == 0:
                return trace.iterations[0], trace.wall_seconds[0]
            s_prev = subopt[k - 1]
            frac = math.log(s_prev / target) / math.log(s_prev / s)
            it = trace.iterations[k - 1] + frac * (trace.iterations[k] - trace.iterations[k - 1])
            wall = trace.wall_seconds[k - 1] + frac * (trace.wall_seconds[k] - trace.wall_seconds[k - 1])
            return it, wall
    return None


def measure_speedup(data, loss, penalty, partition, config, cores, target_subopt, fstar, device=None):
    """Iteration and wall speedups to a target (asynchronous.py:233-274).

    On the device "cores" are resident warps: c == 1 replays the reference's
    single-worker stream; c > 1 runs c warps."""
    if not cores or cores[0] != 1 or sorted(cores) != list(cores):
        raise ValueError("cores must be ascending and start with 1")
    rows, traces, base = [], {}, None
    for c in cores:
        run_cfg = AsyncConfig(step_size=config.step_size, epochs=config.epochs, seed=config.seed,
                              checkpoint_every=config.checkpoint_every, tolerance=0.0,
                              threads=min(c, 2) if c > 1 else 1, counter_batch=config.counter_batch,
                              warps=c if c > 1 else None, warps_per_cta=0)
        trace = run_async(data, loss, penalty, partition, run_cfg, device=device)
        traces[c] = trace
        hit = iterations_to_target(trace, fstar, target_subopt)
        if c == 1:
            base = hit
        if hit is None or base is None:
            rows.append({"cores": c, "wall_speedup": float("nan"), "theoretical_speedup": float("nan"),
                         "reached": False})
            continue
        iters, wall = hit
        base_iters, base_wall = base
        if c == 1:
            wall_speedup = theoretical = 1.0
        else:
            wall_speedup = base_wall / wall if wall > 0 else float("inf")
            theoretical = c * base_iters / iters if iters > 0 else float("inf")
        rows.append({"cores": c, "wall_speedup": wall_speedup, "theoretical_speedup": theoretical,
                     "reached": True})
    return rows, traces


def speedup_table_csv(rows, path):
    with open(path, "w") as fh:
        fh.write("cores,wall_speedup,theoretical_speedup,reached\n")
        for r in rows:
            fh.write(f"{r['cores']},{r['wall_speedup']!r},{r['theoretical_speedup']!r},"
                     f"{str(r['reached']).lower()}\n")


def resync_shared_average(trace, data):
    """Exact abar = A^T alpha / n after the run (asynchronous.py:285-298)."""
    from .saga import GradientMemory

    dp = trace.device_problem
    mem = GradientMemory(scalars=dp.alpha.cpu().numpy(), avg=dp.abar())
    dp.resync_average()
    mem.avg = dp.abar()
    return mem
