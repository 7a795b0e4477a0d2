"""Regularisation path: independent Sparse Proximal SAGA solves over a grid of
penalty weights, sharded across GPUs (BASELINE config 5).

The reference has no path driver (``gen_regularization``, problems.py:100-128,
solves serially inside a bisection).  The path here:

* lambdas: ``n_lambdas`` values log-spaced from lambda_max down to
  ``ratio * lambda_max`` (group lambda_max = max_B ||grad_B f(0)||_2 for the
  group penalty, problems.py:94-97's l1 formula otherwise);
* sharding: one process per GPU (torchrun); lambdas are dealt to ranks
  longest-expected-work-first (small lambda -> denser x -> slower), round
  robin over the sorted list; the matrix is replicated on every rank;
* no collective on the solve path; one ``all_gather_object`` of the per-lambda
  summaries at the end (gloo or NCCL; NVLink carries it on a B200 node);
* each solve reuses the rank's DeviceProblem: the state is reset and only the
  penalty weight changes, so the CSR and the column statistics are uploaded
  and computed once per rank.
"""

from __future__ import annotations

import math
import time

import numpy as np


def lambda_grid(lam_max, n_lambdas=16, ratio=1e-3):
    """Log-spaced from lam_max down to ratio * lam_max (inclusive)."""
    if n_lambdas < 1:
        raise ValueError("n_lambdas must be >= 1")
    if n_lambdas == 1:
        return [float(lam_max)]
    return [float(lam_max * ratio ** (k / (n_lambdas - 1))) for k in range(n_lambdas)]


def assign(lambdas, world):
    """Rank -> list of lambda indices; longest expected work (smallest lambda) first."""
    order = sorted(range(len(lambdas)), key=lambda k: lambdas[k])
    shards = [[] for _ in range(world)]
    for pos, k in enumerate(order):
        shards[pos % world].append(k)
    return shards


def _dist():
    try:
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            return dist
    except ImportError:
        pass
    return None


def run_path(lambdas, solve, rank=None, world=None):
    """Solve every lambda assigned to this rank with ``solve(lam) -> dict`` and
    gather all summaries (every rank returns the full, lambda-ordered list)."""
    dist = _dist()
    if rank is None:
        rank = dist.get_rank() if dist else 0
    if world is None:
        world = dist.get_world_size() if dist else 1
    mine = assign(lambdas, world)[rank]
    local = []
    if getattr(solve, "batch", None) is not None:  # concurrent solves on this rank
        t0 = time.perf_counter()
        outs = solve.batch([lambdas[k] for k in mine])
        dt = time.perf_counter() - t0
        for k, res in zip(mine, outs):
            res = dict(res)
            res.update(index=k, lam=lambdas[k], rank=rank, seconds=dt)
            local.append(res)
    else:
        for k in mine:
            t0 = time.perf_counter()
            res = dict(solve(lambdas[k]))
            res.update(index=k, lam=lambdas[k], rank=rank, seconds=time.perf_counter() - t0)
            local.append(res)
    if dist and world > 1:
        gathered = [None] * world
        dist.all_gather_object(gathered, local)
        allres = [r for part in gathered for r in part]
    else:
        allres = local
    return sorted(allres, key=lambda r: r["index"])


def _summary(dp, updates):
    """Per-lambda result, reduced on the device: objective, Fenchel dual and
    duality gap (a certificate: F(x) - F* <= gap), nnz and norm of x."""
    parts = dp.objective_parts().cpu().numpy()
    obj = float(parts.sum())
    dual = float(dp.dual_objective_dev()[0].item())
    xt = dp.field(0)
    return {"objective": obj, "dual": dual, "gap": obj - dual, "nnz": int((xt != 0).sum().item()),
            "norm": float(dp.torch.linalg.vector_norm(xt).item()), "updates": updates}


def device_solver(data, loss, partition, penalty_kind="group", step="1/2L", epochs=30, seed=0,
                  mode="async", contention=4.0, device=None, keep_x=False, ctas=0, warps_per_cta=0, concurrent=1,
                  flags=0, hot=None, batched=0, nrep=None, nrb=None):
    """A ``solve(lam)`` closure over one DeviceProblem (uploaded once).

    ``concurrent`` > 1 (async mode): ``solve.batch(lams)`` runs that many
    lambdas at a time, each on its own stream with its own state
    (``DeviceProblem.fork``) and 1/concurrent of the SMs.  For config 5 this
    pays twice: the hottest blocks' updates are spread over ``concurrent``
    copies of the state instead of queueing on one set of L2 lines, and each
    solve has fewer updates in flight (smaller tau, larger steps)."""
    from .device import DeviceProblem
    from .penalties import GroupL2Penalty, L1Penalty
    from .saga import resolve_step_size, worker_rng

    pen0 = GroupL2Penalty(0.0) if penalty_kind == "group" else L1Penalty(0.0)
    dp = DeviceProblem(data, loss, pen0, partition, device=device, drop_dead_blocks=True)
    n = data.n_samples
    gamma = resolve_step_size(step, dp.L, n, loss.lambda1 if loss.lambda1 > 0 else None)
    samples = None
    if mode == "deterministic":
        samples = dp.torch.from_numpy(worker_rng(seed, 0).integers(0, n, size=epochs * n)).to(dp.device)

    def solve(lam):
        dp.lam2 = float(lam)
        dp.reset_state()
        if samples is not None:
            dp.replay(samples, gamma)
        else:
            dp.run_async(epochs * n, gamma, seed=seed, contention=contention, ctas=ctas,
                         warps_per_cta=warps_per_cta, flags=flags, hot=hot)
        out = _summary(dp, epochs * n)
        if keep_x:
            out["x"] = dp.field(0).cpu().numpy()
        return out

    solve.problem = dp
    solve.gamma = gamma
    solve.batch = None
    if batched > 0 and penalty_kind == "group" and samples is None:
        # lambda-batched kernel: `batched` states per launch share each sampled row
        bp = BatchedPath(data, loss, partition, B=batched, device=device, nrep=nrep, nrb=nrb)
        bgamma = resolve_step_size(step, bp.dp.L, n, loss.lambda1 if loss.lambda1 > 0 else None)

        def batch(lams):
            out = []
            for w0 in range(0, len(lams), batched):
                wave = list(lams[w0:w0 + batched])
                bp.reset(wave)
                bp.run(epochs * n, bgamma, seed=seed, contention=contention, ctas=ctas, warps_per_cta=warps_per_cta)
                out.extend(bp.summaries(range(len(wave)), epochs * n, keep_x=keep_x))
            return out

        solve.batch = batch
        solve.batched = bp
        return solve
    if concurrent > 1 and samples is None:
        # concurrent group solves: the lane-per-block kernel (fewer instructions
        # per update; with 1/concurrent of the SMs per state its hot blocks no
        # longer queue) unless the caller picked a kernel
        from . import _lib

        if flags == 0 and penalty_kind == "group":
            flags = _lib.FLAG_GROUP_LANE
        torch = dp.torch
        forks = [dp] + [dp.fork() for _ in range(concurrent - 1)]
        streams = [torch.cuda.Stream(dp.device) for _ in range(concurrent)]
        sms = torch.cuda.get_device_properties(dp.device).multi_processor_count
        # 1/concurrent of the SMs each, but never more CTAs than the library's
        # own grid for one solve (small problems cap the warps in flight at n/16)
        own = dp.launch_config(dp._sched(n, ctas=0, warps_per_cta=warps_per_cta, flags=flags,
                                         hot=bool(hot) if hot is not None else False))[0]
        ctas_each = ctas if ctas > 0 else max(1, min(sms // concurrent, own))

        def grid_of(k, m):
            # the SMs left over by sms // m go to the first solves of the wave
            # (assign() orders a rank's lambdas smallest first: the densest,
            # slowest solves)
            if ctas > 0 or sms // m >= own:
                return ctas_each if m == concurrent else (ctas if ctas > 0 else max(1, min(sms // m, own)))
            return sms // m + (1 if k < sms % m else 0)

        def batch(lams):
            out = []
            for w0 in range(0, len(lams), concurrent):
                wave = lams[w0:w0 + concurrent]
                torch.cuda.synchronize(dp.device)
                for k, (f, st, lam) in enumerate(zip(forks, streams, wave)):
                    f.lam2 = float(lam)
                    f.reset_state(stream=st)
                    f.run_async(epochs * n, gamma, seed=seed, contention=contention, ctas=grid_of(k, len(wave)),
                                warps_per_cta=warps_per_cta, flags=flags, hot=hot, stream=st)
                torch.cuda.synchronize(dp.device)
                for f, lam in zip(forks, wave):
                    r = _summary(f, epochs * n)
                    if keep_x:
                        r["x"] = f.field(0).cpu().numpy()
                    out.append(r)
            return out

        solve.batch = batch
        solve.forks = forks
        solve.streams = streams
    return solve


class BatchedPath:
    """B lambda-solves of one group-lasso problem advanced together by the
    lambda-batched kernel (ps_batch_run): one warp per sampled row applies the
    step to all B states, so the sample, the CSR row and the per-row scalar
    work are shared.  State layout [block][q][beta](x, abar) on the device,
    alpha [n][beta]; the problem (CSR, partition, d_B) is the DeviceProblem's,
    uploaded once.

    ``spread`` (default): the DeviceProblem's hot-unit layout renumbers whole
    blocks so that the most frequent ones sit 32 blocks apart (ps_hot_layout,
    as for the staged kernels; nothing is staged here).  Every row commits to
    the Zipf head's blocks; in the natural order those are adjacent and their
    REDs queue in one L2 slice's atomic unit (ncu: 83% busy while the slice
    average is 12%, profiles/ncu_sps_r02.md).  ``field`` returns original
    coordinate order unless asked for the stored one.

    ``nrep`` > 0 (opt-in since the scattered hot-block layout): the x deltas of the ``nrb`` hottest
    blocks go to nrep replica accumulators (one per warp residue), folded into
    the state after each launch (ps_batch_run_rep).  With few states per row a
    hot block's x lines receive a RED from every row, and the per-line atomic
    rate caps the solve (~48 M rows/s at B = 2 whatever the grid)."""

    # replicas of the x-delta accumulators: none by default since the scattered
    # hot blocks of the state layout (csrc/batch.cu bidx: one coordinate sector per
    # KB for the most frequent blocks) -- config 5 rows/s of one epoch with
    # replicas / scattered: B = 2 79 / 115 M, B = 4 43 / 85 M, B = 8 25 / 63 M,
    # B = 16 (no replicas) 25 / 40 M (tools/gpu/exp_batch_scatter.py); replicas on
    # top of the scattered layout cost 20-60%.  nrep / nrb keep the option.
    AUTO_NREP = {1: 0, 2: 0, 4: 0, 8: 0, 16: 0}
    AUTO_NRB = {1: 0, 2: 0, 4: 0, 8: 0, 16: 0}

    def __init__(self, data, loss, partition, B=16, device=None, dp=None, spread=True, nrep=None, nrb=None):
        from . import _lib
        from .device import DeviceProblem
        from .penalties import GroupL2Penalty

        if B not in (1, 2, 4, 8, 16):
            raise ValueError("B must be 1, 2, 4, 8 or 16")
        self.dp = dp if dp is not None else DeviceProblem(data, loss, GroupL2Penalty(0.0), partition, device=device,
                                                          drop_dead_blocks=True, hot_max=None if spread else 0)
        if self.dp.part_kind != "contiguous" or not 1 <= int(self.dp.part.G) <= 16:
            raise ValueError("the batched path needs a contiguous partition with blocks of <= 16 coordinates")
        if int(self.dp.part.max_row_nnz) > 32 or self.dp.row_ptr_type != 0:
            raise ValueError("the batched path needs rows of <= 32 nonzeros and int32 row pointers")
        torch = self.torch = self.dp.torch
        self.B = B
        dev = self.dp.device
        with torch.cuda.device(dev):
            G = int(self.dp.part.G)
            self.state = torch.zeros(int(_lib.load().ps_batch_state_doubles(self.dp.p_dev, G, B)), dtype=torch.float64,
                                     device=dev)
            self.alpha = torch.zeros(self.dp.n * B, dtype=torch.float64, device=dev)
            self.lam2 = torch.zeros(B, dtype=torch.float64, device=dev)
            self.counter = torch.zeros(1, dtype=torch.int64, device=dev)
            self.vec = torch.empty(self.dp.p_dev, dtype=torch.float64, device=dev)
            self._perm_long = self.dp.perm.long() if self.dp.perm is not None else None
            # replicated x-delta accumulators of the nrb hottest blocks (ps_batch_run_rep;
            # needs the spread layout, whose hot units are the blocks r << hot_shift)
            units = self.dp.H // G if self.dp.perm is not None else 0
            nrep = self.AUTO_NREP[B] if nrep is None else nrep
            nrb = self.AUTO_NRB[B] if nrb is None else nrb
            self.nrb = min(int(nrb), units) if nrep > 0 else 0
            self.nrep = int(nrep) if self.nrb > 0 else 0
            self.xrep = (torch.zeros(int(_lib.load().ps_batch_rep_doubles(self.nrep, self.nrb, G, B)),
                                     dtype=torch.float64, device=dev) if self.nrep else None)
        self.slot_base = 0

    def reset(self, lams):
        """x0 = 0, abar = 0, alpha = 0 for every state; lam2[beta] = lams[beta]
        (fewer lambdas than B: the spare states repeat the last one)."""
        lams = list(lams)
        if not 1 <= len(lams) <= self.B:
            raise ValueError("between 1 and B lambdas")
        self.lams = lams
        vals = lams + [lams[-1]] * (self.B - len(lams))
        with self.torch.cuda.device(self.dp.device):
            self.state.zero_()
            self.alpha.zero_()
            self.lam2.copy_(self.torch.tensor(vals, dtype=self.torch.float64))
        self.slot_base = 0

    def run(self, rows, gamma, seed=0, contention=4.0, ctas=0, warps_per_cta=0, samples=None, stream=None):
        """`rows` sampled rows, each applied to every state (asynchronous), or
        the deterministic replay of `samples` (one warp)."""
        from . import _lib

        dp = self.dp
        with self.torch.cuda.device(dp.device):
            ptr = None
            if samples is not None:
                s = self.torch.from_numpy(np.ascontiguousarray(samples, dtype=np.int64)).to(dp.device)
                ptr, rows, self._keep = s.data_ptr(), int(s.numel()), s
            else:
                self.counter.zero_()
            sched = _lib.Sched(ptr, int(rows), int(seed) & (2 ** 64 - 1), int(self.slot_base), self.counter.data_ptr(),
                               0, int(ctas), int(warps_per_cta), 0, float(contention), 0, 0, int(dp.hot_shift), 0, None,
                               None)
            _lib.check(_lib.load().ps_batch_run_rep(dp.csr, dp.part, dp.params(gamma), self.lam2.data_ptr(), self.B,
                                                    self.state.data_ptr(), self.alpha.data_ptr(), sched,
                                                    self.xrep.data_ptr() if self.nrep else None, self.nrep, self.nrb,
                                                    _lib.stream_ptr(stream)))
            if samples is None:
                self.slot_base += int(rows)

    def field(self, beta, f=0, original=True):
        """x (f=0) or abar (f=1) of state beta as a device vector: the p
        coordinates in original order, or (original=False) the padded stored
        order the device CSR uses."""
        from . import _lib

        with self.torch.cuda.device(self.dp.device):
            out = self.torch.empty(self.dp.p_dev, dtype=self.torch.float64, device=self.dp.device)
            _lib.check(_lib.load().ps_batch_field(self.state.data_ptr(), self.dp.p_dev, int(self.dp.part.G), self.B,
                                                  int(self.dp.hot_shift), int(beta), int(f), out.data_ptr(), 0, _lib.stream_ptr()))
            if original and self._perm_long is not None:
                out = out[self._perm_long]
        return out

    def summaries(self, betas, updates, keep_x=False):
        """Objective, Fenchel dual and gap (a certificate), nnz and norm of the
        given states: every evaluation is enqueued first, the results come back
        in ONE device-to-host copy (a state's summary otherwise costs four host
        round trips; 16 states: ~2.5 ms of a 64 ms path)."""
        dp, torch = self.dp, self.torch
        saved = dp.lam2
        recs, xs = [], []
        with torch.cuda.device(dp.device):
            for beta in betas:
                x = self.field(beta, original=False)
                dp.lam2 = float(self.lams[beta])
                parts = dp.objective_parts(x.data_ptr(), 1)  # views of reused scratch: copied by the cat below
                dual = dp.dual_objective_dev(x.data_ptr(), 1)
                recs.append(torch.cat([parts, dual[:1], (x != 0).sum().to(torch.float64).reshape(1),
                                       torch.linalg.vector_norm(x).reshape(1)]))
                if keep_x:
                    xs.append(x[self._perm_long] if self._perm_long is not None else x)
            host = torch.stack(recs).cpu().numpy() if recs else np.zeros((0, 6))
        dp.lam2 = saved
        out = []
        for r, h in enumerate(host):
            obj = float(h[0] + h[1] + h[2])
            rec = {"objective": obj, "dual": float(h[3]), "gap": obj - float(h[3]), "nnz": int(h[4]),
                   "norm": float(h[5]), "updates": updates}
            if keep_x:
                rec["x"] = xs[r].cpu().numpy()
            out.append(rec)
        return out

    def summary(self, beta, updates, keep_x=False):
        """One state's summary (see summaries)."""
        return self.summaries([beta], updates, keep_x=keep_x)[0]


def lambda_max_for(data, partition, penalty_kind="group", device=None):
    from .problems import group_lambda_max, lambda_max

    if penalty_kind == "group":
        return group_lambda_max(data, partition, device=device)
    return lambda_max(data, device=device)


def regularization_path(data, loss, partition, n_lambdas=16, ratio=1e-3, penalty_kind="group", epochs=30,
                        step="1/2L", seed=0, mode="async", device=None, keep_x=False, concurrent=1, batched=None):
    """Config 5 end to end on this rank's GPU (call under torchrun for N GPUs).
    ``batched`` = B > 0: the rank's lambdas B at a time through the
    lambda-batched kernel; 0: ``concurrent`` lambdas at a time as forks (1 = one
    after the other); None (default): the batched kernel with B = the rank's
    share rounded up to a power of two (<= 16) where it applies (asynchronous
    group lasso on contiguous blocks of <= 16, rows of <= 32 nonzeros), else
    the forks."""
    lam_max = lambda_max_for(data, partition, penalty_kind, device=device)
    lams = lambda_grid(lam_max, n_lambdas, ratio)
    solve = None
    if batched is None:
        batched = 0
        if penalty_kind == "group" and mode == "async" and concurrent == 1:
            dist = _dist()
            share = max(len(a) for a in assign(lams, dist.get_world_size() if dist else 1))
            B = 1
            while B < min(16, share):
                B *= 2
            try:
                solve = device_solver(data, loss, partition, penalty_kind, step, epochs, seed, mode, device=device,
                                      keep_x=keep_x, batched=B)
                batched = B
            except ValueError:
                solve = None
    if solve is None:
        solve = device_solver(data, loss, partition, penalty_kind, step, epochs, seed, mode, device=device,
                              keep_x=keep_x, concurrent=concurrent, batched=batched)
    t0 = time.perf_counter()
    res = run_path(lams, solve)
    return {"lambda_max": lam_max, "lambdas": lams, "results": res, "seconds": time.perf_counter() - t0,
            "total_updates": sum(r["updates"] for r in res)}


def path_throughput(results, seconds):
    tot = sum(r["updates"] for r in results)
    return tot / seconds if seconds > 0 else math.inf
