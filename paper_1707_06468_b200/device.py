"""Device-resident problem + solver state: the host runtime around libproxsaga.

``DeviceProblem`` uploads a dataset once (CSR with int32 columns, fp32 values
when that is lossless, int32/int64 row pointers), runs ps_prepare (block
counts, d_B, delta, max row norm — the reference's build_support_index and
lipschitz_constant, data.py:236-297 / losses.py:99-105) and owns the
coordinate state

    coord[p, 4] fp64 = (x_j, abar_j, D_j, reserved)   -- one 32 B sector per j
    alpha[n]   fp64                                  -- the SAGA scalar memory

(saga.py:54-72 GradientMemory / asynchronous.py:44-72 SharedState).  Every
computation goes through the C ABI; torch only provides device memory and
streams.
"""

from __future__ import annotations

import ctypes
import functools

import numpy as np

from . import _lib
from .data import partition_structure
from .penalties import penalty_code


def _torch():
    import torch

    return torch


def _f32_exact(a):
    a = np.asarray(a)
    if a.dtype == np.float32:
        return True
    with np.errstate(over="ignore", invalid="ignore"):
        return bool(np.array_equal(a.astype(np.float32).astype(np.float64), a))


_PINNED = {}


def _pinned_snapshots(torch, nmax, p):
    """Pinned host snapshot buffers of the live monitor, kept across calls
    (cudaHostAlloc of a few MB costs ~0.3 ms, a fifth of a config-2 solve):
    one buffer per device, grown on demand; returns an (nmax, p, 4) view."""
    need = nmax * p * 4
    key = torch.cuda.current_device()
    buf = _PINNED.get(key)
    if buf is None or buf.numel() < need:
        buf = torch.empty(need, dtype=torch.float64, pin_memory=True)
        _PINNED[key] = buf
    return buf[:need].view(nmax, p, 4)


class DeviceProblem:
    """One problem on one GPU.

    Parameters mirror the reference's solver arguments (saga.py:217-218):
    ``data`` (Dataset-like: ``features`` CSR with ``row_offsets``,
    ``col_indices``, ``values``; ``labels``), ``loss`` (``kind``,
    ``lambda1``), ``penalty`` and ``partition`` (BlockPartition-like, ``None``
    = singleton).  Reference objects are accepted duck-typed.
    """

    def __init__(self, data, loss, penalty, partition=None, device=None, drop_dead_blocks=False,
                 value_dtype="auto", hot_max=None, hot_min_frac=1.0 / 512, hot_stride=32, hot_min_rows=4096,
                 index_dtype="auto", _labels=None, _device_csr=None, _shape=None):
        torch = _torch()
        _lib.require_device()
        self.torch = torch
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else
                                   (device.index if isinstance(device, torch.device) else int(device)))
        if _device_csr is not None:
            f, labels = None, None
            self.n, self.p, self.nnz = (int(v) for v in _shape)
        else:
            f = data.features if hasattr(data, "features") else data
            labels = data.labels if _labels is None else _labels
            self.n, self.p = int(f.n_rows), int(f.n_cols)
            self.nnz = int(f.row_offsets[-1])
        if self.n < 1:
            raise ValueError("dataset is empty")
        if self.p >= 2 ** 31:
            raise ValueError("n_cols must fit int32")
        self.loss_kind = loss.kind if loss is not None else "squared"
        self.lambda1 = float(loss.lambda1) if loss is not None else 0.0
        if penalty is None:
            self.pen_code, self.lam2, self.lo, self.hi = _lib.PEN_ZERO, 0.0, -1.0, 1.0
        else:
            self.pen_code, self.lam2, self.lo, self.hi = penalty_code(penalty)
        dev = self.device
        with torch.cuda.device(dev):
            if _device_csr is not None:  # already on the device (K7 generator)
                self.row_ptr, self.col, self.val, self.y = _device_csr
                self.row_ptr_type = _lib.I32 if self.row_ptr.dtype == torch.int32 else _lib.I64
                self.value_type = _lib.F32 if self.val.dtype == torch.float32 else _lib.F64
            else:
                # ---- CSR upload: host arrays go up in their own dtype (a DMA
                # straight from the caller's buffer, async when it is pinned) and
                # are narrowed on the device (int64 -> int32 indices, exact
                # fp64 -> fp32 values), not by a host conversion pass
                def up(a):
                    return torch.from_numpy(np.ascontiguousarray(a)).to(dev, non_blocking=True)

                # int32 row pointers when they fit; index_dtype="int64" keeps the
                # reference's own int64 (data.py:46-48) -- the PS_I64 kernels
                if index_dtype not in ("auto", "int64"):
                    raise ValueError("index_dtype must be 'auto' or 'int64'")
                self.row_ptr_type = _lib.I32 if (self.nnz < 2 ** 31 - 1 and index_dtype == "auto") else _lib.I64
                ro_d = up(f.row_offsets)
                self.row_ptr = ro_d.to(torch.int32 if self.row_ptr_type == _lib.I32 else torch.int64)
                self.col = up(f.col_indices).to(torch.int32)
                val_d, y_d = up(f.values), up(np.asarray(labels))
                if value_dtype == "auto":
                    # fp32 storage when lossless: small arrays are checked on the host
                    # (no device round trip), large fp64 ones on the device
                    def exact32(host, t):
                        if t.dtype == torch.float32:
                            return True
                        if t.numel() <= (1 << 20):
                            return _f32_exact(host)
                        return bool(torch.equal(t.to(torch.float32).to(t.dtype), t))

                    use32 = exact32(f.values, val_d) and exact32(labels, y_d)
                else:
                    use32 = np.dtype(value_dtype) == np.float32
                self.value_type = _lib.F32 if use32 else _lib.F64
                tdt = torch.float32 if use32 else torch.float64
                self.val = val_d.to(tdt)
                self.y = y_d.to(tdt)
            self.csr = _lib.Csr(self.n, self.p, self.nnz, self.row_ptr.data_ptr(), self.col.data_ptr(),
                                self.val.data_ptr(), self.y.data_ptr(), self.row_ptr_type, self.value_type)
            # ---- partition (+ hot-column renumbering for singleton layouts)
            self._setup_partition(partition)
            self.H, self.hot_shift, self.perm, self._perm_np, self.p_dev = 0, 0, None, None, self.p
            self.hot_unit = 1 if self.part_kind == "singleton" else int(self.part.G)
            if hot_max is None:
                # staged columns: 512, or 1024 when the coordinate records (32 B each)
                # do not fit in L2 -- then every staged column saves HBM round trips,
                # not just L2 ones (config 3: 1.31 -> 1.69 G updates/s; config 2 and
                # 4, whose records are L2-resident, gain nothing from 1024)
                hot_max = 1024 if 32 * self.p > 96 * (1 << 20) else 512
            if self.part_kind in ("singleton", "contiguous") and hot_max > 0 and self.n >= hot_min_rows:
                # hot_max columns (singleton), or whole blocks up to 1024 staged coordinates
                units = hot_max if self.hot_unit == 1 else max(1, min(4 * hot_max, 1024) // self.hot_unit)
                self._hot_layout(int(units), float(hot_min_frac), int(hot_stride))
            # ---- state
            # one zeroed allocation (one fill) for coord[p, 4], alpha[n] and the
            # counter.  The coordinate records start 64 KiB past a 2 MiB boundary:
            # the staged (hot) records sit 1 KiB apart from the base, and their
            # L2 slices -- hence the fast kernel's time, 1.72 to 2.02 ms on
            # config 2 -- depend on the base offset (tools/exp_align.py)
            pad = (1 << 21) // 8
            state = torch.zeros(4 * self.p_dev + self.n + 1 + 2 * pad, dtype=torch.float64, device=dev)
            o = ((-state.data_ptr()) % (1 << 21)) // 8 + (1 << 16) // 8
            self._state = state
            self.coord = state[o:o + 4 * self.p_dev].view(self.p_dev, 4)
            self.alpha = state[o + 4 * self.p_dev:o + 4 * self.p_dev + self.n]
            self.counter = state[o + 4 * self.p_dev + self.n:o + 4 * self.p_dev + self.n + 1].view(torch.int64)
            self.stats = _lib.Stats()
            _lib.check(_lib.load().ps_prepare(self.csr, self.part, self.coord.data_ptr(), self.stats,
                                              _lib.stream_ptr()))
        self.delta = float(self.stats.max_count) / self.n if self.stats.max_count > 0 else 0.0
        self.n_dead = int(self.stats.n_dead)
        if self.n_dead and not drop_dead_blocks:
            from .data import DeadBlockError

            raise DeadBlockError(np.flatnonzero(self.block_stats()[0] == 0))
        self.L = (0.25 if self.loss_kind == "logistic" else 1.0) * float(self.stats.max_row_sqnorm) + self.lambda1
        self.slot_base = 0
        self._scratch = None
        self._out = torch.zeros(4, dtype=torch.float64, device=dev)
        self._grad = None

    @classmethod
    def from_device_csr(cls, row_ptr, col, val, y, p, loss, penalty, partition=None, device=None, **kw):
        """A problem whose CSR already lives on the device (torch tensors:
        row_ptr int32/int64[n+1], col int32[nnz], val / y fp32 or fp64)."""
        n = int(row_ptr.numel()) - 1
        return cls(None, loss, penalty, partition, device=device, drop_dead_blocks=True,
                   _device_csr=(row_ptr, col, val, y), _shape=(n, p, int(col.numel())), **kw)

    @classmethod
    def for_index(cls, features, partition, device=None):
        """Statistics-only instance (no labels needed): build_support_index / L."""
        class _D:
            pass

        d = _D()
        d.features = features
        return cls(d, None, None, partition, device=device, drop_dead_blocks=True,
                   _labels=np.zeros(features.n_rows))

    # ------------------------------------------------------------------
    def _setup_partition(self, partition):
        torch, dev = self.torch, self.device
        kind, G = ("singleton", 1) if partition is None else partition_structure(partition)
        if self.pen_code == _lib.PEN_GROUP and kind == "singleton":
            kind, G = "contiguous", 1  # per-coordinate blocks through the block path
        if kind == "contiguous" and G > 32:
            kind = "general"
        self.part_kind = kind
        p = self.p
        if kind == "singleton":
            nb = p
            self.part = _lib.Part(_lib.PART_SINGLETON, 1, nb)
        elif kind == "contiguous":
            nb = -(-p // G)
            self.part = _lib.Part(_lib.PART_CONTIG, G, nb)
        else:
            bo = np.asarray(partition.block_of, dtype=np.int64)
            nb = int(partition.n_blocks)
            order = np.argsort(bo, kind="stable")
            ptr = np.zeros(nb + 1, dtype=np.int64)
            np.cumsum(np.bincount(bo, minlength=nb), out=ptr[1:])
            self.block_of = torch.from_numpy(bo.astype(np.int32)).to(dev)
            self.blk_ptr = torch.from_numpy(ptr.astype(np.int32)).to(dev)
            self.blk_coords = torch.from_numpy(order.astype(np.int32)).to(dev)
            self.row_blk = torch.zeros(max(self.nnz, 1), dtype=torch.int32, device=dev)
            self.row_g = torch.zeros(self.n, dtype=torch.int32, device=dev)
            self.spos = torch.zeros(max(self.nnz, 1), dtype=torch.int32, device=dev)
            self.part = _lib.Part(_lib.PART_GENERAL, 0, nb, self.block_of.data_ptr(), self.blk_ptr.data_ptr(),
                                  self.blk_coords.data_ptr(), 0, 0, self.row_blk.data_ptr(),
                                  self.row_g.data_ptr(), self.spos.data_ptr(), 0)
        self.n_blocks = nb
        self.blk_count = torch.zeros(nb, dtype=torch.int32, device=dev)
        self.blk_weight = torch.zeros(nb, dtype=torch.float64, device=dev)
        self.part.blk_count = self.blk_count.data_ptr()
        self.part.blk_weight = self.blk_weight.data_ptr()

    def _hot_layout(self, hot_max, min_frac, stride):
        """ps_hot_layout: the most frequent units (columns, or whole blocks of a
        contiguous partition) are stored strided at the front and staged in
        shared memory by the async kernel; the device CSR is remapped and its
        rows re-sorted in place; coordinates are padded to whole units."""
        torch, dev = self.torch, self.device
        G = self.hot_unit
        ws = torch.empty(-(-self.p // G), dtype=torch.int32, device=dev)
        self.perm = torch.empty(self.p, dtype=torch.int32, device=dev)
        H, S, pp = ctypes.c_int32(0), ctypes.c_int32(stride), ctypes.c_int64(0)
        _lib.check(_lib.load().ps_hot_layout(self.csr, self.col.data_ptr(), self.val.data_ptr(), G, hot_max,
                                             min_frac, ctypes.byref(S), ws.data_ptr(), self.perm.data_ptr(),
                                             ctypes.byref(H), ctypes.byref(pp), _lib.stream_ptr()))
        self.H = H.value * G          # staged coordinate slots
        self.hot_shift = S.value.bit_length() - 1
        self.p_dev = int(pp.value)
        self.csr.n_cols = self.p_dev
        self._perm_np = None  # host copy made on first use (perm_np)

    @property
    def perm_np(self):
        """original -> stored coordinate index (host int64), or None without a hot layout"""
        if self.perm is not None and self._perm_np is None:
            self._perm_np = self.perm.cpu().numpy().astype(np.int64)
        return self._perm_np

    @property
    def unit_perm_np(self):
        G = self.hot_unit
        pn = self.perm_np
        return pn[::G] // G if (pn is not None and G > 1) else pn

    def _to_stored(self, v):
        """original-order vector -> stored (permuted, padded) order"""
        if self.perm_np is None:
            return np.ascontiguousarray(v, dtype=np.float64)
        out = np.zeros(self.p_dev)
        out[self.perm_np] = v
        return out

    def _to_original(self, v):
        return v if self.perm_np is None else np.asarray(v)[self.perm_np]

    def block_stats(self):
        c, w = self.blk_count.cpu().numpy(), self.blk_weight.cpu().numpy()
        if self.perm_np is not None:
            c, w = c[self.unit_perm_np], w[self.unit_perm_np]
        return c, w, self.stats

    # ------------------------------------------------------------------
    def params(self, gamma=1.0):
        return _lib.Params(_lib.LOSS[self.loss_kind], self.pen_code, self.lambda1, self.lam2, self.lo,
                           self.hi, float(gamma))

    def reset_state(self, stream=None):
        """x0 = 0, alpha = 0, abar = 0 (PAPER.md:1195-1199 / saga.py:231-232)."""
        _lib.check(_lib.load().ps_state_reset(self.coord.data_ptr(), self.p_dev, self.alpha.data_ptr(), self.n,
                                              self.counter.data_ptr(), _lib.stream_ptr(stream)))
        self.slot_base = 0

    def _sched(self, count, samples=None, seed=0, batch=0, ctas=0, warps_per_cta=0, contention=0.0,
               hot=True, hot_period=0, flags=0, trace=None):
        tv, tdx = trace if trace is not None else (None, None)
        return _lib.Sched(samples, int(count), int(seed) & (2 ** 64 - 1), int(self.slot_base),
                          self.counter.data_ptr(), int(batch), int(ctas), int(warps_per_cta),
                          int(self.H if hot else 0), float(contention), int(hot_period), int(flags),
                          int(self.hot_shift), 0, tv, tdx)

    def launch_config(self, sched):
        c, w, b = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int64()
        _lib.check(_lib.load().ps_launch_config(self.csr, self.part, sched, ctypes.byref(c), ctypes.byref(w),
                                                ctypes.byref(b)))
        return c.value, w.value, b.value

    def _scratch_for(self, sched):
        _, _, nbytes = self.launch_config(sched)
        if nbytes == 0:
            return None
        if self._scratch is None or self._scratch.numel() * 8 < nbytes:
            self._scratch = self.torch.empty((nbytes + 7) // 8, dtype=self.torch.float64, device=self.device)
        return self._scratch.data_ptr()

    def replay(self, samples, gamma, stream=None, trace=None):
        """Deterministic replay of a sample sequence (saga.py:248-256) on one warp.
        ``trace`` = (v, dx) device pointers (p doubles each): the last step's
        gradient estimate and applied delta on its extended support."""
        torch = self.torch
        if isinstance(samples, torch.Tensor) and samples.is_cuda:
            s = samples.to(torch.int64)
        else:
            s = torch.from_numpy(np.ascontiguousarray(samples, dtype=np.int64)).to(self.device)
        if s.numel() == 0:
            return
        if int(s.min()) < 0 or int(s.max()) >= self.n:
            raise IndexError("sample index out of range")
        sched = self._sched(s.numel(), samples=s.data_ptr(), trace=trace)
        scr = self._scratch_for(sched)
        _lib.check(_lib.load().ps_run(self.csr, self.part, self.params(gamma), self.coord.data_ptr(),
                                      self.alpha.data_ptr(), sched, scr, _lib.stream_ptr(stream)))
        self._keep = s

    def run_async(self, count, gamma, seed=0, batch=0, ctas=0, warps_per_cta=0, contention=4.0, hot=None,
                  hot_period=0, flags=0, stream=None):
        """`count` lock-free updates (asynchronous.py:131-210), continuing the
        sampler stream where the previous call stopped.  ``contention`` = c of
        the per-coordinate step gamma_j = gamma min(1, c D_j / tau) (0: plain
        gamma)."""
        with self.torch.cuda.stream(stream if stream is not None else self.torch.cuda.current_stream(self.device)):
            self.counter.zero_()
        if hot is None:  # shared-memory staging pays for hot columns; for hot blocks the strided layout suffices
            hot = self.part_kind == "singleton"
        sched = self._sched(count, seed=seed, batch=batch, ctas=ctas, warps_per_cta=warps_per_cta,
                            contention=contention, hot=hot, hot_period=hot_period, flags=flags)
        scr = self._scratch_for(sched)
        _lib.check(_lib.load().ps_run(self.csr, self.part, self.params(gamma), self.coord.data_ptr(),
                                      self.alpha.data_ptr(), sched, scr, _lib.stream_ptr(stream)))
        self.slot_base += int(count)

    def run_async_monitored(self, total, every, gamma, seed=0, batch=0, ctas=0, warps_per_cta=0, contention=4.0,
                            hot=None, hot_period=0, flags=0, gap=False, device_snaps=False):
        """`total` lock-free updates in ONE launch with the reference's live
        monitor (asynchronous.py:181-198, ps_run_monitored): each time the
        progress counter crosses a multiple of `every`, the live coordinate
        records are copied (an inconsistent snapshot, as snapshot_x is) while
        the warps keep going.  The objectives (and with ``gap`` the Fenchel
        duals) of the snapshots are evaluated afterwards; a checkpoint's time is
        its snapshot's device time plus one measured objective evaluation (the
        time the monitor would need to know it).  Checkpoint 0 (the starting
        state) and the last one (the consistent state after the launch) are
        evaluated in place, without a copy.  ``device_snaps``: x-only snapshots
        into device memory, copied by a few CTAs beside the solve (whose default
        grid leaves them their SMs; PS_FLAG_MON_DEVICE_X) -- for problems whose
        records would take longer than an epoch to copy to the host.  Returns
        (iterations, objectives, seconds[, duals])."""
        torch = self.torch
        if hot is None:
            hot = self.part_kind == "singleton"
        nmax = int(-(-int(total) // int(every))) + 2
        # checkpoint 0 and the final one are evaluated in place (below): no copies of them
        sched = self._sched(total, seed=seed, batch=batch, ctas=ctas, warps_per_cta=warps_per_cta,
                            contention=contention, hot=hot, hot_period=hot_period,
                            flags=flags | _lib.FLAG_MON_ENDS_IN_PLACE | (_lib.FLAG_MON_DEVICE_X if device_snaps else 0))
        scr = self._scratch_for(sched)
        if device_snaps:
            snaps = torch.empty((nmax, self.p_dev), dtype=torch.float64, device=self.device)  # x only
        else:
            snaps = _pinned_snapshots(torch, nmax, self.p_dev)  # DMA targets
        counts = (ctypes.c_int64 * nmax)()
        ms = (ctypes.c_float * nmax)()
        ns = ctypes.c_int32(0)
        L = _lib.load()
        outs = torch.zeros((nmax, 4), dtype=torch.float64, device=self.device)
        duals = torch.zeros((nmax, 2), dtype=torch.float64, device=self.device) if gap else None

        def evaluate(j, ptr):
            _lib.check(L.ps_objective(self.csr, self.part, self.params(), ptr, 4, outs[j].data_ptr(),
                                      _lib.stream_ptr()))
            if gap:
                _lib.check(L.ps_dual_objective(self.csr, self.part, self.params(), ptr, 4, duals[j].data_ptr(),
                                               _lib.stream_ptr()))

        # checkpoint 0 is the state the launch starts from: evaluated in place,
        # stream-ordered before it (no copy, no host round trip)
        evaluate(0, self.coord.data_ptr())
        _lib.check(L.ps_run_monitored(self.csr, self.part, self.params(gamma), self.coord.data_ptr(),
                                      self.alpha.data_ptr(), sched, scr, _lib.stream_ptr(), int(every), nmax,
                                      snaps.data_ptr(), counts, ms, ctypes.byref(ns)))
        self.slot_base += int(total)
        k = ns.value
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        buf = None
        for j in range(1, k):
            stride = 4
            if j == k - 1:
                ptr = self.coord.data_ptr()  # the final snapshot is the (consistent) state after the launch
            elif device_snaps:
                ptr, stride = snaps[j].data_ptr(), 1
            else:
                if buf is None:
                    buf = torch.empty((self.p_dev, 4), dtype=torch.float64, device=self.device)
                buf.copy_(snaps[j])
                ptr = buf.data_ptr()
            if j == 1:
                e0.record()
            _lib.check(L.ps_objective(self.csr, self.part, self.params(), ptr, stride, outs[j].data_ptr(),
                                      _lib.stream_ptr()))
            if j == 1:
                e1.record()
            if gap:
                _lib.check(L.ps_dual_objective(self.csr, self.part, self.params(), ptr, stride, duals[j].data_ptr(),
                                               _lib.stream_ptr()))
        o = outs[:k].cpu().numpy()  # synchronizes
        t_eval = e0.elapsed_time(e1) / 1e3 if k > 1 else 0.0
        objs = [float(v[0] + v[1] + v[2]) for v in o]  # the order objective() sums in
        its = [int(counts[j]) for j in range(k)]
        secs = [float(ms[j]) / 1e3 + (t_eval if j > 0 else 0.0) for j in range(k)]
        if gap:
            return its, objs, secs, duals[:k, 0].cpu().numpy().tolist()
        return its, objs, secs

    def run_async_checkpointed(self, total, every, gamma, seed=0, ring=4, graph=False, gap=False, **kw):
        """`total` async updates in segments of `every`; after each segment x is
        snapshotted on the device and the objective of the snapshot is evaluated
        on a side stream while the next segment runs (the reference's monitor,
        asynchronous.py:187-198, without host round trips).  Returns
        (iterations, objectives, seconds) with times from device timestamps
        (%globaltimer via ps_timestamp), measured from the first launch to the
        end of each checkpoint's objective.

        ``graph``: the whole sequence (per segment: counter reset, SPS launch,
        snapshot, objective on the side stream) is captured once into a CUDA
        graph and replayed, so a segment costs its device time and not the
        ~0.1 ms of host work per launch (a config-2 epoch is ~0.1 ms of GPU
        time).  Capture does not execute anything; the replay is the run.
        Worth it when the segments are short and many (bench time-to-target);
        the capture + instantiation costs about what eager enqueueing does.

        ``gap``: also evaluate the Fenchel dual of each snapshot on the side
        stream (ps_dual_objective) and return the duals as a fourth list
        (duality gap = objective - dual)."""
        torch = self.torch
        if getattr(self, "_side", None) is None:
            self._side = torch.cuda.Stream(self.device)
        side = self._side
        nseg = -(-int(total) // int(every))
        snaps = [torch.empty(self.p_dev, dtype=torch.float64, device=self.device) for _ in range(min(ring, nseg))]
        outs = torch.zeros((nseg, 4), dtype=torch.float64, device=self.device)
        douts = torch.zeros((nseg, 2), dtype=torch.float64, device=self.device) if gap else None
        ev_obj = [torch.cuda.Event() for _ in range(nseg)]
        ev_snap = [torch.cuda.Event() for _ in range(nseg)]
        stamps = torch.zeros(nseg + 1, dtype=torch.int64, device=self.device)  # %globaltimer, ns
        L = _lib.load()

        def stamp(k, stream):
            _lib.check(L.ps_timestamp(stamps.data_ptr() + 8 * k, _lib.stream_ptr(stream)))

        def enqueue(main):
            stamp(0, main)
            done, its = 0, []
            for k in range(nseg):
                cnt = min(int(every), int(total) - done)
                self.run_async(cnt, gamma, seed=seed, stream=main, **kw)
                done += cnt
                its.append(done)
                buf = snaps[k % len(snaps)]
                if k >= len(snaps):
                    main.wait_event(ev_obj[k - len(snaps)])  # ring slot free again
                _lib.check(L.ps_coord_get(self.coord.data_ptr(), self.p_dev, 0, buf.data_ptr(),
                                          _lib.stream_ptr(main)))
                ev_snap[k].record(main)
                side.wait_event(ev_snap[k])
                _lib.check(L.ps_objective(self.csr, self.part, self.params(), buf.data_ptr(), 1,
                                          outs[k].data_ptr(), _lib.stream_ptr(side)))
                if gap:
                    _lib.check(L.ps_dual_objective(self.csr, self.part, self.params(), buf.data_ptr(), 1,
                                                   douts[k].data_ptr(), _lib.stream_ptr(side)))
                stamp(k + 1, side)
                ev_obj[k].record(side)
            main.wait_event(ev_obj[-1])  # join the side stream
            return its

        if graph:
            base0 = self.slot_base
            g = torch.cuda.CUDAGraph()
            torch.cuda.synchronize(self.device)
            with torch.cuda.graph(g):
                its = enqueue(torch.cuda.current_stream(self.device))
            self.slot_base = base0 + int(total)
            g.replay()
        else:
            its = enqueue(torch.cuda.current_stream(self.device))
        torch.cuda.synchronize(self.device)
        objs = outs[:, :3].sum(dim=1).cpu().numpy().tolist()
        st = stamps.cpu().numpy()
        secs = [float(st[k + 1] - st[0]) / 1e9 for k in range(nseg)]
        if gap:
            return its, objs, secs, douts[:, 0].cpu().numpy().tolist()
        return its, objs, secs

    # ------------------------------------------------------------------
    def objective_parts(self, x_ptr=None, stride=4, stream=None):
        """Device tensor [mean loss, l2 term, penalty] (ps_objective)."""
        if x_ptr is None:
            x_ptr = self.coord.data_ptr()
        _lib.check(_lib.load().ps_objective(self.csr, self.part, self.params(), x_ptr, stride,
                                            self._out.data_ptr(), _lib.stream_ptr(stream)))
        return self._out[:3]

    def objective(self):
        v = self.objective_parts().cpu().numpy()
        return float(v[0] + v[1] + v[2])

    def dual_objective_dev(self, x_ptr=None, stride=4, out=None, stream=None):
        """Device tensor [D, c]: the Fenchel dual value at the dual point induced
        by x (ps_dual_objective) and the scaling c applied to it."""
        torch = self.torch
        if x_ptr is None:
            x_ptr = self.coord.data_ptr()
        if out is None:
            if getattr(self, "_dout", None) is None:
                self._dout = torch.zeros(2, dtype=torch.float64, device=self.device)
            out = self._dout
        _lib.check(_lib.load().ps_dual_objective(self.csr, self.part, self.params(), x_ptr, stride,
                                                 out.data_ptr(), _lib.stream_ptr(stream)))
        return out

    def duality_gap(self):
        """(primal, dual, gap) at the current x, all evaluated on the device;
        gap = P(x) - D(theta(x)) >= 0 and 0 exactly at the optimum."""
        prim = self.objective()
        dual = float(self.dual_objective_dev()[0].item())
        return prim, dual, prim - dual

    def objective_parts_of(self, x):
        t = self.torch.from_numpy(self._to_stored(x)).to(self.device)
        v = self.objective_parts(t.data_ptr(), 1).cpu().numpy()
        return [float(a) for a in v]

    def objective_of(self, x):
        a, b, c = self.objective_parts_of(x)
        return a + b + c

    def smooth_gradient_of(self, x):
        t = self.torch.from_numpy(self._to_stored(x)).to(self.device)
        g = self.torch.empty(self.p_dev, dtype=self.torch.float64, device=self.device)
        _lib.check(_lib.load().ps_smooth_gradient(self.csr, self.params(), t.data_ptr(), 1, g.data_ptr(),
                                                  _lib.stream_ptr()))
        return self._to_original(g.cpu().numpy())

    def fixed_point_residual(self, gamma):
        """saga.py:299-317 at the current x."""
        if self._grad is None:
            self._grad = self.torch.empty(self.p_dev, dtype=self.torch.float64, device=self.device)
        _lib.check(_lib.load().ps_fixed_point_residual(self.csr, self.part, self.params(gamma),
                                                       self.coord.data_ptr(), self._grad.data_ptr(),
                                                       self._out.data_ptr() + 24, _lib.stream_ptr()))
        return float(self._out[3].item())

    def resync_average(self):
        _lib.check(_lib.load().ps_resync_average(self.csr, self.alpha.data_ptr(), self.coord.data_ptr(),
                                                 _lib.stream_ptr()))

    def field(self, f):
        """Field f (0 x, 1 abar, 2 D) of every coordinate, in ORIGINAL column order."""
        out = self.torch.empty(self.p, dtype=self.torch.float64, device=self.device)
        if self.perm is not None:
            _lib.check(_lib.load().ps_coord_get_perm(self.coord.data_ptr(), self.p, f, self.perm.data_ptr(),
                                                     out.data_ptr(), _lib.stream_ptr()))
        else:
            _lib.check(_lib.load().ps_coord_get(self.coord.data_ptr(), self.p, f, out.data_ptr(),
                                                _lib.stream_ptr()))
        return out

    def x(self):
        return self.field(0).cpu().numpy()

    def abar(self):
        return self.field(1).cpu().numpy()

    def weights(self):
        return self.field(2).cpu().numpy()

    def set_x(self, x):
        t = self.torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(self.device)
        if self.perm is not None:
            _lib.check(_lib.load().ps_coord_set_perm(self.coord.data_ptr(), self.p, 0, self.perm.data_ptr(),
                                                     t.data_ptr(), _lib.stream_ptr()))
        else:
            _lib.check(_lib.load().ps_coord_set(self.coord.data_ptr(), self.p, 0, t.data_ptr(), _lib.stream_ptr()))

    def fork(self):
        """Another solve of the same problem on the same GPU (e.g. a second
        lambda of a path running concurrently on its own stream): shares the
        device CSR, partition, layout and column statistics; owns x, abar,
        alpha, the progress counter and the sampler position.  D is copied."""
        import copy

        torch = self.torch
        other = copy.copy(self)
        with torch.cuda.device(self.device):
            other.coord = self.coord.clone()
            other.alpha = torch.zeros_like(self.alpha)
            other.counter = torch.zeros_like(self.counter)
            other._out = torch.zeros_like(self._out)
        for name in ("_scratch", "_side", "_grad", "_keep", "_dout"):
            if hasattr(other, name):
                setattr(other, name, None)
        other.slot_base = 0
        other.reset_state()
        return other

    def mean_blocks_per_row(self):
        """g-bar: mean number of distinct blocks per row (contiguous partitions;
        rows keyed by (row, col // G) on the device)."""
        if getattr(self, "_gbar", None) is None:
            torch = self.torch
            G = int(self.part.G) if self.part_kind == "contiguous" else 1
            rp = self.row_ptr.to(torch.int64)
            rows = torch.repeat_interleave(torch.arange(self.n, device=self.device), rp[1:] - rp[:-1])
            keys = rows * (self.p_dev // G + 1) + self.col.to(torch.int64) // G
            self._gbar = float(torch.unique(keys).numel()) / self.n
        return self._gbar

    def bytes_per_update(self, mean_k=None):
        """Algorithmic bytes per update (SURVEY.md §8d formulas).
        singleton: 2 s_ptr + s_y + 2 s_st + k (s_idx + s_val + 5 s_st);
        blocks of G (g blocks, m = G g coordinates per row):
        2 s_ptr + k (s_idx + s_val) + s_y + 2 s_st + 3 m s_st + k s_st + g s_st."""
        s_ptr = 4 if self.row_ptr_type == _lib.I32 else 8
        s_val = 4 if self.value_type == _lib.F32 else 8
        k = self.nnz / self.n if mean_k is None else mean_k
        if self.part_kind == "contiguous":
            g = self.mean_blocks_per_row()
            m = int(self.part.G) * g
            return 2 * s_ptr + k * (4 + s_val) + s_val + 2 * 8 + 3 * m * 8 + k * 8 + g * 8
        return 2 * s_ptr + s_val + 2 * 8 + k * (4 + s_val + 5 * 8)


def _on_device(fn):
    """Run a DeviceProblem method with the problem's GPU as the current device,
    so the library (which launches on cudaGetDevice()) and the default stream
    (torch's current stream of that device) match the state's memory."""

    @functools.wraps(fn)
    def wrapped(self, *args, **kwargs):
        with self.torch.cuda.device(self.device):
            return fn(self, *args, **kwargs)

    return wrapped


for _name in ("launch_config", "_scratch_for", "reset_state", "replay", "run_async", "run_async_monitored",
              "run_async_checkpointed", "objective_parts", "objective", "dual_objective_dev", "duality_gap",
              "objective_parts_of", "objective_of", "smooth_gradient_of", "fixed_point_residual",
              "resync_average", "field", "set_x", "fork", "block_stats", "mean_blocks_per_row"):
    setattr(DeviceProblem, _name, _on_device(getattr(DeviceProblem, _name)))
del _name
