"""Deterministic parity at the FULL BASELINE sizes of configs 3 and 4, through
the production layout (per-step goldens on a prefix of the
index sequence for the configs the reference cannot hold).

The device problem is the one the bench solves: generated on the device (K7),
hot-column layout with the default number of staged columns (1024 / 512 hot
columns renumbered to stride-32 positions, rows re-sorted, coordinates
padded), int32 row pointers.  A 2e5-step prefix of the reference's PCG64
stream (saga.py:45-51, 233-235) is replayed by the deterministic kernel and by
the C oracle on a host copy of the same CSR (the sampled rows; every other row
empty, so the oracle's alpha / abar arithmetic still divides by the full n).
The oracle's per-column weights D_j = n / n_j come from a host histogram of the
whole device column array (independent of the device's ps_prepare), and L
from a host pass over the row norms.

Tolerances: x within 1e-9 relative (the deterministic bar), alpha and abar
within 1e-9, D and L exact / 1e-14.
"""

import numpy as np
import pytest

import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems

pytestmark = pytest.mark.gpu

STEPS = 200_000
CHUNK = 1 << 27


def _host_stats(dp):
    """Column histogram and max row sqnorm of the device CSR, on the host, chunked."""
    import torch

    counts = np.zeros(dp.p_dev, dtype=np.int64)
    for s in range(0, dp.nnz, CHUNK):
        counts += np.bincount(dp.col[s:s + CHUNK].cpu().numpy(), minlength=dp.p_dev)
    rp = dp.row_ptr.cpu().numpy().astype(np.int64)
    msq = 0.0
    rows_per = max(1, CHUNK // max(1, int(rp[1] - rp[0])))
    for r0 in range(0, dp.n, rows_per):
        r1 = min(dp.n, r0 + rows_per)
        v = dp.val[int(rp[r0]):int(rp[r1])].to(torch.float64).cpu().numpy()
        sq = np.add.reduceat(v * v, rp[r0:r1] - rp[r0]) if r1 > r0 else np.zeros(0)
        msq = max(msq, float(sq.max()))
    return counts, rp, msq


def _oracle_for_prefix(dp, c, rp, seq, counts):
    """Oracle problem holding only the sampled rows (others empty), with the
    full-matrix weights."""
    from oracle import oracle as O
    import torch

    rows = np.unique(seq)
    lens = rp[rows + 1] - rp[rows]
    ptr = np.zeros(dp.n + 1, dtype=np.int64)
    k = np.zeros(dp.n, dtype=np.int64)
    k[rows] = lens
    np.cumsum(k, out=ptr[1:])
    starts = torch.from_numpy(rp[rows]).to(dp.device)
    ln = torch.from_numpy(lens).to(dp.device)
    idx = torch.repeat_interleave(starts - torch.cumsum(ln, 0) + ln, ln) + torch.arange(int(ln.sum()),
                                                                                      device=dp.device)
    col = dp.col[idx].cpu().numpy().astype(np.int64)
    val = dp.val[idx].to(torch.float64).cpu().numpy()
    y = dp.y.to(torch.float64).cpu().numpy()
    P = O.OracleProblem(ptr, col, val, y, dp.p_dev, loss="logistic", lambda1=c["loss"].lambda1, penalty="l1",
                        lam2=c["penalty"].lam2)
    n = dp.n
    with np.errstate(divide="ignore"):
        P.d_B[:] = np.where(counts > 0, n / np.maximum(counts, 1), 0.0)  # data.py:259-261, dead -> 0
    return P


@pytest.mark.parametrize("which", [3, 4])
def test_full_size_prefix_replay_matches_oracle(cuda, which):
    import torch

    c = problems.config3() if which == 3 else problems.config4()
    dp = c["problem"]
    assert dp.perm is not None and dp.H > 0 and dp.hot_shift == 5  # the production layout
    assert dp.H == (1024 if which == 3 else 512)
    counts, rp, msq = _host_stats(dp)
    # K5 weights and L against the host histogram / row norms
    w = dp.coord[:, 2].cpu().numpy()
    with np.errstate(divide="ignore"):
        want = np.where(counts > 0, dp.n / np.maximum(counts, 1), 0.0)
    assert np.array_equal(w[: len(want)], want)
    assert dp.L == pytest.approx(0.25 * msq + c["loss"].lambda1, rel=1e-14)
    gamma = pb.resolve_step_size(c["step"], dp.L, dp.n, c["loss"].lambda1)
    seq = pb.worker_rng(0, 0).integers(0, dp.n, size=STEPS)
    dp.reset_state()
    dp.replay(seq, gamma)
    P = _oracle_for_prefix(dp, c, rp, seq, counts)
    x, alpha, abar = P.run_sequential(gamma, seq)
    xd = dp.coord[:, 0].cpu().numpy()  # stored (permuted) order, as the oracle's CSR
    rel = np.max(np.abs(xd - x)) / np.max(np.abs(x))
    assert rel <= 1e-9, f"config {which}: rel {rel:.3e}"
    ad = dp.alpha.cpu().numpy()
    assert np.max(np.abs(ad - alpha)) <= 1e-9 * max(1.0, np.max(np.abs(alpha)))
    abd = dp.coord[:, 1].cpu().numpy()
    assert np.max(np.abs(abd - abar)) <= 1e-9 * max(1e-300, np.max(np.abs(abar)))
    del dp, c
    torch.cuda.empty_cache()


def test_int64_row_pointers_match_reference(cuda, small_cases, golden_small):
    """PS_I64 row pointers (the int64 kernel instantiations): a golden case
    replayed with row_ptr forced to int64 (the reference's own CSR dtype,
    data.py:46-48)."""
    from paper_1707_06468_b200 import _lib
    from paper_1707_06468_b200.device import DeviceProblem

    for name in ("cfg2_small", "grp_contig"):
        case, g = small_cases[name], golden_small
        dp = DeviceProblem(case["data"], case["loss"], case["penalty"], case["partition"],
                           drop_dead_blocks=case["drop_dead"], index_dtype="int64")
        assert dp.row_ptr_type == _lib.I64
        mu = case["loss"].lambda1
        gamma = pb.resolve_step_size(case["step"], dp.L, dp.n, mu if mu > 0 else None)
        seq = pb.worker_rng(case["seed"], 0).integers(0, dp.n, size=case["steps"])
        done = 0
        for kk, s in enumerate(case["segments"]):
            dp.replay(seq[done:s], gamma)
            done = s
            ref = g[f"{name}__x"][kk]
            assert np.max(np.abs(dp.x() - ref)) <= 1e-9 * max(np.max(np.abs(ref)), 1e-300)
        # and the asynchronous kernels on the int64 layout reach the same objective region
        dp.reset_state()
        dp.run_async(20 * dp.n, gamma, seed=3)
        assert np.isfinite(dp.objective())
