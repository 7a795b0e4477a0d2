"""Convergence with / without the CTA-shared loads of stored block 0 (hshare):
the B = 8 instance of tests/test_gpu_batch.py, relative distance of each state's
objective from a 150-epoch deterministic replay after 40 / 60 / 80 epochs."""
import sys, json
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[2]; sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems, _lib
from paper_1707_06468_b200.device import DeviceProblem
from paper_1707_06468_b200.lambda_path import BatchedPath
from paper_1707_06468_b200.saga import resolve_step_size, worker_rng
rng = np.random.default_rng(11)
data = problems._zipf_logistic(rng, 8000, 40000, 20, 1.1, 100)
part = pb.contiguous_partition(data.n_features, 10)
lam1 = 1.0 / data.n_samples
loss = pb.Loss("logistic", lam1)
lmax = pb.group_lambda_max(data, part)
factors = (0.5, 0.2, 0.1, 0.05, 0.03, 0.02, 0.01, 0.005)
lams = [f * lmax for f in factors]
n = data.n_samples
frefs = []
for lam in lams[-3:]:
    dp = DeviceProblem(data, loss, pb.GroupL2Penalty(lam), part, drop_dead_blocks=True, hot_max=0)
    gamma = resolve_step_size("1/2L", dp.L, n, lam1)
    dp.replay(worker_rng(99, 0).integers(0, n, size=300 * n), gamma)
    frefs.append(dp.objective())
VARIANTS = [(0, 0, 0), (-1, 128, 0), (-1, 128, 4)] * 2 if len(sys.argv) < 2 else [tuple(int(t) for t in v.split(":")) for v in sys.argv[1].split(",")]
for nhot, hstride, hs in VARIANTS:
    _lib.check(_lib.load().ps_batch_tune2(nhot, hstride, hs, -1))
    for seed in (3, 4, 5):
        bp = BatchedPath(data, loss, part, B=8)
        gamma = resolve_step_size("1/2L", bp.dp.L, n, lam1)
        bp.reset(lams)
        out = {}
        done = 0
        for ep in (40, 60, 80):
            bp.run((ep - done) * n, gamma, seed=seed); done = ep
            sm = bp.summaries(range(5, 8), 0)
            out[ep] = [float(f"{(s['objective'] - f) / abs(f):.3e}") for s, f in zip(sm, frefs)]
        print(json.dumps({"nhot": nhot, "hstride": hstride, "hshare": hs, "seed": seed, "rel_gap_last3_lambdas": out}), flush=True)
        del bp
