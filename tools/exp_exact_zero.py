"""lambda2 = 2 lambda_max (optimum x = 0): nonzeros left after a 30-epoch
async solve (count, max |x_j|, relative objective error), per commit variant
and seed (test_zero_commits_keep_exact_zeros).  The fetch-add flush measured
with it has been removed from the kernel.
    python tools/exp_exact_zero.py"""
import json, sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import _lib, problems
from paper_1707_06468_b200.device import DeviceProblem
from paper_1707_06468_b200.saga import resolve_step_size

rng = np.random.default_rng(3)
data = problems._zipf_logistic(rng, 8000, 50000, 20, 1.1, 100)
lam1 = 1.0 / data.n_samples
dp = DeviceProblem(data, pb.Loss("logistic", lam1), pb.L1Penalty(2.0 * pb.lambda_max(data)),
                   pb.singleton_partition(data.n_features), drop_dead_blocks=True)
gamma = resolve_step_size("1/2L", dp.L, dp.n, lam1)
out = {}
for name, fl in (("default", 0), ("zero_immediate", _lib.FLAG_ZERO_IMMEDIATE)):
    nz = []
    for seed in range(8):
        dp.reset_state()
        dp.run_async(30 * dp.n, gamma, seed=seed, flags=fl)
        x = dp.x()
        nz.append((int(np.count_nonzero(x)), float(np.abs(x).max()), float((dp.objective() - np.log(2.0)) / np.log(2.0))))
    out[name] = nz
print(json.dumps(out), flush=True)
