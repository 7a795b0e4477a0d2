"""hot3 diagnosis at one CTA: abar consistency (live abar vs A^T alpha / n) after an async run."""
import json, sys
from pathlib import Path
import numpy as np, torch
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems
from paper_1707_06468_b200.saga import resolve_step_size
FL = [int(v) for v in sys.argv[1].split(",")]
rng = np.random.default_rng(3)
data = problems._zipf_logistic(rng, 8000, 50000, 20, 1.1, 100)
lam = 1.0 / 8000
dp = pb.DeviceProblem(data, pb.Loss("logistic", lam), pb.L1Penalty(lam), pb.singleton_partition(50000), drop_dead_blocks=True)
g = resolve_step_size("1/2L", dp.L, dp.n, lam)
for fl in FL:
    for ep in (5,):
        dp.reset_state(); dp.run_async(ep * dp.n, g, seed=5, flags=fl, ctas=1, warps_per_cta=32)
        live = dp.abar(); x = dp.x(); dp.resync_average(); ref = dp.abar()
        d = np.abs(live - ref); j = int(np.argmax(d))
        print(json.dumps({"flags": fl, "epochs": ep, "abar_maxdiff": float(d.max()), "at": j, "live": float(live[j]), "ref": float(ref[j]),
                          "n_bad": int((d > 1e-12).sum()), "x_nnz": int((x != 0).sum()), "obj": dp.objective()}), flush=True)
