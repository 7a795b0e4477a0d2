"""hot3 vs hot2 on the n=8000 fast-kernel test instance at several grid sizes."""
import json, sys
from pathlib import Path
import numpy as np, torch
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems
from paper_1707_06468_b200.saga import resolve_step_size, worker_rng
FL = [int(v) for v in sys.argv[1].split(",")]
rng = np.random.default_rng(3)
data = problems._zipf_logistic(rng, 8000, 50000, 20, 1.1, 100)
lam = 1.0 / 8000
dp = pb.DeviceProblem(data, pb.Loss("logistic", lam), pb.L1Penalty(lam), pb.singleton_partition(50000), drop_dead_blocks=True)
g = resolve_step_size("1/2L", dp.L, dp.n, lam)
dp.reset_state(); dp.replay(worker_rng(99, 0).integers(0, dp.n, size=200 * dp.n), g); fref = dp.objective()
for ctas in [int(c) for c in (sys.argv[2] if len(sys.argv) > 2 else "1,2,8,32,148").split(",")]:
    for fl in FL:
        r = []
        for seed in (5, 6):
            dp.reset_state(); dp.run_async(60 * dp.n, g, seed=seed, flags=fl, ctas=ctas, warps_per_cta=32); r.append((dp.objective() - fref) / fref)
        print(json.dumps({"ctas": ctas, "flags": fl, "rel": r}), flush=True)
