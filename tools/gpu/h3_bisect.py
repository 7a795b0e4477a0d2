"""hot3 stability bisect: the n=8000 fast-kernel test instance (fp64 values) and
config 3 (6 epochs), for a list of flag values."""
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
for vd in ("float64", "auto"):
    dp = pb.DeviceProblem(data, pb.Loss("logistic", lam), pb.L1Penalty(lam), pb.singleton_partition(50000), drop_dead_blocks=True, value_dtype=vd)
    g = resolve_step_size("1/2L", dp.L, dp.n, lam)
    dp.reset_state(); dp.replay(worker_rng(99, 0).integers(0, dp.n, size=200 * dp.n), g); fref = dp.objective()
    for fl in FL:
        r = []
        for seed in (5, 6):
            dp.reset_state(); dp.run_async(60 * dp.n, g, seed=seed, flags=fl); r.append((dp.objective() - fref) / fref)
        print(json.dumps({"inst": vd, "flags": fl, "rel": r}), flush=True)
c = problems.config3(); dp = c["problem"]; g = pb.resolve_step_size(c["step"], dp.L, dp.n, c["loss"].lambda1)
for fl in FL:
    dp.reset_state(); dp.run_async(6 * dp.n, g, seed=3, flags=fl)
    print(json.dumps({"inst": "cfg3", "flags": fl, "obj6": dp.objective()}), flush=True)
