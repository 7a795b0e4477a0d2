"""v1 vs v2 hot kernel on a config-3-like instance with H=1024 staged columns:
per-epoch objective and the abar drift |abar - A^T alpha / n| (tools/gpu)."""
import sys, json
from pathlib import Path
import numpy as np, torch
ROOT = Path(__file__).resolve().parents[2]; sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
hm = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
c = problems.device_zipf_problem(n, int(1.5 * n), 0, 30, 1.2, 10_000, 1e-7, False, seed=0, hot_max=hm)
dp = c["problem"]
gamma = pb.resolve_step_size("1/2L", dp.L, dp.n, c["loss"].lambda1)
print("H", dp.H, "shift", dp.hot_shift, flush=True)
for flags in [4194304, 0]:
    dp.reset_state()
    objs = []
    for e in range(6):
        dp.run_async(dp.n, gamma, seed=3, flags=flags)
        objs.append(dp.objective())
    live = dp.abar(); dp.resync_average(); drift = float(np.max(np.abs(live - dp.abar())))
    print(json.dumps({"flags": flags, "objs": objs, "abar_drift": drift}), flush=True)
