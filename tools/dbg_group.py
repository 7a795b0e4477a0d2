import json, sys
from pathlib import Path
import numpy as np, torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems
cfg = problems.config5(seed=1, n=20000, p=200_000)
d, part, loss = cfg["data"], cfg["partition"], cfg["loss"]
lam = 0.1 * pb.group_lambda_max(d, part)
for hm, hp in ((40, 1000000), (40, 8), (1024, 8), (10, 8)):
    dp = pb.DeviceProblem(d, loss, pb.GroupL2Penalty(lam), part, drop_dead_blocks=True, hot_min_rows=0, hot_max=hm)
    gamma = pb.resolve_step_size("1/2L", dp.L, dp.n, loss.lambda1)
    res = []
    for ep in range(3):
        dp.run_async(dp.n, gamma, seed=2, hot_period=hp, ctas=8)
        x = dp.x(); ab = dp.abar()
        res.append((float(dp.objective()), int(np.isnan(x).sum()), int(np.isnan(ab).sum()), float(np.nanmax(np.abs(x)))))
    c, w, _ = dp.launch_config(dp._sched(1, hot=True, ctas=8))
    print(json.dumps({"hot_max": hm, "H": dp.H, "hp": hp, "grid": [c, w], "res": res}), flush=True)
dp = pb.DeviceProblem(d, loss, pb.GroupL2Penalty(lam), part, drop_dead_blocks=True, hot_min_rows=0, hot_max=40)
gamma = pb.resolve_step_size("1/2L", dp.L, dp.n, loss.lambda1)
for ep in range(3):
    dp.run_async(dp.n, gamma, seed=2, hot=False, ctas=8)
print(json.dumps({"nohot": float(dp.objective())}))
