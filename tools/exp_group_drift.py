"""Config 5 at lambda_max with hot-block staging: abar drift and x norm after a run."""
import json, sys
from pathlib import Path
import numpy as np, torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems, lambda_path as lp
cfg = problems.config5(seed=0)
d, part, loss = cfg["data"], cfg["partition"], cfg["loss"]
lam_max = pb.group_lambda_max(d, part)
solve = lp.device_solver(d, loss, part, epochs=1, mode="async")
dp, gamma, n = solve.problem, solve.gamma, d.n_samples
dp.lam2 = lam_max
for tag, kw in (("hot", dict(hot=True)), ("cold", dict(hot=False)), ("hot_1cta", dict(hot=True, ctas=1)),
                ("hot_c0", dict(hot=True, contention=0.0)), ("hot_delta", dict(hot=True, flags=32))):
    dp.reset_state()
    for ep in range(10):
        dp.run_async(n, gamma, seed=3, **kw)
    torch.cuda.synchronize()
    x = dp.field(0)
    live = dp.abar(); dp.resync_average(); drift = float(np.max(np.abs(live - dp.abar())))
    xs = x.cpu().numpy()
    print(json.dumps({"tag": tag, "obj": dp.objective(), "abar_drift": drift, "x_nnz": int((xs != 0).sum()),
                      "x_max": float(np.abs(xs).max()), "x_hot_max": float(np.abs(xs[:dp.H * 32]).max())}), flush=True)
