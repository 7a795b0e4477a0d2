"""Config 5 group kernels: throughput and convergence per lambda
(lane-per-block with / without hot-block staging vs the warp-cooperative kernel)."""
import json, sys
from pathlib import Path
import torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems, lambda_path as lp
cfg = problems.config5(seed=0)
d, part, loss = cfg["data"], cfg["partition"], cfg["loss"]
lam_max = pb.group_lambda_max(d, part)
solve = lp.device_solver(d, loss, part, epochs=1, mode="async")
dp, gamma, n = solve.problem, solve.gamma, d.n_samples
print(json.dumps({"H": dp.H, "hot_shift": dp.hot_shift, "p_dev": dp.p_dev}), flush=True)
epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 30
grid = [("hot", dict(hot=True)), ("hot_div2", dict(hot=True, flags=2 << 8)), ("hot_div4", dict(hot=True, flags=4 << 8)),
        ("hot_div16", dict(hot=True, flags=16 << 8)), ("hot_div4_c8", dict(hot=True, flags=4 << 8, contention=8.0)),
        ("warp_cold", dict(hot=False, flags=64))]
for frac in (1.0, 0.3, 0.01):
    dp.lam2 = frac * lam_max
    for tag, kw in grid:
        dp.reset_state(); objs = []; ms = 0.0
        for ep in range(epochs):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); dp.run_async(n, gamma, seed=3, **kw); e.record(); torch.cuda.synchronize()
            ms += s.elapsed_time(e)
            if ep % 5 == 4: objs.append(round(dp.objective(), 12))
        print(json.dumps({"frac": frac, "tag": tag, "Mups": epochs * n / ms / 1e3, "obj": objs}), flush=True)
