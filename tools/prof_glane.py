"""One config-5 solve on the lane-per-block kernel with 9 CTAs (the per-solve
grid of the 16-way concurrent lambda path), for ncu."""
import sys, json
from pathlib import Path
import torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems, lambda_path as lp
cfg = problems.config5(seed=0)
d, part, loss = cfg["data"], cfg["partition"], cfg["loss"]
lam = 0.01 * pb.group_lambda_max(d, part)
solve = lp.device_solver(d, loss, part, epochs=1, mode="async")
dp = solve.problem; dp.lam2 = lam
for rep in range(2):
    dp.reset_state()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); dp.run_async(3 * d.n_samples, solve.gamma, seed=rep, ctas=9, flags=128, hot=False); e.record()
    torch.cuda.synchronize()
    print(json.dumps({"Mups": 3 * d.n_samples / s.elapsed_time(e) / 1e3}), flush=True)
