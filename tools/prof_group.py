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
hot = len(sys.argv) > 1 and sys.argv[1] == "hot"
for _ in range(3):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); dp.run_async(d.n_samples * 3, solve.gamma, seed=1, hot=hot); e.record(); torch.cuda.synchronize()
    print(json.dumps({"hot": hot, "Mups": 3 * d.n_samples / s.elapsed_time(e) / 1e3}), flush=True)
