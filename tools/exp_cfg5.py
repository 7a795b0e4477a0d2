"""Config 5 (group-lasso logistic, n=1e5, p=1e7, G=10): per-lambda solve throughput."""
import json, sys, time
from pathlib import Path
import torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems, lambda_path as lp
t0 = time.time()
cfg = problems.config5(seed=0)
print(json.dumps({"gen_s": time.time() - t0}), flush=True)
d, part, loss = cfg["data"], cfg["partition"], cfg["loss"]
t0 = time.time()
lam_max = pb.group_lambda_max(d, part)
solve = lp.device_solver(d, loss, part, epochs=int(sys.argv[1]) if len(sys.argv) > 1 else 5, mode="async")
dp = solve.problem
print(json.dumps({"prep_s": time.time() - t0, "lam_max": lam_max, "delta": dp.delta, "n_dead": dp.n_dead,
                  "max_slots": dp.stats.max_slots, "nblocks": dp.n_blocks}), flush=True)
for frac in (1.0, 0.1, 0.01, 0.001):
    torch.cuda.synchronize(); t0 = time.time()
    r = solve(frac * lam_max)
    torch.cuda.synchronize(); dt = time.time() - t0
    print(json.dumps({"lam": frac * lam_max, "Mups": r["updates"] / dt / 1e6, "obj": r["objective"], "nnz": r["nnz"], "s": dt}), flush=True)
