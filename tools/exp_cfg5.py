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
ep = int(sys.argv[1]) if len(sys.argv) > 1 else 5
gamma = solve.gamma
for frac, hot in ((1.0, True), (1.0, False), (0.01, True), (0.01, False), (0.001, False)):
    dp.lam2 = frac * lam_max
    dp.reset_state()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(ep):
        dp.run_async(d.n_samples, gamma, seed=1, hot=hot)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    xt = dp.field(0)
    print(json.dumps({"lam": frac * lam_max, "hot": hot, "Mups": ep * d.n_samples / ms / 1e3, "kernel_ms": ms, "obj": dp.objective(),
                      "nnz": int((xt != 0).sum().item())}), flush=True)
