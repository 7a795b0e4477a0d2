"""Config 5 convergence: fast group kernel vs generic kernel vs deterministic, per lambda."""
import json, sys
from pathlib import Path
import torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems, lambda_path as lp
n_arg = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
p_arg = int(sys.argv[2]) if len(sys.argv) > 2 else 10_000_000
cfg = problems.config5(seed=0, n=n_arg, p=p_arg)
d, part, loss = cfg["data"], cfg["partition"], cfg["loss"]
lam_max = pb.group_lambda_max(d, part)
solve = lp.device_solver(d, loss, part, epochs=1, mode="async")
dp, gamma, n = solve.problem, solve.gamma, d.n_samples
print(json.dumps({"n": n, "p": d.n_features, "H": dp.H, "lam_max": lam_max}), flush=True)
for frac in (1.0, 0.1, 0.01):
    lam = frac * lam_max
    dp.lam2 = lam
    for tag, kw in (("c2", dict(contention=2.0)), ("c4", dict(contention=4.0)), ("c2_delta", dict(contention=2.0, flags=32)),
                    ("c8", dict(contention=8.0))):
        dp.reset_state(); objs = []
        for ep in range(30):
            dp.run_async(n, gamma, seed=3, **kw)
            if ep % 5 == 4: objs.append(round(dp.objective(), 12))
        print(json.dumps({"frac": frac, "tag": tag, "obj": objs}), flush=True)
    dp.reset_state()
    seq = pb.worker_rng(0, 0).integers(0, n, size=n)
    objs = []
    for ep in range(int(sys.argv[3]) if len(sys.argv) > 3 else 3):
        dp.replay(seq, gamma); objs.append(round(dp.objective(), 12))
    print(json.dumps({"frac": frac, "tag": "det", "obj": objs}), flush=True)
