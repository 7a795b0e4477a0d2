"""Config 5 lambda path on one GPU with K concurrent solves (forks on K
streams, 148/K CTAs each): total throughput and per-lambda objectives."""
import json, sys, time
from pathlib import Path
import numpy as np, torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems, lambda_path as lp
cfg = problems.config5(seed=0)
d, part, loss = cfg["data"], cfg["partition"], cfg["loss"]
lams = lp.lambda_grid(pb.group_lambda_max(d, part), 16, 1e-3)
epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 30
ref = None
flags = int(sys.argv[3]) if len(sys.argv) > 3 else 0
hot = (sys.argv[4] == "hot") if len(sys.argv) > 4 else None
for K in [int(k) for k in (sys.argv[1] if len(sys.argv) > 1 else "1,2,4,8,16").split(",")]:
    solve = lp.device_solver(d, loss, part, epochs=epochs, mode="async", concurrent=K, flags=flags, hot=hot)
    if K > 1:
        solve.batch(lams[:K])  # warm
    else:
        solve(lams[0])
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    res = lp.run_path(lams, solve, rank=0, world=1)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    objs = np.array([r["objective"] for r in res])
    if ref is None:
        ref = objs
    print(json.dumps({"K": K, "ms": ms, "Mups": 16 * epochs * d.n_samples / ms / 1e3,
                      "max_rel_vs_K1": float(np.max(np.abs(objs - ref) / np.abs(ref))),
                      "objs": [round(o, 9) for o in objs]}), flush=True)
    del solve
    torch.cuda.empty_cache()
