"""Config 5 lambda path (16 concurrent solves, lane kernel): zero blocks the
prox keeps at zero skipped (skip=1, the default now) or stored
(PS_FLAG_GROUP_STORE_ZEROS, skip=0).  Total time and per-lambda duality-gap certificates; then each
lambda alone with the same per-solve grid, to see where the time goes.
    python tools/exp_path_skip.py"""
import json, sys
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import _lib, lambda_path as lp, problems

cfg = problems.config5(seed=0)
d, part, loss = cfg["data"], cfg["partition"], cfg["loss"]
lams = lp.lambda_grid(pb.group_lambda_max(d, part), 16, 1e-3)
out = {}
for rep in range(2):
    for skip in (0, 1):
        fl = _lib.FLAG_GROUP_LANE | (0 if skip else _lib.FLAG_GROUP_STORE_ZEROS)
        solve = lp.device_solver(d, loss, part, epochs=30, mode="async", concurrent=16, flags=fl)
        solve.batch(lams)  # warm-up
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); res = solve.batch(lams); e.record(); torch.cuda.synchronize()
        out.setdefault(skip, []).append({"ms": s.elapsed_time(e),
                                         "rel_gap": [float(f"{r['gap'] / abs(r['objective']):.2e}") for r in res]})
        if rep == 0:  # per-lambda times, one solve at a time on the concurrent path's grid
            dp = solve.problem
            per = []
            for lam in lams:
                dp.lam2 = float(lam); dp.reset_state()
                s.record()
                dp.run_async(30 * dp.n, solve.gamma, seed=0, ctas=9, flags=fl, hot=False)
                e.record(); torch.cuda.synchronize()
                per.append(round(s.elapsed_time(e), 1))
            out.setdefault(f"per_lambda_ms_{skip}", per)
        del solve
        torch.cuda.empty_cache()
print(json.dumps(out), flush=True)
