"""Configs 3/4: convergence profile of long asynchronous runs (per-epoch
checkpoints, stop-the-world schedule), the fixed-point residual at the end,
for a time-to-1e-6 measurement against a long-run F*.
    python tools/exp_big_ttt.py 3 [epochs] [hot_max]"""
import json, sys, time
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems

which = int(sys.argv[1])
epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 100
kw = {"hot_max": int(sys.argv[3])} if len(sys.argv) > 3 else {}
c = problems.config3(**kw) if which == 3 else problems.config4(**kw)
dp = c["problem"]
gamma = pb.resolve_step_size(c["step"], dp.L, dp.n, c["loss"].lambda1)
dp.run_async(dp.n // 10, gamma, seed=1)
dp.reset_state()
t0 = time.time()
import os
hp = int(os.environ.get("HP", "0"))  # flush period override (0: library default)
its, objs, secs = dp.run_async_checkpointed(epochs * dp.n, dp.n, gamma, seed=3, hot_period=hp)
res = dp.fixed_point_residual(gamma)
f, dual, gap = dp.duality_gap()
print(json.dumps({"cfg": which, "H": dp.H, "hp": hp, "epochs": epochs, "wall_s": time.time() - t0, "gamma": gamma, "L": dp.L,
                  "obj": [round(o, 15) for o in objs], "secs": [round(s, 5) for s in secs],
                  "residual_end": res, "gap_end": gap, "f_end": f}), flush=True)
