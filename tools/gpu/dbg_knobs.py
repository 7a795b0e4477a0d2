"""v2 stability knobs on a config-3-like instance with H=1024 (tools/gpu)."""
import sys, json
from pathlib import Path
import numpy as np, torch
ROOT = Path(__file__).resolve().parents[2]; sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems
n = 2_000_000
c = problems.device_zipf_problem(n, int(1.5 * n), 0, 30, 1.2, 10_000, 1e-7, False, seed=0, hot_max=1024)
dp = c["problem"]
gamma = pb.resolve_step_size("1/2L", dp.L, dp.n, c["loss"].lambda1)
V2, V1, NOCL = 8388608, 4194304, 2097152
for name, kw in [("v1", dict(flags=V1)), ("v2", dict(flags=V2)), ("v2 nocluster", dict(flags=V2 | NOCL)),
                 ("v2 period16", dict(flags=V2, hot_period=16)), ("v2 c=2", dict(flags=V2, contention=2.0)),
                 ("v2 nc2", dict(flags=V2 | (2 << 24))), ("v1 nocluster", dict(flags=V1 | NOCL))]:
    dp.reset_state()
    objs = []
    for e in range(4):
        dp.run_async(dp.n, gamma, seed=3, **kw)
        objs.append(round(dp.objective(), 5))
    print(json.dumps({"name": name, "objs": objs}), flush=True)
