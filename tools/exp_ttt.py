"""Time to 1e-6 (bench.time_to_target: per-epoch launches, pipelined checkpoints)
and single-launch 30-epoch throughput on config 2 over (warps/CTA, period, c)."""
import json, sys
from pathlib import Path
import numpy as np, torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems
from bench import time_to_target
cfg = problems.config2(seed=0)
import os
dp = pb.DeviceProblem(cfg["data"], cfg["loss"], cfg["penalty"], cfg["partition"], drop_dead_blocks=True,
                      hot_max=int(os.environ.get("HOT_MAX", "256")))
print(json.dumps({"H": dp.H}), flush=True)
n = dp.n
gamma = pb.resolve_step_size("1/2L", dp.L, n, cfg["loss"].lambda1)
fstar = json.loads((ROOT / "tests/golden/cfg2_fstar.json").read_text())["fstar"]
grid = sys.argv[1] if len(sys.argv) > 1 else "32:24:4,32:24:6,32:16:4,24:16:4,24:16:6,32:32:6"
for g in grid.split(","):
    f = g.split(":")
    wpc, hp, c = f[0], f[1], f[2]
    kw = dict(warps_per_cta=int(wpc), hot_period=int(hp), contention=float(c),
              flags=int(f[3]) if len(f) > 3 else 0)
    dp.reset_state(); dp.run_async_checkpointed(2 * n, n, gamma, seed=3, **kw)  # warm
    tt = []
    for r in range(3):
        dp.reset_state()
        its, objs, walls = dp.run_async_checkpointed(30 * n, n, gamma, seed=7 + r, graph=True, **kw)
        rel = [(o - fstar) / abs(fstar) for o in objs]
        hit = next((i for i, x in enumerate(rel) if x <= 1e-6), None)
        tt.append((walls[hit] if hit is not None else None, hit + 1 if hit is not None else None))
    ms = []
    for r in range(3):
        dp.reset_state()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); dp.run_async(30 * n, gamma, seed=50 + r, **kw); e.record(); torch.cuda.synchronize()
        ms.append(s.elapsed_time(e))
    print(json.dumps({"wpc": wpc, "hp": hp, "c": c, "flags": kw["flags"], "ttt_ms_epochs": [(round(a * 1e3, 3) if a else None, b) for a, b in tt],
                      "solve_Mups": round(30 * n / np.mean(ms) / 1e3, 1)}), flush=True)
