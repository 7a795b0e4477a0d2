"""Batch (slots per counter claim) vs convergence, fixed concurrency; flags=4 scrambles slot order."""
import json, sys
from pathlib import Path
import torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems
cfg = problems.config2(seed=0)
dp = pb.DeviceProblem(cfg["data"], cfg["loss"], cfg["penalty"], cfg["partition"], drop_dead_blocks=True)
n = dp.n
gamma = pb.resolve_step_size("1/2L", dp.L, n, cfg["loss"].lambda1)
fstar = json.loads((ROOT / "tests/golden/cfg2_fstar.json").read_text())["fstar"]
for batch, flags, wpc in [(1, 0, 32), (1, 4, 32), (4, 4, 32), (64, 0, 32), (64, 4, 32), (1, 0, 8), (64, 0, 8)]:
    dp.reset_state()
    gaps = []
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(3):
        dp.run_async(n * 10, gamma, seed=11, batch=batch, ctas=148, warps_per_cta=wpc, contention=2.0, hot=False,
                     flags=flags)
        gaps.append((dp.objective() - fstar) / abs(fstar))
    e.record(); torch.cuda.synchronize()
    print(json.dumps({"batch": batch, "flags": flags, "wpc": wpc, "Mups": 30 * n / s.elapsed_time(e) / 1e3,
                      "gap": [float(f"{g:.2e}") for g in gaps]}), flush=True)
