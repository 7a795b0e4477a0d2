"""Concurrency vs convergence on config 2 (unstaged and staged)."""
import json, sys
from pathlib import Path
import numpy as np, torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems

cfg = problems.config2(seed=0)
dp = pb.DeviceProblem(cfg["data"], cfg["loss"], cfg["penalty"], cfg["partition"], drop_dead_blocks=True)
n = dp.n
gamma = pb.resolve_step_size("1/2L", dp.L, n, cfg["loss"].lambda1)
fstar = json.loads((ROOT / "tests/golden/cfg2_fstar.json").read_text())["fstar"]

def run(tag, epochs, per_launch=1, **kw):
    dp.reset_state()
    gaps, kms = [], 0.0
    for _ in range(epochs // per_launch):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        dp.run_async(n * per_launch, gamma, seed=11, **kw)
        e.record(); torch.cuda.synchronize(); kms += s.elapsed_time(e)
        gaps.append((dp.objective() - fstar) / abs(fstar))
    hit = next((i + 1 for i, g in enumerate(gaps) if g <= 1e-6), None)
    print(json.dumps({"tag": tag, "Mups": epochs * n / kms / 1e3, "launch_to_1e-6": hit, "per_launch": per_launch,
                      "gap": [float(f"{g:.2e}") for g in gaps[max(0, len(gaps) // 6 - 1)::max(1, len(gaps) // 6)]]}), flush=True)

W = dict(ctas=148, warps_per_cta=32)
exps = sys.argv[1] if len(sys.argv) > 1 else "all"
run("nohot_w32_b32_pl10_c2", 30, per_launch=10, hot=False, batch=32, contention=2.0, **W)
run("nohot_w32_b4_pl10_c2", 30, per_launch=10, hot=False, batch=4, contention=2.0, **W)
run("nohot_w14_b4_c2", 30, hot=False, batch=4, contention=2.0, ctas=148, warps_per_cta=14)
run("nohot_w7_b4_c2", 30, hot=False, batch=4, contention=2.0, ctas=148, warps_per_cta=7)
run("nohot_w32_b4_c8", 30, hot=False, batch=4, contention=8.0, **W)
run("nohot_w32_b4_c0", 30, hot=False, batch=4, contention=0.0, ctas=148, warps_per_cta=2)
run("hot_w32_b32_pl10_hp16_c2", 30, per_launch=10, batch=32, contention=2.0, hot_period=16, **W)
run("hot_w14_b4_hp8_c2", 30, batch=4, contention=2.0, hot_period=8, ctas=148, warps_per_cta=14)
run("hot_w32_b4_hp16_c2_pl5", 30, per_launch=5, batch=4, contention=2.0, hot_period=16, **W)
