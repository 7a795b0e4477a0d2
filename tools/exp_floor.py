"""Diagnose the convergence plateau of hot-column staging on config 2."""
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

def run(tag, phases):
    dp.reset_state()
    gaps = []
    kms = 0.0
    for epochs, kw in phases:
        for _ in range(epochs):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            dp.run_async(n, gamma, seed=11, **kw)
            e.record()
            torch.cuda.synchronize()
            kms += s.elapsed_time(e)
            gaps.append((dp.objective() - fstar) / abs(fstar))
    live = dp.abar(); dp.resync_average(); drift = float(np.max(np.abs(live - dp.abar())))
    res = dp.fixed_point_residual(gamma)
    hit = next((i + 1 for i, g in enumerate(gaps) if g <= 1e-6), None)
    print(json.dumps({"tag": tag, "Mups": len(gaps) * n / kms / 1e3, "ep_to_1e-6": hit,
                      "gap": [float(f"{g:.2e}") for g in gaps[4::5]], "final": gaps[-1],
                      "abar_drift": drift, "residual": res}), flush=True)

B = dict(ctas=148, warps_per_cta=32)
for hp in (8, 16, 32):
    run(f"w32_hp{hp}_b4_c2", [(30, dict(B, contention=2.0, hot_period=hp, batch=4))])
run("w16_hp16_b4_c2", [(30, dict(ctas=148, warps_per_cta=16, contention=2.0, hot_period=16, batch=4))])
run("w24_hp16_b4_c2", [(30, dict(ctas=148, warps_per_cta=24, contention=2.0, hot_period=16, batch=4))])
run("w16_hp16_b4_c4", [(30, dict(ctas=148, warps_per_cta=16, contention=4.0, hot_period=16, batch=4))])
