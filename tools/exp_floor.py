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

for wpc in (32, 16):
    for hp in (4, 8, 16, 32):
        run(f"wpc{wpc}_hp{hp}_c2", [(30, dict(ctas=148, warps_per_cta=wpc, contention=2.0, hot_period=hp))])
run("wpc32_hp8_c4", [(30, dict(ctas=148, warps_per_cta=32, contention=4.0, hot_period=8))])
run("wpc32_hp8_c1", [(30, dict(ctas=148, warps_per_cta=32, contention=1.0, hot_period=8))])
run("wpc32_hp8_c2_live", [(30, dict(ctas=148, warps_per_cta=32, contention=2.0, hot_period=8, flags=2))])
run("nohot_wpc32", [(30, dict(ctas=148, warps_per_cta=32, contention=2.0, hot=False))])
