"""Plateau diagnosis for the fast kernel's hot staging (config 2): hot step
scaling, staged count, and switching staging off after the plateau."""
import json, sys
from pathlib import Path
import numpy as np, torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems

cfg = problems.config2(seed=0)
fstar = json.loads((ROOT / "tests/golden/cfg2_fstar.json").read_text())["fstar"]
cache = {}

def prob(hot_max):
    if hot_max not in cache:
        cache[hot_max] = pb.DeviceProblem(cfg["data"], cfg["loss"], cfg["penalty"], cfg["partition"],
                                          drop_dead_blocks=True, hot_max=hot_max)
    return cache[hot_max]

def run(tag, phases, hot_max=256):
    dp = prob(hot_max)
    n = dp.n
    gamma = pb.resolve_step_size("1/2L", dp.L, n, cfg["loss"].lambda1)
    dp.reset_state()
    gaps, kms, ms = [], 0.0, []
    for epochs, kw in phases:
        for _ in range(epochs):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            dp.run_async(n, gamma, seed=11, **kw)
            e.record()
            torch.cuda.synchronize()
            kms += s.elapsed_time(e)
            ms.append(s.elapsed_time(e))
            gaps.append((dp.objective() - fstar) / abs(fstar))
    hit = next((i + 1 for i, g in enumerate(gaps) if g <= 1e-6), None)
    print(json.dumps({"tag": tag, "H": dp.H, "Mups": len(gaps) * n / kms / 1e3, "ep_to_1e-6": hit,
                      "ms_to_1e-6": sum(ms[:hit]) if hit else None,
                      "gap": [float(f"{g:.2e}") for g in gaps[4::5]], "final": gaps[-1]}), flush=True)

S = dict(contention=4.0, hot_period=16)
for hp in (16, 24, 32):
    for c in (3.0, 4.0, 6.0):
        run(f"w32_hp{hp}_c{c}", [(30, dict(S, hot_period=hp, contention=c))])
