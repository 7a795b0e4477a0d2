"""Configs 3/4: fast-kernel CTA shape A/B (32 warps/CTA, 64 registers, NC=2
spills, vs the 24-warp variant), half-epoch launches, alternating order.
    python tools/exp_big_wpc.py 4"""
import json, sys
from pathlib import Path
import torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems

which = int(sys.argv[1])
c = problems.config3() if which == 3 else problems.config4()
dp = c["problem"]
gamma = pb.resolve_step_size("1/2L", dp.L, dp.n, c["loss"].lambda1)
variants = {"w32": dict(warps_per_cta=32), "w24": dict(warps_per_cta=24), "w24_hp24": dict(warps_per_cta=24, hot_period=24)}
dp.run_async(dp.n // 4, gamma, seed=5)
res = {k: [] for k in variants}
for rep in range(3):
    for k in (list(variants) if rep % 2 == 0 else list(variants)[::-1]):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); dp.run_async(dp.n // 2, gamma, seed=7 + rep, **variants[k]); e.record(); torch.cuda.synchronize()
        res[k].append(round(dp.n / 2 / s.elapsed_time(e) / 1e3, 1))
print(json.dumps({"cfg": which, "Mups": res}), flush=True)
