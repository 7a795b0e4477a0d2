"""Static split: convergence + time per epoch (per-epoch launches) on config 2."""
import json, sys
from pathlib import Path
import torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems
cfg = problems.config2(seed=0)
dp = pb.DeviceProblem(cfg["data"], cfg["loss"], cfg["penalty"], cfg["partition"], drop_dead_blocks=True, hot_max=int(sys.argv[1]) if len(sys.argv) > 1 else 1024)
n = dp.n
gamma = pb.resolve_step_size("1/2L", dp.L, n, cfg["loss"].lambda1)
fstar = json.loads((ROOT / "tests/golden/cfg2_fstar.json").read_text())["fstar"]

def run(tag, epochs=30, **kw):
    dp.reset_state()
    gaps, ms = [], []
    for _ in range(epochs):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        dp.run_async(n, gamma, seed=11, **kw)
        e.record(); torch.cuda.synchronize(); ms.append(s.elapsed_time(e))
        gaps.append((dp.objective() - fstar) / abs(fstar))
    hit = next((i + 1 for i, g in enumerate(gaps) if g <= 1e-6), None)
    t_hit = sum(ms[:hit]) if hit else None
    print(json.dumps({"tag": tag, "Mups": epochs * n / sum(ms) / 1e3, "ep_to_1e-6": hit, "kernel_ms_to_1e-6": t_hit,
                      "gap": [float(f"{g:.2e}") for g in gaps[4::5]]}), flush=True)

print(json.dumps({"H": dp.H}))
for fl, tag in ((0, "both_staged"), (32, "abar_direct"), (64, "x_direct"), (96, "both_direct")):
    run(f"{tag}_hp16_c3", ctas=148, warps_per_cta=24, contention=3.0, hot_period=16, flags=fl)
