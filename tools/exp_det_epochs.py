"""Config 2: relative gap per epoch of the deterministic (sequential) SPS
replay -- the reference algorithm's own convergence per epoch, to compare
with the async solver's epochs to 1e-6."""
import json, sys, time
from pathlib import Path
import numpy as np, torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems
from paper_1707_06468_b200.saga import worker_rng
cfg = problems.config2(seed=0)
dp = pb.DeviceProblem(cfg["data"], cfg["loss"], cfg["penalty"], cfg["partition"], drop_dead_blocks=True)
n = dp.n
gamma = pb.resolve_step_size("1/2L", dp.L, n, cfg["loss"].lambda1)
fstar = json.loads((ROOT / "tests/golden/cfg2_fstar.json").read_text())["fstar"]
seq = worker_rng(0, 0).integers(0, n, size=16 * n)
gaps = []
t = time.time()
for ep in range(16):
    dp.replay(seq[ep * n:(ep + 1) * n], gamma)
    gaps.append((dp.objective() - fstar) / abs(fstar))
print(json.dumps({"det_rel_gap_per_epoch": [float(f"{g:.3e}") for g in gaps], "s": time.time() - t}))
