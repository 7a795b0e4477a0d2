"""Configs 3/4 on the device: generation, prep, async throughput and convergence."""
import json, sys, time
from pathlib import Path
import numpy as np, torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems
which = int(sys.argv[1]); scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
t0 = time.time()
if which == 3:
    c = problems.config3(n=int(2e7 * scale), p=int(3e7 * scale))
else:
    c = problems.config4(n=int(4.5e7 * scale), p=int(1e6 * max(scale, 0.05)))
torch.cuda.synchronize()
dp = c["problem"]
print(json.dumps({"cfg": which, "n": dp.n, "p": dp.p, "nnz": dp.nnz, "gen+prep_s": time.time() - t0, "H": dp.H,
                  "delta": dp.delta, "n_dead": dp.n_dead, "L": dp.L, "mem_GB": torch.cuda.memory_allocated() / 1e9}), flush=True)
gamma = pb.resolve_step_size("1/2L", dp.L, dp.n, c["loss"].lambda1)
f0 = dp.objective()
objs, ms = [f0], []
for ep in range(c["epochs"] * 2):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); dp.run_async(dp.n, gamma, seed=5); e.record(); torch.cuda.synchronize()
    ms.append(s.elapsed_time(e)); objs.append(dp.objective())
live = dp.abar(); dp.resync_average(); drift = float(np.max(np.abs(live - dp.abar())))
print(json.dumps({"Mups_per_epoch": [round(dp.n / m / 1e3, 1) for m in ms], "obj": objs,
                  "abar_drift": drift, "bytes_per_update": dp.bytes_per_update()}), flush=True)
