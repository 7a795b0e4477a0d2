"""A/B of the fast kernel's CSR L2 prefetch distance on the large configs
(ps_sched_t.flags bits 16..19: 15 = off, d = distance).  The prefetch was
measured (config 3 -3%, config 4 +-0) and removed from
the kernel, so on the current library every variant runs the same code.
    python tools/exp_prefetch.py 3 [dists...]"""
import json, sys
from pathlib import Path
import torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems

which = int(sys.argv[1])
dists = [int(v) for v in sys.argv[2:]] or [15, 2, 4, 8, 16]
c = problems.config3() if which == 3 else problems.config4()
dp = c["problem"]
gamma = pb.resolve_step_size("1/2L", dp.L, dp.n, c["loss"].lambda1)
dp.run_async(dp.n // 4, gamma, seed=5)  # warm-up
res = {d: [] for d in dists}
for rep in range(3):
    for d in (dists if rep % 2 == 0 else dists[::-1]):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); dp.run_async(dp.n // 2, gamma, seed=5 + rep, flags=d << 16); e.record()
        torch.cuda.synchronize()
        res[d].append(round(dp.n / 2 / s.elapsed_time(e) / 1e3, 1))
print(json.dumps({"cfg": which, "Mups": {("off" if d == 15 else d): v for d, v in res.items()}}), flush=True)
