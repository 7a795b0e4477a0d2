"""One async launch on a full-size large config (3 or 4) for ncu:
    python tools/prof_big.py 4 [fraction_of_epoch]"""
import json, sys
from pathlib import Path
import torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems
which = int(sys.argv[1]); frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.25
flags = int(sys.argv[3]) if len(sys.argv) > 3 else 0
c = problems.config3() if which == 3 else problems.config4()
dp = c["problem"]
gamma = pb.resolve_step_size("1/2L", dp.L, dp.n, c["loss"].lambda1)
count = int(dp.n * frac)
dp.run_async(count, gamma, seed=1, flags=flags)  # warm (launch 0)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); dp.run_async(count, gamma, seed=2, flags=flags); e.record(); torch.cuda.synchronize()  # launch 1 (profiled)
ms = s.elapsed_time(e)
print(json.dumps({"cfg": which, "count": count, "ms": ms, "Mups": count / ms / 1e3, "bytes_per_update": dp.bytes_per_update(),
                  "GBps": count * dp.bytes_per_update() / ms / 1e6}), flush=True)
