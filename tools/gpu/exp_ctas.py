"""Updates/s vs number of CTAs (one per SM) for the async hot kernel:
per-SM-bound kernels scale linearly, globally bound ones saturate.
    python tools/gpu/exp_ctas.py 2|3 [flags]"""
import sys, json
from pathlib import Path
import torch
ROOT = Path(__file__).resolve().parents[2]; sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems
which = int(sys.argv[1]); flags = int(sys.argv[2]) if len(sys.argv) > 2 else 0
if which == 2:
    c = problems.config2(seed=0)
    dp = pb.DeviceProblem(c["data"], c["loss"], c["penalty"], c["partition"], drop_dead_blocks=True)
    step = "1/2L"
else:
    c = problems.config3() if which == 3 else problems.config4(); dp = c["problem"]; step = c["step"]
gamma = pb.resolve_step_size(step, dp.L, dp.n, c["loss"].lambda1)
out = {}
for ctas in [148, 74, 38, 148]:
    dp.reset_state()
    dp.run_async(dp.n, gamma, seed=1, ctas=ctas, flags=flags)  # warm
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cnt = dp.n * (3 if which == 2 else 1)
    s.record(); dp.run_async(cnt, gamma, seed=2, ctas=ctas, flags=flags); e.record(); torch.cuda.synchronize()
    out[ctas] = round(cnt / s.elapsed_time(e) / 1e3, 1)
print(json.dumps({"cfg": which, "flags": flags, "Mups_by_ctas": out}), flush=True)
