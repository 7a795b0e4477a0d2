"""Configs 3/4: async throughput vs the staged hot set size and flush period."""
import json, sys
from pathlib import Path
import torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems
which = int(sys.argv[1])
for hm in [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "256,1024").split(",")]:
    c = problems.config3(hot_max=hm) if which == 3 else problems.config4(hot_max=hm)
    dp = c["problem"]
    gamma = pb.resolve_step_size("1/2L", dp.L, dp.n, c["loss"].lambda1)
    for hp in (16, 24, 32):
        dp.reset_state()
        dp.run_async(dp.n // 4, gamma, seed=1, hot_period=hp)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); dp.run_async(dp.n, gamma, seed=2, hot_period=hp); e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e)
        print(json.dumps({"cfg": which, "hot_max": hm, "H": dp.H, "hp": hp, "Mups": dp.n / ms / 1e3,
                          "obj_after_1.25ep": dp.objective()}), flush=True)
    del c, dp
    torch.cuda.empty_cache()
