"""Configs 3/4: full-epoch objective and throughput vs the staged hot set size."""
import json, sys
from pathlib import Path
import torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems
which = int(sys.argv[1])
mf = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0 / 512
for hm in [int(x) for x in sys.argv[2].split(",")]:
    c = problems.config3(hot_max=hm, hot_min_frac=mf) if which == 3 else problems.config4(hot_max=hm, hot_min_frac=mf)
    dp = c["problem"]
    gamma = pb.resolve_step_size("1/2L", dp.L, dp.n, c["loss"].lambda1)
    dp.reset_state()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); dp.run_async(c["epochs"] * dp.n, gamma, seed=2); e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    print(json.dumps({"cfg": which, "hot_max": hm, "H": dp.H, "epochs": c["epochs"], "Mups": c["epochs"] * dp.n / ms / 1e3,
                      "objective": dp.objective()}), flush=True)
    del c, dp
    torch.cuda.empty_cache()
