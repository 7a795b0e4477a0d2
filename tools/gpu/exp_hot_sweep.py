"""sps_hot_kernel: staged columns (hot_max) x flush period on configs 2/3/4:
30/10/5-epoch launch updates/s and, for config 2, epochs to 1e-6 (tools/gpu).
    python tools/gpu/exp_hot_sweep.py 2|3|4"""
import sys, json, math
from pathlib import Path
import torch
ROOT = Path(__file__).resolve().parents[2]; sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems
which = int(sys.argv[1])
fstar = json.loads((ROOT / "tests" / "golden" / "cfg2_fstar.json").read_text())["fstar"] if which == 2 else None
for hm in (256, 512, 1024):
    if which == 2:
        c = problems.config2(seed=0)
        dp = pb.DeviceProblem(c["data"], c["loss"], c["penalty"], c["partition"], drop_dead_blocks=True, hot_max=hm)
        ep = 30
    else:
        c = problems.config3(hot_max=hm) if which == 3 else problems.config4(hot_max=hm)
        dp = c["problem"]; ep = c["epochs"]
    gamma = pb.resolve_step_size("1/2L", dp.L, dp.n, c["loss"].lambda1)
    for hp in (16, 24, 32):
        dp.reset_state(); dp.run_async(dp.n, gamma, seed=1, hot_period=hp); dp.reset_state()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); dp.run_async(ep * dp.n, gamma, seed=2, hot_period=hp); e.record(); torch.cuda.synchronize()
        rec = {"cfg": which, "hot_max": hm, "H": dp.H, "period": hp, "Mups": ep * dp.n / s.elapsed_time(e) / 1e3}
        if which == 2:
            dp.reset_state()
            its, objs, secs = dp.run_async_monitored(ep * dp.n, dp.n, gamma, seed=3, hot_period=hp)
            rel = [(o - fstar) / abs(fstar) for o in objs]
            k = next((i for i, r in enumerate(rel) if r <= 1e-6), None)
            rec["epochs_to_1e-6"] = (its[k - 1] + math.log(rel[k-1] / 1e-6) / math.log(rel[k-1] / rel[k]) * (its[k] - its[k-1])) / dp.n if k else None
            rec["final_rel"] = rel[-1]
        else:
            rec["residual"] = dp.fixed_point_residual(gamma)
        print(json.dumps(rec), flush=True)
    del dp, c
    torch.cuda.empty_cache()
