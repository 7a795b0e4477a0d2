"""Time to a 1e-6 relative gap vs the hot kernel's flush period (512 staged
columns): configs 3/4 stop-the-world per-epoch checkpoints against a long-run
F*, config 2 the live monitor against tests/golden/cfg2_fstar.json (tools/gpu).
    python tools/gpu/exp_period_ttt.py 2|3|4"""
import sys, json, math
from pathlib import Path
import torch
ROOT = Path(__file__).resolve().parents[2]; sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems


def cross(its, secs, rel, n):
    prev = (1.0, 0.0, 0)
    for it, s, r in zip(its, secs, rel):
        if r <= 1e-6:
            a = prev[0]
            fr = math.log(a / 1e-6) / math.log(a / r) if a > r else 1.0
            return prev[1] + fr * (s - prev[1]), (prev[2] + fr * (it - prev[2])) / n
        prev = (r, s, it)
    return None, None


which = int(sys.argv[1])
if which == 2:
    c = problems.config2(seed=0)
    dp = pb.DeviceProblem(c["data"], c["loss"], c["penalty"], c["partition"], drop_dead_blocks=True, hot_max=512)
    fstar = json.loads((ROOT / "tests" / "golden" / "cfg2_fstar.json").read_text())["fstar"]
    ep = 30
else:
    c = problems.config3(hot_max=512) if which == 3 else problems.config4(hot_max=512)
    dp = c["problem"]
    ep = 20
gamma = pb.resolve_step_size("1/2L", dp.L, dp.n, c["loss"].lambda1)
if which != 2:
    dp.reset_state(); dp.run_async((60 if which == 3 else 40) * dp.n, gamma, seed=7)
    fstar = dp.objective()
for hp in (24, 28, 32):
    for rep in range(3 if which == 2 else 2):
        dp.reset_state()
        if which == 2:
            its, objs, secs = dp.run_async_monitored(ep * dp.n, dp.n, gamma, seed=11 + rep, hot_period=hp)
            its, objs, secs = its[1:], objs[1:], secs[1:]
        else:
            its, objs, secs = dp.run_async_checkpointed(ep * dp.n, dp.n, gamma, seed=11 + rep, graph=True, hot_period=hp)
        rel = [max((o - fstar) / abs(fstar), 1e-300) for o in objs]
        s, e = cross(its, secs, rel, dp.n)
        dp.reset_state()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(); dp.run_async((ep if which == 2 else 5) * dp.n, gamma, seed=21, hot_period=hp); t1.record(); torch.cuda.synchronize()
        print(json.dumps({"cfg": which, "period": hp, "seconds_to_1e-6": s, "epochs_to_1e-6": e, "final_rel": rel[-1],
                          "Mups": (ep if which == 2 else 5) * dp.n / t0.elapsed_time(t1) / 1e3}), flush=True)
