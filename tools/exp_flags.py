"""A/B of kernel variants selected by ps_sched_t.flags values:
config 2 -- 30-epoch solve under the live monitor: epochs and time to a 1e-6
relative gap, final gap, updates/s; configs 3/4 -- per-epoch time early/late
and the final fixed-point residual of a long run.
    python tools/exp_flags.py 2|3|4 epochs flag[,flag...]"""
import json, math, sys
from pathlib import Path
import torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems

which = int(sys.argv[1])
epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 30
FLAGS = [int(v) for v in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0]
if which == 2:
    c = problems.config2(seed=0)
    dp = pb.DeviceProblem(c["data"], c["loss"], c["penalty"], c["partition"], drop_dead_blocks=True)
    fstar = json.loads((ROOT / "tests" / "golden" / "cfg2_fstar.json").read_text())["fstar"]
    step = "1/2L"
else:
    c = problems.config3() if which == 3 else problems.config4()
    dp = c["problem"]
    fstar = None
    step = c["step"]
gamma = pb.resolve_step_size(step, dp.L, dp.n, c["loss"].lambda1)
out = {}
for rep in range(2):
    for fl in FLAGS:
        zm = fl

        dp.reset_state()
        if which == 2:
            its, objs, secs = dp.run_async_monitored(epochs * dp.n, dp.n, gamma, seed=11 + rep, flags=fl)
            rel = [(o - fstar) / abs(fstar) for o in objs]
            hit = next((k for k, r in enumerate(rel) if r <= 1e-6), None)
            ep = None
            if hit:
                a, b = rel[hit - 1], rel[hit]
                fr = math.log(a / 1e-6) / math.log(a / b)
                ep = (its[hit - 1] + fr * (its[hit] - its[hit - 1])) / dp.n
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            dp.reset_state()
            s.record(); dp.run_async(epochs * dp.n, gamma, seed=31 + rep, flags=fl); e.record(); torch.cuda.synchronize()
            out.setdefault(zm, []).append({"epochs_to_1e-6": ep, "final_rel": rel[-1],
                                           "Mups": epochs * dp.n / s.elapsed_time(e) / 1e3})
        else:
            its, objs, secs = dp.run_async_checkpointed(epochs * dp.n, dp.n, gamma, seed=11 + rep, flags=fl)
            res = dp.fixed_point_residual(gamma)
            k = max(1, epochs // 4)
            out.setdefault(zm, []).append({"ms_epoch_first": 1e3 * (secs[k] - secs[0]) / k,
                                           "ms_epoch_last": 1e3 * (secs[-1] - secs[-1 - k]) / k,
                                           "obj_end": objs[-1], "residual_end": res})
print(json.dumps({"cfg": which, "res": out}), flush=True)
