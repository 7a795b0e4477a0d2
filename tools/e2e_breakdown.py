import json, sys, time
from pathlib import Path
import numpy as np, torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems
cfg = problems.config2(seed=0)
d, loss, pen, part = cfg["data"], cfg["loss"], cfg["penalty"], cfg["partition"]
idx = pb.build_support_index(d.features, part, drop_dead_blocks=True)
for rep in range(3):
    torch.cuda.synchronize(); t = [time.perf_counter()]
    dp = pb.DeviceProblem(d, loss, pen, part, drop_dead_blocks=True); torch.cuda.synchronize(); t.append(time.perf_counter())
    gamma = pb.resolve_step_size("1/2L", dp.L, dp.n, loss.lambda1)
    f0 = dp.objective(); t.append(time.perf_counter())
    its, objs, secs = dp.run_async_checkpointed(30 * dp.n, 30 * dp.n, gamma, seed=1); t.append(time.perf_counter())
    x = dp.x(); t.append(time.perf_counter())
    tr = pb.run_async(d, loss, pen, part, pb.AsyncConfig(step_size="1/2L", epochs=30, seed=2, threads=2, checkpoint_every=30 * d.n_samples), index=idx)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    print(json.dumps({"construct_ms": 1e3*(t[1]-t[0]), "obj0_ms": 1e3*(t[2]-t[1]), "solve_ms": 1e3*(t[3]-t[2]), "x_ms": 1e3*(t[4]-t[3]), "api_total_ms": 1e3*(t[5]-t[4]), "solve_dev_s": secs}), flush=True)
# construction breakdown
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
dp = pb.DeviceProblem(d, loss, pen, part, drop_dead_blocks=True); torch.cuda.synchronize()
pr.disable(); pstats.Stats(pr).sort_stats("cumulative").print_stats(12)
