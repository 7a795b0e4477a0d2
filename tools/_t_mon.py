import sys, json
sys.path.insert(0, "/root/repo")
import torch, paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems
cfg = problems.config2(seed=0)
dp = pb.DeviceProblem(cfg["data"], cfg["loss"], cfg["penalty"], cfg["partition"], drop_dead_blocks=True)
n = dp.n; gamma = pb.resolve_step_size("1/2L", dp.L, n, cfg["loss"].lambda1)
fstar = json.load(open("/root/repo/tests/golden/cfg2_fstar.json"))["fstar"]
for rep in range(3):
    dp.reset_state()
    its, objs, secs = dp.run_async_monitored(30 * n, n, gamma, seed=7 + rep)
    rel = [(o - fstar) / fstar for o in objs]
    hit = next((i for i, r in enumerate(rel) if r <= 1e-6), None)
    print(json.dumps({"n_ckpt": len(its), "its_k": [round(i / n, 2) for i in its[:14]], "hit": hit,
                      "t_hit_ms": secs[hit] * 1e3 if hit is not None else None, "ep_hit": its[hit] / n if hit is not None else None,
                      "t_total_ms": secs[-1] * 1e3, "final_rel": rel[-1]}), flush=True)
dp.reset_state()
its, objs, secs = dp.run_async_checkpointed(30 * n, n, gamma, seed=7, graph=True)
rel = [(o - fstar) / fstar for o in objs]; hit = next((i for i, r in enumerate(rel) if r <= 1e-6), None)
print(json.dumps({"graph": True, "t_hit_ms": secs[hit] * 1e3, "ep": its[hit] / n}))
