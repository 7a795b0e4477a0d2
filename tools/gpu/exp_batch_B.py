"""Per-GPU lambda-path rate for the shard a rank gets at N = 1/2/4/8 GPUs
(16/N lambdas, rank 0's longest-work-first share): the lambda-batched kernel
with B = 16/N states vs concurrent forks (tools/gpu)."""
import sys, json, time
from pathlib import Path
import torch
ROOT = Path(__file__).resolve().parents[2]; sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems, lambda_path as lp
E = 30
cfg = problems.config5(seed=0)
d, part, loss = cfg["data"], cfg["partition"], cfg["loss"]
lams = lp.lambda_grid(pb.group_lambda_max(d, part), 16, 1e-3)
for world in (1, 2, 4, 8):
    mine = [lams[k] for k in lp.assign(lams, world)[0]]
    B = len(mine)
    modes = ((dict(batched=B), "batched"),) + (((dict(concurrent=B), "concurrent"),) if "--forks" in sys.argv else ())
    for kw, tag in modes:
        s = lp.device_solver(d, loss, part, epochs=E, mode="async", **kw)
        s.batch(mine); torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(); s.batch(mine); ev1.record(); torch.cuda.synchronize(); ts.append(ev0.elapsed_time(ev1))
        ms = sorted(ts)[1]
        print(json.dumps({"n_gpus": world, "lambdas_per_rank": B, "mode": tag, "ms": ms,
                          "per_gpu_Mups": B * E * d.n_samples / ms / 1e3}), flush=True)
        del s; torch.cuda.empty_cache()
