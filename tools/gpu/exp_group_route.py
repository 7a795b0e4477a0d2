"""run_async for group lasso: the lambda-batched kernel with one state against the
coordinate-record group kernel (AsyncConfig.group_batched), wall seconds per epoch
on config 5's instance (n = 1e5, p = 1e7) and on smaller ones."""
import sys, json, time
from pathlib import Path
import numpy as np, torch
ROOT = Path(__file__).resolve().parents[2]; sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems

def run(data, part, loss, lam, epochs, tag):
    idx = pb.build_support_index(data.features, part, drop_dead_blocks=True)
    out = {"case": tag}
    for gb in (True, False):
        cfg = pb.AsyncConfig(step_size="1/2L", epochs=epochs, seed=2, threads=2, group_batched=gb)
        pb.run_async(data, loss, pb.GroupL2Penalty(lam), part, cfg, index=idx)  # warm
        t0 = time.perf_counter(); tr = pb.run_async(data, loss, pb.GroupL2Penalty(lam), part, cfg, index=idx); torch.cuda.synchronize()
        out["batched" if gb else "group_kernel"] = {"call_s": round(time.perf_counter() - t0, 5),
            "s_per_epoch": round((tr.wall_seconds[-1] - tr.wall_seconds[1]) / (epochs - 1), 6), "obj": tr.objective[-1]}
    print(json.dumps(out), flush=True)

cfg5 = problems.config5(seed=0)
d, part, loss = cfg5["data"], cfg5["partition"], cfg5["loss"]
lmax = pb.group_lambda_max(d, part)
run(d, part, loss, 0.1 * lmax, 20, "config5 0.1 lmax")
run(d, part, loss, 0.003 * lmax, 20, "config5 0.003 lmax")
for n, p in ((8000, 40000), (30000, 200000)):
    rng = np.random.default_rng(11)
    dd = problems._zipf_logistic(rng, n, p, 20, 1.1, 100)
    pp = pb.contiguous_partition(p, 10)
    ll = pb.Loss("logistic", 1.0 / n)
    run(dd, pp, ll, 0.1 * pb.group_lambda_max(dd, pp), 20, f"n={n} p={p}")
