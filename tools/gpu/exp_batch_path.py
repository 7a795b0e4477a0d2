"""Config 5 lambda path: concurrent forks (lane kernel) vs the lambda-batched
kernel, 16 lambdas x E epochs on one GPU: updates/s (lambda-updates) and the
per-lambda certified relative gaps (tools/gpu)."""
import sys, json, time
from pathlib import Path
import numpy as np, torch
ROOT = Path(__file__).resolve().parents[2]; sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems, lambda_path as lp
E = int(sys.argv[1]) if len(sys.argv) > 1 else 30
cfg = problems.config5(seed=0)
d, part, loss = cfg["data"], cfg["partition"], cfg["loss"]
lams = lp.lambda_grid(pb.group_lambda_max(d, part), 16, 1e-3)
upd = 16 * E * d.n_samples
def timed(solve, tag):
    solve.batch(lams)  # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter(); res = solve.batch(lams); torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(json.dumps({"mode": tag, "s": dt, "Mups": upd / dt / 1e6,
                      "rel_gap": [float(f"{r['gap'] / abs(r['objective']):.2e}") for r in res],
                      "obj": [round(r["objective"], 8) for r in res]}), flush=True)
for kw, tag in [(dict(batched=16), "batched16"), (dict(batched=16, warps_per_cta=8), "batched16_w8"),
                (dict(batched=8), "batched8"), (dict(concurrent=16), "concurrent16")]:
    s = lp.device_solver(d, loss, part, epochs=E, mode="async", **kw)
    timed(s, tag)
    del s
    torch.cuda.empty_cache()
