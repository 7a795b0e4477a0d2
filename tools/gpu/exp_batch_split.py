"""Config 5 at one GPU: the 16 lambdas as one B=16 launch vs two concurrent
B=8 launches (two streams, one shared DeviceProblem) vs four B=4 launches;
one epoch of rows per state."""
import sys, json
from pathlib import Path
import torch
ROOT = Path(__file__).resolve().parents[2]; sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems, lambda_path as lp
cfg = problems.config5(seed=0)
d, part, loss = cfg["data"], cfg["partition"], cfg["loss"]
lams = lp.lambda_grid(pb.group_lambda_max(d, part), 16, 1e-3)
base = lp.BatchedPath(d, loss, part, B=16)
dp = base.dp
gamma = pb.resolve_step_size("1/2L", dp.L, d.n_samples, loss.lambda1)
for B, ctas_div in ((16, 1), (8, 2), (4, 4), (8, 1), (4, 1)):
    k = 16 // B
    bps = [base] if B == 16 else [lp.BatchedPath(d, loss, part, B=B, dp=dp) for _ in range(k)]
    sts = [torch.cuda.Stream() for _ in range(k)]
    ctas = 0 if ctas_div == 1 else 148 // ctas_div
    def go(seed):
        for j, (bp, st) in enumerate(zip(bps, sts)):
            bp.reset(lams[j * B:(j + 1) * B]) if seed == 1 else None
            bp.run(d.n_samples, gamma, seed=seed, stream=st, ctas=ctas)
    torch.cuda.synchronize(); go(1); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); go(2); torch.cuda.synchronize(); e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    print(json.dumps({"B": B, "launches": k, "ctas_each": ctas, "ms": ms, "Mlam_updates": 16 * d.n_samples / ms / 1e3}), flush=True)
