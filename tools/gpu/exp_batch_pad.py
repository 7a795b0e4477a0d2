"""lambda-batched kernel: L2-slice placement knobs (ps_batch_tune) -- the
state's region pad (B = 16) and the replica chunk stride (B = 2, 4), rows/s of
one config-5 epoch."""
import sys, json
from pathlib import Path
import torch
ROOT = Path(__file__).resolve().parents[2]; sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems, lambda_path as lp, _lib
cfg = problems.config5(seed=0)
d, part, loss = cfg["data"], cfg["partition"], cfg["loss"]
lams = lp.lambda_grid(pb.group_lambda_max(d, part), 16, 1e-3)
dp = None
def rate(B, rpad, rstride, reps=2):
    global dp
    _lib.check(_lib.load().ps_batch_tune(rpad, rstride))
    bp = lp.BatchedPath(d, loss, part, B=B, dp=dp)
    dp = bp.dp
    gamma = pb.resolve_step_size("1/2L", bp.dp.L, d.n_samples, loss.lambda1)
    bp.reset(lams[:B]); bp.run(d.n_samples, gamma, seed=1); torch.cuda.synchronize()
    ms = []
    for r in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); bp.run(d.n_samples, gamma, seed=2 + r); e.record(); torch.cuda.synchronize(); ms.append(s.elapsed_time(e))
    print(json.dumps({"B": B, "rpad": rpad, "rstride": rstride, "nrep": bp.nrep, "ms": min(ms), "Mrows": d.n_samples / min(ms) / 1e3}), flush=True)
    del bp; torch.cuda.empty_cache()
for rpad in (0, 128, 160, 544, 1056, 4256, 65568):
    rate(16, rpad, 0)
for B in (2, 4, 8):
    for rs in (0, 128, 136, 256, 520):
        rate(B, 0, rs)
