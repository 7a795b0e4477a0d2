"""One lambda-batched launch (B states, default 16; config 5, one epoch of rows) for ncu (tools/gpu).
    python tools/gpu/prof_batch.py [warps_per_cta] [B]"""
import sys, json
from pathlib import Path
import torch
ROOT = Path(__file__).resolve().parents[2]; sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems, lambda_path as lp
cfg = problems.config5(seed=0)
d, part, loss = cfg["data"], cfg["partition"], cfg["loss"]
lams = lp.lambda_grid(pb.group_lambda_max(d, part), 16, 1e-3)
B = int(sys.argv[2]) if len(sys.argv) > 2 else 16
bp = lp.BatchedPath(d, loss, part, B=B)
gamma = pb.resolve_step_size("1/2L", bp.dp.L, d.n_samples, loss.lambda1)
wpc = int(sys.argv[1]) if len(sys.argv) > 1 else 0
bp.reset(lams[:B])
bp.run(d.n_samples, gamma, seed=1, warps_per_cta=wpc)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); bp.run(d.n_samples, gamma, seed=2, warps_per_cta=wpc); e.record(); torch.cuda.synchronize()
print(json.dumps({"ms": s.elapsed_time(e), "Mrows": d.n_samples / s.elapsed_time(e) / 1e3}))
