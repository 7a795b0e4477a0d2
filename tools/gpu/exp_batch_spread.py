"""lambda-batched kernel on config 5: natural block order vs the spread hot-unit
layout (BatchedPath(spread=...)), rows/s of one epoch for several B, and the
30-epoch objectives of both layouts for B=16."""
import sys, json
from pathlib import Path
import torch
ROOT = Path(__file__).resolve().parents[2]; sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems, lambda_path as lp
cfg = problems.config5(seed=0)
d, part, loss = cfg["data"], cfg["partition"], cfg["loss"]
lams = lp.lambda_grid(pb.group_lambda_max(d, part), 16, 1e-3)
for spread in (False, True):
    for B in (16, 8, 2):
        bp = lp.BatchedPath(d, loss, part, B=B, spread=spread)
        gamma = pb.resolve_step_size("1/2L", bp.dp.L, d.n_samples, loss.lambda1)
        bp.reset(lams[:B]); bp.run(d.n_samples, gamma, seed=1); torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); bp.run(d.n_samples, gamma, seed=2); e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e)
        out = {"spread": spread, "B": B, "ms_epoch": ms, "Mrows": d.n_samples / ms / 1e3, "Mlam_updates": B * d.n_samples / ms / 1e3}
        if B == 16:
            bp.reset(lams); bp.run(30 * d.n_samples, gamma, seed=3); torch.cuda.synchronize()
            out["obj30"] = [round(bp.summary(b, 0)["objective"], 10) for b in (0, 8, 15)]
            out["gap30"] = [bp.summary(b, 0)["gap"] for b in (0, 8, 15)]
        print(json.dumps(out), flush=True)
        del bp; torch.cuda.empty_cache()
