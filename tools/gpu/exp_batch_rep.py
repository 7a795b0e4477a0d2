"""lambda-batched kernel with replicated x-delta accumulators for the hottest
blocks (ps_batch_run_rep): rows/s of one config-5 epoch per B and replica
count, and the 30-epoch certified gaps of B = 2 / 16 with and without them."""
import sys, json
from pathlib import Path
import torch
ROOT = Path(__file__).resolve().parents[2]; sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems, lambda_path as lp
cfg = problems.config5(seed=0)
d, part, loss = cfg["data"], cfg["partition"], cfg["loss"]
lams = lp.lambda_grid(pb.group_lambda_max(d, part), 16, 1e-3)
reps = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "0,2,4,8").split(",")]
nrbs = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "32").split(",")]
for B in (16, 8, 4, 2):
    for nrep in reps:
        for nrb in (nrbs if nrep else [0]):
            bp = lp.BatchedPath(d, loss, part, B=B, nrep=nrep, nrb=nrb)
            gamma = pb.resolve_step_size("1/2L", bp.dp.L, d.n_samples, loss.lambda1)
            bp.reset(lams[:B]); bp.run(d.n_samples, gamma, seed=1); torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); bp.run(d.n_samples, gamma, seed=2); e.record(); torch.cuda.synchronize()
            ms = s.elapsed_time(e)
            out = {"B": B, "nrep": nrep, "nrb": bp.nrb, "ms_epoch": ms, "Mrows": d.n_samples / ms / 1e3,
                   "Mlam_updates": B * d.n_samples / ms / 1e3}
            if B in (2, 16):
                bp.reset(lams[:B]); bp.run(30 * d.n_samples, gamma, seed=3); torch.cuda.synchronize()
                out["rel_gap30"] = [float(f"{bp.summary(b, 0)['gap'] / abs(bp.summary(b, 0)['objective']):.2e}") for b in range(B)]
            print(json.dumps(out), flush=True)
            del bp; torch.cuda.empty_cache()
