"""lambda-batched kernel: scattered hot blocks (ps_batch_tune2) -- the nhot
most frequent blocks keep one sector per hstride doubles in each region's pad.
Rows/s of one config-5 epoch (after two warm epochs) per (B, nhot, hstride);
the 3-epoch objectives of state 0 and B-1 as a sanity check.
    python tools/gpu/exp_batch_scatter.py "B:nhot:hstride[:nrep[:nrb[:hshare[:hab]]]],..." """
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
def rate(B, nhot, hstride, nrep=None, nrb=None, hshare=4, hab=-1, reps=3):
    global dp
    L = _lib.load()
    _lib.check(L.ps_batch_tune2(nhot, hstride, hshare, hab))
    bp = lp.BatchedPath(d, loss, part, B=B, dp=dp, nrep=nrep, nrb=nrb)
    dp = bp.dp
    gamma = pb.resolve_step_size("1/2L", bp.dp.L, d.n_samples, loss.lambda1)
    # the B smallest lambdas (every block alive: the most REDs)
    bp.reset(lams[16 - B:]); bp.run(2 * d.n_samples, gamma, seed=1); torch.cuda.synchronize()
    ms = []
    for r in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); bp.run(d.n_samples, gamma, seed=2 + r); e.record(); torch.cuda.synchronize(); ms.append(s.elapsed_time(e))
    objs = [bp.summary(b, 0)["objective"] for b in (0, B - 1)]
    print(json.dumps({"B": B, "nhot": nhot, "hstride": hstride, "nrep": bp.nrep, "nrb": bp.nrb, "hshare": hshare, "hab": hab, "ms": round(min(ms), 3),
                      "Mrows": round(d.n_samples / min(ms) / 1e3, 2), "obj": objs}), flush=True)
    del bp; torch.cuda.empty_cache()
for v in sys.argv[1].split(","):
    f = [int(t) for t in v.split(":")]
    rate(f[0], f[1], f[2], nrep=(f[3] if len(f) > 3 else None), nrb=(f[4] if len(f) > 4 else None), hshare=(f[5] if len(f) > 5 else 4), hab=(f[6] if len(f) > 6 else -1))
