"""Thread-per-sample kernel (PS_FLAG_LANE, lane.cuh) vs the warp kernel:
exactness at one CTA on the n=8000 instance, then config 2 (30 epochs under
the live monitor: epochs to 1e-6, final gap; one-launch updates/s) for several
warps per CTA."""
import json, math, sys
from pathlib import Path
import numpy as np, torch
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems
from paper_1707_06468_b200.saga import resolve_step_size, worker_rng
LANE = 8388608
rng = np.random.default_rng(3)
data = problems._zipf_logistic(rng, 8000, 50000, 20, 1.1, 100)
lam = 1.0 / 8000
dp = pb.DeviceProblem(data, pb.Loss("logistic", lam), pb.L1Penalty(lam), pb.singleton_partition(50000), drop_dead_blocks=True)
g = resolve_step_size("1/2L", dp.L, dp.n, lam)
dp.reset_state(); dp.replay(worker_rng(99, 0).integers(0, dp.n, size=200 * dp.n), g); fref = dp.objective()
for ctas, wpc in ((1, 4), (4, 4), (148, 4)):
    r = []
    for seed in (5, 6):
        dp.reset_state(); dp.run_async(60 * dp.n, g, seed=seed, flags=LANE, ctas=ctas, warps_per_cta=wpc)
        r.append((dp.objective() - fref) / fref)
    live = dp.abar(); dp.resync_average(); ab_err = float(np.max(np.abs(live - dp.abar())))
    print(json.dumps({"inst": "n8000", "ctas": ctas, "wpc": wpc, "rel": r, "abar_err": ab_err}), flush=True)
c = problems.config2(seed=0)
dp = pb.DeviceProblem(c["data"], c["loss"], c["penalty"], c["partition"], drop_dead_blocks=True)
fstar = json.loads((ROOT / "tests" / "golden" / "cfg2_fstar.json").read_text())["fstar"]
gamma = pb.resolve_step_size("1/2L", dp.L, dp.n, c["loss"].lambda1)
n = dp.n
for fl, wpc in ((0, 0), (LANE, 2), (LANE, 4), (LANE, 8)):
    for rep in range(2):
        dp.reset_state()
        its, objs, secs = dp.run_async_monitored(30 * n, n, gamma, seed=11 + rep, flags=fl, warps_per_cta=wpc)
        rel = [(o - fstar) / abs(fstar) for o in objs]
        hit = next((k for k, x in enumerate(rel) if x <= 1e-6), None)
        ep = None
        if hit:
            a_, b_ = rel[hit - 1], rel[hit]
            ep = (its[hit - 1] + math.log(a_ / 1e-6) / math.log(a_ / b_) * (its[hit] - its[hit - 1])) / n
        dp.reset_state()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); dp.run_async(30 * n, gamma, seed=31 + rep, flags=fl, warps_per_cta=wpc); e.record(); torch.cuda.synchronize()
        print(json.dumps({"inst": "cfg2", "flags": fl, "wpc": wpc, "epochs_to_1e-6": ep, "final_rel": rel[-1],
                          "Mups": 30 * n / s.elapsed_time(e) / 1e3, "ms": s.elapsed_time(e)}), flush=True)
