"""The reference's literal ProxASAGA (contention 0 = plain gamma, delta commits
PS_FLAG_DELTA_ZERO) vs warps in flight on the test instance of
tests/test_gpu_fast.py: relative gap after 60 epochs (tools/gpu)."""
import sys, json
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[2]; sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems
from paper_1707_06468_b200.device import DeviceProblem
rng = np.random.default_rng(3)
data = problems._zipf_logistic(rng, 8000, 50000, 20, 1.1, 100)
lam = 1.0 / data.n_samples
dp = DeviceProblem(data, pb.Loss("logistic", lam), pb.L1Penalty(lam), pb.singleton_partition(data.n_features),
                   drop_dead_blocks=True)
gamma = pb.resolve_step_size("1/2L", dp.L, dp.n, lam)
dp.replay(pb.worker_rng(99, 0).integers(0, dp.n, size=200 * dp.n), gamma)
fref = dp.objective()
for ctas, wpc, hot in [(8, 1, False), (16, 1, False), (37, 1, False), (74, 1, False), (148, 1, False),
                       (148, 2, False), (148, 4, False), (148, 8, False), (0, 0, False), (0, 0, True)]:
    out = {}
    for name, kw in (("literal", dict(contention=0.0, flags=32)), ("default", dict())):
        dp.reset_state()
        dp.run_async(60 * dp.n, gamma, seed=7, ctas=ctas, warps_per_cta=wpc, hot=hot, **kw)
        out[name] = (dp.objective() - fref) / abs(fref)
    print(json.dumps({"ctas": ctas, "wpc": wpc, "hot": hot, "launch": dp.launch_config(dp._sched(dp.n, ctas=ctas, warps_per_cta=wpc))[:2], **out}), flush=True)
