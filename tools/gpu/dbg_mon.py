import sys, json
sys.path.insert(0, '/root/repo')
import torch, paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems, _lib
c = problems.config2(); d = c["data"]
dp = pb.DeviceProblem(d, c["loss"], c["penalty"], c["partition"], drop_dead_blocks=True)
g = pb.resolve_step_size("1/2L", dp.L, dp.n, c["loss"].lambda1)
for dev, fl in ((True, 0), (True, _lib.FLAG_NO_CLUSTER), (False, 0)):
    for rep in range(2):
        dp.reset_state()
        its, objs, secs = dp.run_async_monitored(30 * dp.n, dp.n, g, seed=3, device_snaps=dev, flags=fl)
        print(json.dumps({"dev": dev, "flags": fl, "n": len(its), "its": [round(i / dp.n, 2) for i in its][:8], "secs_ms": [round(s * 1e3, 3) for s in secs][:8]}))
