"""Can a small kernel run beside the hot solve when the solve leaves SMs free?"""
import sys, json
sys.path.insert(0, '/root/repo')
import torch, paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems
c = problems.config2(); d = c["data"]
dp = pb.DeviceProblem(d, c["loss"], c["penalty"], c["partition"], drop_dead_blocks=True)
g = pb.resolve_step_size("1/2L", dp.L, dp.n, c["loss"].lambda1)
side = torch.cuda.Stream()
buf = torch.zeros(1 << 20, device="cuda")
for ctas in (148, 140, 128):
    dp.reset_state(); torch.cuda.synchronize()
    e0, e1, s0, s1 = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    e0.record()
    dp.run_async(30 * dp.n, g, seed=1, ctas=ctas)
    e1.record()
    with torch.cuda.stream(side):
        torch.cuda._sleep(1000)
        s0.record(side); buf.add_(1.0); s1.record(side)
    torch.cuda.synchronize()
    print(json.dumps({"ctas": ctas, "solve_ms": e0.elapsed_time(e1), "side_start_ms": e0.elapsed_time(s0), "side_end_ms": e0.elapsed_time(s1)}))
