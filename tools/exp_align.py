"""Fast-kernel time vs the byte offset of the coordinate records (config 2):
the hot records are 1 KiB apart, so their L2 slices depend on the base."""
import json, sys
from pathlib import Path
import torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems

cfg = problems.config2(seed=0)
strides = [int(v) for v in sys.argv[1].split(",")] if len(sys.argv) > 1 else [32]
offsets = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else \
    [0, 64, 128, 256, 512, 1024, 2048, 4096, 8192, 16384, 65536, 262144]
out = {}
for stride in strides:
  dp = pb.DeviceProblem(cfg["data"], cfg["loss"], cfg["penalty"], cfg["partition"], drop_dead_blocks=True,
                        hot_stride=stride)
  gamma = pb.resolve_step_size("1/2L", dp.L, dp.n, cfg["loss"].lambda1)
  orig = dp.coord.clone()
  big = torch.zeros(4 * dp.p_dev + (1 << 21), dtype=torch.float64, device="cuda")
  base = big.data_ptr()
  al = (-(base) % (1 << 21)) // 8  # doubles to a 2 MiB boundary
  res = {}
  dp.run_async(3 * dp.n, gamma, seed=1)  # warm-up
  for rep in range(2):
    for off in offsets:
        o = al + off // 8
        view = big[o:o + 4 * dp.p_dev].view(dp.p_dev, 4)
        view.copy_(orig)
        dp.coord = view
        dp.reset_state()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); dp.run_async(30 * dp.n, gamma, seed=5); e.record(); torch.cuda.synchronize()
        res.setdefault(off, []).append(round(s.elapsed_time(e), 3))
  out[f"stride{stride}_ms_by_offset_bytes"] = res
  del dp, big
print(json.dumps(out), flush=True)
