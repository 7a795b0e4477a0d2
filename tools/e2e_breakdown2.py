"""Where the time of one run_async API call goes (config 2, pinned host data)."""
import json, sys, time
from pathlib import Path
import numpy as np, torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems, device
cfg = problems.config2(seed=0)
d, loss, pen, part = cfg["data"], cfg["loss"], cfg["penalty"], cfg["partition"]
keep = []
def pin(a):
    t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory(); keep.append(t); return t.numpy()
f0 = d.features
pd = pb.Dataset(pb.CsrMatrix(f0.n_rows, f0.n_cols, pin(f0.row_offsets), pin(f0.col_indices), pin(f0.values)), pin(d.labels))
idx = pb.build_support_index(d.features, part, drop_dead_blocks=True)
T = {}
def wrap(obj, name):
    fn = getattr(obj, name)
    def w(*a, **k):
        torch.cuda.synchronize(); t = time.perf_counter(); r = fn(*a, **k); torch.cuda.synchronize()
        T[name] = T.get(name, 0.0) + (time.perf_counter() - t) * 1e3; return r
    setattr(obj, name, w)
for nm in ("__init__", "_hot_layout", "_setup_partition", "run_async_monitored", "run_async_checkpointed", "objective", "objective_parts", "x", "reset_state", "launch_config"):
    wrap(device.DeviceProblem, nm)
for rep in range(4):
    T.clear()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    tr = pb.run_async(pd, loss, pen, part, pb.AsyncConfig(step_size="1/2L", epochs=30, seed=2, threads=2, checkpoint_every=30 * d.n_samples), index=idx)
    _ = tr.final_x[0]; torch.cuda.synchronize()
    tot = (time.perf_counter() - t0) * 1e3
    print(json.dumps({"total_ms": round(tot, 3), **{k: round(v, 3) for k, v in T.items()}}), flush=True)
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
tr = pb.run_async(pd, loss, pen, part, pb.AsyncConfig(step_size="1/2L", epochs=30, seed=2, threads=2, checkpoint_every=30 * d.n_samples), index=idx)
torch.cuda.synchronize(); pr.disable(); pstats.Stats(pr).sort_stats("tottime").print_stats(14)
