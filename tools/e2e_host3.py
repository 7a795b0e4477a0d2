"""Where the host time of one run_async call goes (config 2, pinned data):
perf_counter stamps around the call's steps, no synchronisation added."""
import sys, time, json
from pathlib import Path
import numpy as np, torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems, device, saga, asynchronous, _lib
cfg = problems.config2(seed=0)
d, loss, pen, part = cfg["data"], cfg["loss"], cfg["penalty"], cfg["partition"]
keep = []
def pin(a):
    t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory(); keep.append(t); return t.numpy()
f0 = d.features
pd = pb.Dataset(pb.CsrMatrix(f0.n_rows, f0.n_cols, pin(f0.row_offsets), pin(f0.col_indices), pin(f0.values)), pin(d.labels))
idx = pb.build_support_index(d.features, part, drop_dead_blocks=True)
ac = pb.AsyncConfig(step_size="1/2L", epochs=30, seed=2, threads=2, checkpoint_every=30 * d.n_samples)
T = []
def stamp(tag): T.append((tag, time.perf_counter()))
def wrap(obj, name):
    fn = getattr(obj, name)
    def w(*a, **k):
        stamp(name + ">"); r = fn(*a, **k); stamp(name + "<"); return r
    setattr(obj, name, w)
for nm in ("__init__", "_hot_layout", "_setup_partition", "run_async_monitored", "launch_config", "_scratch_for", "x", "objective", "_sched", "params"):
    wrap(device.DeviceProblem, nm)
L = _lib.load()
for nm in ("ps_prepare", "ps_run_monitored", "ps_objective", "ps_hot_layout", "ps_launch_config"):
    f = getattr(L, nm)
    def mk(f, nm):
        def w(*a):
            stamp(nm + ">"); r = f(*a); stamp(nm + "<"); return r
        return w
    setattr(L, nm, mk(f, nm))
for _ in range(3):
    tr = pb.run_async(pd, loss, pen, part, ac, index=idx); _ = tr.final_x[0]
torch.cuda.synchronize()
for rep in range(2):
    T.clear(); torch.cuda.synchronize(); t0 = time.perf_counter()
    tr = pb.run_async(pd, loss, pen, part, ac, index=idx); _ = tr.final_x[0]
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"total {1e3 * (t1 - t0):.3f} ms")
    prev = t0
    for tag, t in T:
        print(f"  {1e6 * (t - t0):8.1f} us (+{1e6 * (t - prev):7.1f})  {tag}")
        prev = t
    print(f"  {1e6 * (t1 - t0):8.1f} us (+{1e6 * (t1 - prev):7.1f})  end")
