"""Run the async kernel on config 2 for profiling: warm-up epochs then a few
profiled epochs with a fixed launch configuration.
    python tools/prof_async.py --ctas 148 --wpc 32 --hp 8 --c 4 [--nohot] [--epochs 3]"""
import argparse, json, sys
from pathlib import Path
import torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems

ap = argparse.ArgumentParser()
ap.add_argument("--ctas", type=int, default=148)
ap.add_argument("--wpc", type=int, default=32)
ap.add_argument("--hp", type=int, default=8)
ap.add_argument("--c", type=float, default=4.0)
ap.add_argument("--nohot", action="store_true")
ap.add_argument("--epochs", type=int, default=3)
ap.add_argument("--warm", type=int, default=2)
ap.add_argument("--batch", type=int, default=32)
ap.add_argument("--per_launch", type=int, default=1)
ap.add_argument("--grid", default="")
ap.add_argument("--flags", type=int, default=0)
ap.add_argument("--hot_max", type=int, default=256)
a = ap.parse_args()
cfg = problems.config2(seed=0)
_dps = {}
def get_dp(hm):
    if hm not in _dps:
        _dps.clear()
        _dps[hm] = pb.DeviceProblem(cfg["data"], cfg["loss"], cfg["penalty"], cfg["partition"], drop_dead_blocks=True, hot_max=hm)
    return _dps[hm]
dp = get_dp(a.hot_max)
gamma = pb.resolve_step_size("1/2L", dp.L, dp.n, cfg["loss"].lambda1)
def one(a):
    dp = get_dp(a.hot_max)
    kw = dict(ctas=a.ctas, warps_per_cta=a.wpc, contention=a.c, hot=not a.nohot, hot_period=a.hp, batch=a.batch, flags=a.flags)
    dp.reset_state()
    for _ in range(a.warm):
        dp.run_async(dp.n * a.per_launch, gamma, seed=1, **kw)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(a.epochs):
        dp.run_async(dp.n * a.per_launch, gamma, seed=2, **kw)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    print(json.dumps({"cfg": {k: v for k, v in vars(a).items() if k != "grid"}, "H": dp.H, "ms": ms,
                      "Mups": a.epochs * a.per_launch * dp.n / ms / 1e3}), flush=True)

if a.grid:
    import copy
    for g in a.grid.split(","):
        b = copy.copy(a)
        for kv in g.split(";"):
            k, v = kv.split("=")
            setattr(b, k, type(getattr(a, k))(v) if not isinstance(getattr(a, k), bool) else v == "1")
        one(b)
else:
    one(a)
