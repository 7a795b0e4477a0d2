"""Sweep warps-in-flight x contention scale on BASELINE config 2: throughput of
the async kernel and relative suboptimality after each epoch (device objective).

    python tools/sweep_async.py [--epochs 30] [--grid "ctas:wpc:c,..."]
"""

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_1707_06468_b200 as pb  # noqa: E402
from paper_1707_06468_b200 import problems  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--epochs", type=int, default=30)
    ap.add_argument("--grid", default="")
    ap.add_argument("--config", type=int, default=2)
    args = ap.parse_args()
    cfg = problems.config2(seed=0)
    data = cfg["data"]
    dp = pb.DeviceProblem(data, cfg["loss"], cfg["penalty"], cfg["partition"], drop_dead_blocks=True)
    n = data.n_samples
    gamma = pb.resolve_step_size(cfg["step"], dp.L, n, cfg["loss"].lambda1)
    fstar = json.loads((ROOT / "tests/golden/cfg2_fstar.json").read_text())["fstar"]
    grid = []
    if args.grid:
        for g in args.grid.split(","):
            f = g.split(":") + ["0", "0", "0"]
            grid.append((int(f[0]), int(f[1]), float(f[2]), int(f[3]), int(f[4])))
    else:
        for ctas, wpc in [(148, 8), (296, 8), (148, 16), (148, 32)]:
            for k in (1.0, 2.0, 4.0):
                for hp in (-1, 0, 64, 256):
                    grid.append((ctas, wpc, k, hp, 0))
    print(json.dumps({"H": dp.H, "L": dp.L}), flush=True)
    for ctas, wpc, k, hp, fl in grid:
        dp.reset_state()
        torch.cuda.synchronize()
        gaps, kms = [], 0.0
        for ep in range(args.epochs):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            dp.run_async(n, gamma, seed=11, ctas=ctas, warps_per_cta=wpc, contention=k, hot=hp >= 0,
                         hot_period=max(hp, 0), flags=fl)
            e.record()
            torch.cuda.synchronize()
            kms += s.elapsed_time(e)
            f = dp.objective()
            gaps.append((f - fstar) / abs(fstar))
            if not np.isfinite(f) or f > 100:
                break
        ups = len(gaps) * n / (kms / 1e3)
        hit = next((i + 1 for i, g in enumerate(gaps) if g <= 1e-6), None)
        print(json.dumps({"ctas": ctas, "wpc": wpc, "warps": ctas * wpc, "c": k, "hot_period": hp, "flags": fl,
                          "updates_per_s": ups,
                          "kernel_ms_total": kms, "epochs_to_1e-6": hit,
                          "gap": [float(f"{g:.3e}") for g in gaps[::max(1, len(gaps) // 10)]] + [float(f"{gaps[-1]:.3e}")]}), flush=True)


if __name__ == "__main__":
    main()
