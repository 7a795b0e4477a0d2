"""Configs 3/4: the local-view flag (bit 27) against the default, per
(flags : period : c) variant -- per-epoch objectives of a stop-the-world run,
ms per epoch, final duality gap and fixed-point residual.
    python tools/gpu/exp_big_lv.py 3|4 epochs "flags:hp:c,..." """
import json, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems

which, epochs = int(sys.argv[1]), int(sys.argv[2])
c = problems.config3() if which == 3 else problems.config4()
dp = c["problem"]
gamma = pb.resolve_step_size(c["step"], dp.L, dp.n, c["loss"].lambda1)
dp.run_async(dp.n // 10, gamma, seed=1)
for v in sys.argv[3].split(","):
    fl, hp, cc = v.split(":")
    dp.reset_state()
    its, objs, secs = dp.run_async_checkpointed(epochs * dp.n, dp.n, gamma, seed=3, hot_period=int(hp),
                                                contention=float(cc), flags=int(fl))
    res = dp.fixed_point_residual(gamma)
    f, dual, gap = dp.duality_gap()
    print(json.dumps({"cfg": which, "H": dp.H, "variant": v, "ms_epoch": round(1e3 * (secs[-1] - secs[0]) / epochs, 3),
                      "obj": [round(o, 13) for o in objs[::2]], "gap_end": gap, "rel_gap_end": gap / abs(f),
                      "residual_end": res}), flush=True)
