"""F* for BASELINE config 2 from the C oracle (pinned to the reference by
tests/test_oracle.py and by ref_large.npz's 30-epoch reference run).

Protocol of diagnostics.py:153-200 (reference_optimum): sequential SPS from
zero with growing epoch budgets until the fixed-point residual (saga.py:299-317)
is <= 1e-9; writes tests/golden/cfg2_fstar.json.
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402
from paper_1707_06468_b200 import problems  # noqa: E402


def main():
    c = problems.config2(seed=0)
    P = O.from_dataset(c["data"], c["loss"], c["penalty"], c["partition"])
    gamma = 1.0 / (2.0 * P.lipschitz())
    n = P.n
    x = a = ab = None
    epochs, t0 = 0, time.time()
    seq_seed = 9999
    res = np.inf
    while res > 1e-9 and epochs < 1000:
        chunk = 50
        seq = O.sample_sequence(seq_seed, n, chunk * n, worker_id=epochs)
        x, a, ab = P.run_sequential(gamma, seq, x, a, ab)
        epochs += chunk
        res = P.fixed_point_residual(x, gamma)
        print(f"epochs {epochs}: F={P.objective(x):.15f} residual={res:.3e} ({time.time() - t0:.0f}s)", flush=True)
    out = {"config": "cfg2 seed 0", "fstar": P.objective(x), "residual": res, "epochs": epochs,
           "gamma": gamma, "nnz_x": int(np.count_nonzero(x)), "source": "oracle sequential SPS (C), 1/2L"}
    (Path(__file__).resolve().parent / "cfg2_fstar.json").write_text(json.dumps(out, indent=1) + "\n")
    print(out)


if __name__ == "__main__":
    main()
