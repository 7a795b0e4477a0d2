"""FISTA goldens from the UNMODIFIED reference (build container only).

    python tests/golden/make_fista.py

Runs the reference's run_fista (fista.py:61-111: backtracking from L/100,
x0 = 0, deterministic) on small seeded cases and records the objective
trace, the curvature estimates and the final iterate into
tests/golden/ref_fista.npz, for tests/test_gpu_fista.py.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import ref_loader  # noqa: E402
from tests.golden import cases  # noqa: E402
from tests.golden.make_golden import data_hash, to_ref  # noqa: E402

OUT = Path(__file__).resolve().parent / "ref_fista.npz"
CASES = {"acc_l1": 300, "grp_contig": 300, "box_sq": 200, "cfg1": 200, "grp_random": 200}


def main():
    sg = ref_loader.load()
    small = cases.small_cases()
    out = {}
    for name, iters in CASES.items():
        case = small[name]
        data, loss, pen, part = to_ref(sg, case)
        tr = sg.run_fista(data, loss, pen, part, max_iters=iters)
        out[f"{name}__obj"] = np.array(tr.objective)
        out[f"{name}__x"] = np.asarray(tr.final_x)
        out[f"{name}__iters"] = np.array(iters)
        out[f"{name}__hash"] = np.array(data_hash(data.features, data.labels))
        print(f"  {name}: {iters} iterations, F={tr.objective[-1]:.15g}", flush=True)
    np.savez_compressed(OUT, **out)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
