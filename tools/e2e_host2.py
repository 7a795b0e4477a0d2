"""Host-side cost of the pieces of one run_async call (config 2, pinned data), cProfile cumulative."""
import sys, time, cProfile, pstats, io
from pathlib import Path
import numpy as np, torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems
cfg = problems.config2(seed=0)
d, loss, pen, part = cfg["data"], cfg["loss"], cfg["penalty"], cfg["partition"]
keep = []
def pin(a):
    t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory(); keep.append(t); return t.numpy()
f0 = d.features
pd = pb.Dataset(pb.CsrMatrix(f0.n_rows, f0.n_cols, pin(f0.row_offsets), pin(f0.col_indices), pin(f0.values)), pin(d.labels))
idx = pb.build_support_index(d.features, part, drop_dead_blocks=True)
ac = pb.AsyncConfig(step_size="1/2L", epochs=30, seed=2, threads=2, checkpoint_every=30 * d.n_samples)
for _ in range(3):
    tr = pb.run_async(pd, loss, pen, part, ac, index=idx); _ = tr.final_x[0]
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(5):
    tr = pb.run_async(pd, loss, pen, part, ac, index=idx); _ = tr.final_x[0]
torch.cuda.synchronize(); pr.disable()
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(40); print(s.getvalue()[:6000])
