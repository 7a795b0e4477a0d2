"""Timeline of one run_async API call (config 2, pinned host data): every GPU
activity (kernels, copies, memsets) with its start/end relative to the call,
from torch.profiler (CUPTI), plus the host-side gaps between them."""
import json, sys, time
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
pd = pb.Dataset(pb.CsrMatrix(f0.n_rows, f0.n_cols, pin(f0.row_offsets), pin(f0.col_indices), pin(f0.values)),
                pin(d.labels))
idx = pb.build_support_index(d.features, part, drop_dead_blocks=True)
ac = pb.AsyncConfig(step_size="1/2L", epochs=30, seed=2, threads=2, checkpoint_every=30 * d.n_samples)
for _ in range(3):
    tr = pb.run_async(pd, loss, pen, part, ac, index=idx); _ = tr.final_x[0]
torch.cuda.synchronize()
tw = []
for _ in range(5):
    t0 = time.perf_counter(); tr = pb.run_async(pd, loss, pen, part, ac, index=idx); _ = tr.final_x[0]
    torch.cuda.synchronize(); tw.append((time.perf_counter() - t0) * 1e3)
print(json.dumps({"call_ms": [round(t, 3) for t in tw]}))
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    with torch.profiler.record_function("CALL"):
        tr = pb.run_async(pd, loss, pen, part, ac, index=idx); _ = tr.final_x[0]
        torch.cuda.synchronize()
evs = prof.events()
call = [e for e in evs if e.name == "CALL"][0]
t0 = call.time_range.start
rows = []
for e in evs:
    dev = getattr(e, "device_type", None)
    if str(dev).endswith("CUDA"):
        rows.append((e.time_range.start - t0, e.time_range.end - t0, e.name[:70]))
rows.sort()
print(f"call (host) {call.time_range.end - t0:.0f} us")
for s, en, nm in rows:
    print(f"{s:9.0f} {en:9.0f} {en - s:8.0f}  {nm}")
