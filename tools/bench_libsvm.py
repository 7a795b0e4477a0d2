"""LibSVM ingestion: device parser (csrc/io.cu) vs the host routine on a
config-2-shaped file (1e5 rows x 20 nnz, values with 6 significant digits),
plus a repr-formatted file (17-digit values: host-converted lines)."""
import io, json, sys, time
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import problems


def text_of(data, fmt):
    f = data.features
    out = []
    for i in range(f.n_rows):
        c, v = f.row(i)
        out.append(f"{data.labels[i]:g} " + " ".join(f"{a + 1}:{fmt(b)}" for a, b in zip(c, v)))
    return "\n".join(out) + "\n"


cfg = problems.config2(seed=0)
d = cfg["data"]
for name, fmt in (("6 significant digits", lambda x: f"{x:.6g}"), ("repr (17 digits)", lambda x: repr(float(x)))):
    t = text_of(d, fmt)
    mb = len(t) / 1e6
    pb.parse_libsvm(io.StringIO(t[:200000].rsplit("\n", 1)[0] + "\n"), device="auto")  # warm
    res = {}
    for dev in ("auto", None):
        t0 = time.perf_counter()
        ds = pb.parse_libsvm(io.StringIO(t), device=dev)
        res["device" if dev else "host"] = time.perf_counter() - t0
    print(json.dumps({"file": name, "MB": round(mb, 1), "rows": ds.n_samples, "nnz": ds.features.nnz,
                      "device_s": round(res["device"], 4), "host_s": round(res["host"], 3),
                      "device_MBps": round(mb / res["device"], 1), "host_MBps": round(mb / res["host"], 2)}),
          flush=True)
