"""Copy the round's evidence from gpurun_out/ (scratch) into profiles/ (tracked):
the bench line + detail sidecar, the ncu launch list, the hot kernel's DRAM
traffic per launch (ncu --set full) and a metrics table of every capture.
    python tools/collect_profiles.py r02"""
import csv, json, shutil, sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
G, P = ROOT / "gpurun_out", ROOT / "profiles"
line = (G / f"bench_{tag}.json").read_text().strip().splitlines()[-1]
(P / f"bench_{tag}_latest.json").write_text(line + "\n")
shutil.copy(G / f"bench_detail_{tag}.json", P / f"bench_detail_{tag}.json")
shutil.copy(G / f"launches_{tag}.csv", P / f"launches_{tag}.csv")


def raw(name):
    rows = list(csv.reader(open(G / f"{name}.raw.csv")))
    return dict(zip(rows[0], rows[2]))


def num(v):
    return float(v.replace(",", ""))


KEYS = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sectors.sum", "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "lts__d_atomic_input_cycles_active.max.pct_of_peak_sustained_elapsed",
        "lts__t_sectors_srcunit_tex_op_red.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio"]
table = {}
for name in (f"prof_hot_{tag}_c2", f"prof_hot_{tag}_c3", f"prof_hot_{tag}_c4", f"prof_batch_{tag}"):
    try:
        r = raw(name)
    except FileNotFoundError:
        continue
    table[name] = {k: r[k] for k in KEYS if k in r}
(P / f"ncu_metrics_{tag}.json").write_text(json.dumps(table, indent=1) + "\n")
c2 = raw(f"prof_hot_{tag}_c2")
unit = {k: v for k, v in zip(*list(csv.reader(open(G / f"prof_hot_{tag}_c2.raw.csv")))[:2])}


def to_bytes(key):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit[key]]
    return int(round(num(c2[key]) * scale))


old = json.loads((P / f"ncu_traffic_{tag}.json").read_text())
rd, wr = to_bytes("dram__bytes_read.sum"), to_bytes("dram__bytes_write.sum")
old.update(dram_read_bytes=rd, dram_write_bytes=wr, dram_bytes_per_launch=rd + wr,
           lts_sectors=int(num(c2["lts__t_sectors.sum"])), warp_instructions=int(num(c2["smsp__inst_executed.sum"])),
           duration_ms_ncu=num(c2["gpu__time_duration.sum"]) * ({"ms": 1, "us": 1e-3, "s": 1e3}[unit["gpu__time_duration.sum"]]))
(P / f"ncu_traffic_{tag}.json").write_text(json.dumps(old, indent=1) + "\n")
print(json.dumps(table, indent=1))
