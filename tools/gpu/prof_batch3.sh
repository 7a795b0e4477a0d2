# ncu --set full of the lambda-batched kernel with the scattered hot blocks at B=16 and B=2
cap() {
  local name=$1; shift
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:sps_group_batch --launch-skip 1 -c 1 -o /tmp/$name -f "$@" > gpurun_out/$name.log 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/$name.raw.csv 2>/dev/null
}
cap prof_batch16_r02c python tools/gpu/prof_batch.py 0 16
cap prof_batch2_r02c python tools/gpu/prof_batch.py 0 2
python - <<'PY'
import csv
keys = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "lts__d_atomic_input_cycles_active.max", "lts__d_atomic_input_cycles_active.avg", "lts__t_sector_hit_rate.pct",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors_op_red.sum", "lts__t_requests_op_red.sum",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__t_requests_pipe_lsu_mem_global_op_red.sum", "lts__cycles_elapsed.max", "lts__cycles_elapsed.avg"]
for name in ("prof_batch16_r02c", "prof_batch2_r02c"):
    rows = list(csv.reader(open(f"gpurun_out/{name}.raw.csv")))
    hdr, units, vals = rows[0], rows[1], rows[2]
    print("==", name)
    for k in keys:
        if k in hdr:
            i = hdr.index(k); print(f"{k} = {vals[i]} {units[i]}")
PY
