timeout 900 python tools/gpu/exp_batch_scatter.py "16:-1:128,8:-1:128,4:-1:128,2:-1:128,1:-1:128" 2>&1 | tail -5
bash tools/gpu/sc10.sh
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread --clock-control none -k regex:sps_group_batch --launch-skip 1 -c 1 python tools/gpu/prof_batch.py 0 16 2>&1 | grep -E "duration|inst_executed|issue_active|registers"
python -m pytest tests/test_gpu_batch.py -x -q 2>&1 | tail -2
