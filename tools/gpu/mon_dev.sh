timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_abi.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 1500 python -c "
import json, sys
sys.argv=['bench.py']
import bench, torch
peak = 6537.6
for w in (3, 4):
    r = bench.big_config_bench(w, peak, with_cpu=False)
    t = r['time_to_1e-6']
    print(json.dumps({'config': w, 'value': r['value'], 'ttt_s': t['seconds'], 'ttt_epochs': t['epochs'], 'stop_the_world': t['stop_the_world'], 'final_rel': t['final_rel_gap']}), flush=True)
"
