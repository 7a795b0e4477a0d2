timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_step.py tests/test_gpu_acceptance.py tests/test_gpu_large.py tests/test_gpu_batch.py tests/test_gpu_fista.py tests/test_gpu_big_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 300 python -c "
import sys, json; sys.argv=['bench.py']
import bench
print(json.dumps(bench.config1_bench()))
"
