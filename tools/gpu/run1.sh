set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -m pytest tests/test_gpu_fast.py tests/test_gpu_acceptance.py -x -q 2>&1 | tail -15
timeout 300 python tools/exp_flags.py 2 30 4194304,0 2>&1 | tail -3
timeout 600 python tools/exp_flags.py 3 10 4194304,0 2>&1 | tail -3
timeout 600 python tools/exp_flags.py 4 5 4194304,0 2>&1 | tail -3
