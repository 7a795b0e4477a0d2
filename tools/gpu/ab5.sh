timeout 300 python tools/exp_flags.py 2 30 4194304,0,67108864 2>&1 | tail -1
timeout 600 python tools/exp_flags.py 3 10 4194304,0 2>&1 | tail -1
