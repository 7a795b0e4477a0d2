timeout 300 python tools/exp_flags.py 2 30 4194304,0,16777216,50331648 2>&1 | tail -1
timeout 600 python tools/exp_flags.py 3 10 4194304,0,16777216 2>&1 | tail -1
