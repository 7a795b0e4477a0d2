timeout 300 python tools/exp_flags.py 2 30 16777216,33554432,50331648 2>&1 | tail -1
timeout 600 python tools/exp_flags.py 3 10 16777216,33554432,50331648 2>&1 | tail -1
