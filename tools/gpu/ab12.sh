timeout 600 python tools/gpu/dbg_h1024.py 2000000 1024 2>&1 | tail -3
timeout 300 python tools/exp_flags.py 2 30 4194304,0 2>&1 | tail -1
timeout 600 python tools/exp_flags.py 3 10 4194304,0 2>&1 | tail -1
timeout 900 python tools/exp_flags.py 4 5 4194304,0 2>&1 | tail -1
