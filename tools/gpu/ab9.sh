timeout 600 python tools/gpu/dbg_h1024.py 2000000 1024 2>&1 | tail -4
timeout 600 python tools/gpu/dbg_h1024.py 2000000 512 2>&1 | tail -4
timeout 300 python tools/exp_flags.py 2 30 4194304,8388608,0 2>&1 | tail -1
timeout 600 python tools/exp_flags.py 3 10 4194304,8388608,0 2>&1 | tail -1
