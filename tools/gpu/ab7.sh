timeout 300 python tools/exp_flags.py 2 30 4194304,16777216,33554432 2>&1 | tail -1
timeout 600 python tools/exp_flags.py 3 10 4194304,16777216,33554432 2>&1 | tail -1
timeout 300 python tools/gpu/exp_ctas.py 2 16777216 2>&1 | tail -1
timeout 300 python tools/gpu/exp_ctas.py 2 4194304 2>&1 | tail -1
timeout 600 python tools/gpu/exp_ctas.py 3 16777216 2>&1 | tail -1
