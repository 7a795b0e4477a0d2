set -x
timeout 300 python tools/exp_flags.py 2 30 4194304,0 2>&1 | tail -1
timeout 600 python tools/exp_flags.py 3 10 4194304,0 2>&1 | tail -1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:sps_hot_kernel --launch-skip 1 -c 1 -o gpurun_out/prof_hot_v2b -f python tools/prof_async.py --batch 0 --wpc 32 --hp 24 --c 4 --per_launch 30 --hot_max 512 --warm 1 --epochs 1 > gpurun_out/prof_hot_v2b.log 2>&1
