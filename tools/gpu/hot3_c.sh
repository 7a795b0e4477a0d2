# hot3 with the asm CAS idiom (diag bit 27) vs hot2 (flag 8388608): configs 2/3/4
timeout 600 python tools/exp_flags.py 2 30 268435456,536870912,8388608 > gpurun_out/h3_ab2.log 2>&1; tail -1 gpurun_out/h3_ab2.log
timeout 900 python tools/exp_flags.py 3 10 268435456,536870912,8388608 > gpurun_out/h3_ab3.log 2>&1; tail -1 gpurun_out/h3_ab3.log
timeout 900 python tools/exp_flags.py 4 5 268435456,536870912,8388608 > gpurun_out/h3_ab4.log 2>&1; tail -1 gpurun_out/h3_ab4.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:sps_hot3 --launch-skip 1 -c 1 -o /tmp/h3c2 -f python tools/prof_async.py --batch 0 --wpc 32 --hp 24 --c 4 --per_launch 30 --hot_max 512 --warm 1 --epochs 1 --flags 268435456 > gpurun_out/h3_ncu.log 2>&1
ncu -i /tmp/h3c2.ncu-rep --page raw --csv > gpurun_out/h3c2.raw.csv 2>/dev/null
ncu -i /tmp/h3c2.ncu-rep --page source --csv --print-source sass > gpurun_out/h3c2.sass.csv 2>/dev/null
